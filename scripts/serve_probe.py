"""Serving probe (diagnostic): rec_serve at a fixed offered Poisson rate for several stream
counts; prints achieved QPS, p95, batches, mean batch size.
usage: python scripts/serve_probe.py --config rmc3 --rate 300000 --streams 8,16"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import workloads as W
    from paper_2203_07424_b200 import RecModel
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="rmc1")
    ap.add_argument("--rate", type=float, default=250000)
    ap.add_argument("--queries", type=int, default=100000)
    ap.add_argument("--streams", default="8,16")
    ap.add_argument("--d", type=int, default=1024)
    ap.add_argument("--tau", type=float, default=0.0)
    a = ap.parse_args()
    cfg = W.SHORT[a.config]
    ms = [int(x) for x in a.streams.split(",")]
    m = RecModel(cfg, seed=1, max_batch=a.d, streams=max(ms))
    out = {}
    for st in ms:
        tr = W.poisson_trace(a.rate, a.queries, seed=12)
        m.rec_profile(False)  # resets the host-time counters of the submit path
        rep = m.rec_serve(tr, cfg.sla_ms, st, a.d, fusion_timeout_ms=a.tau, warmup_frac=0.1)
        out[st] = {k: (round(v, 3) if isinstance(v, float) else v) for k, v in rep.items()
                   if k in ("offered_qps", "achieved_qps", "p50_ms", "p95_ms", "batches", "mean_batch",
                            "stable", "breakdown_ms")}
        nb = max(1, rep.get("batches", 1))
        # host microseconds per batch: node-param update, graph launch, slot wait, whole submit
        out[st]["host_us_per_batch"] = [round(m.rec_profile_read(k)[0] * 1e3 / nb, 2) for k in (5, 6, 7, 8)]
    print(json.dumps({"config": cfg.name, "rate": a.rate, "tau": a.tau, "by_streams": out}))


if __name__ == "__main__":
    main()
