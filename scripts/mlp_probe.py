"""Dense-stage timing (diagnostic): fused MLP chain vs per-layer GEMMs, small and large
batches, bf16 tensor-pipe utilisation = algorithmic flops / time / peak.
usage: [REC_MLP=layers] [REC_CARVEOUT=max] python scripts/mlp_probe.py --config rmc3"""
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
    ap.add_argument("--batches", default="1024,4096,16384,65536")
    a = ap.parse_args()
    cfg = W.SHORT[a.config]
    bs = [int(x) for x in a.batches.split(",")]
    m = RecModel(cfg.with_(rows=1000), seed=1, max_batch=max(bs))
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 1590.0
    fb = sum(2 * x * y for x, y in zip(cfg.bottom[:-1], cfg.bottom[1:]))
    w = [cfg.dim + cfg.num_tables * (cfg.num_tables + 1) // 2] + list(cfg.top)
    ft = sum(2 * x * y for x, y in zip(w[:-1], w[1:]))
    out = {"config": cfg.name, "mlp": os.environ.get("REC_MLP", "chain"),
           "carveout": os.environ.get("REC_CARVEOUT", "default"), "rows": {}}
    for B in bs:
        it = 200 if B <= 4096 else 50
        tb = m.rec_bench_mlp(0, B, it)
        ti = m.rec_bench_mlp(2, B, it)
        tt = m.rec_bench_mlp(1, B, it)
        out["rows"][B] = {"bottom_us": round(1e3 * tb, 2), "interact_us": round(1e3 * ti, 2),
                          "interact_top_us": round(1e3 * tt, 2),
                          "bottom_tc_frac": round(fb * B / (tb * 1e-3) / 1e12 / peak, 4),
                          "top_tc_frac": round(ft * B / ((tt - ti) * 1e-3) / 1e12 / peak, 4) if tt > ti else None}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
