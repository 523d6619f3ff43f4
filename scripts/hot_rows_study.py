"""Hot-row partition study on one B200.

RMC1 shapes (10 x 1M x 32, pooling 80) with Zipf(0.9) indices (G2z, hot rows scattered).
Three handles of the same model:
  plain   - no remap, no window
  remap   - rec_hot_remap from a profiling sample, persisting window = capacity / models
  remap0  - rec_hot_remap, no window (the layout change alone)
For each: SLS GB/s of back-to-back synthetic-index launches (rec_bench_sls, PDL), saturation
QPS (bench.saturation, 16 co-located streams) and lambda* at p95 <= 20 ms (m = 8, d = 1024).
Prints one JSON object.
usage: python scripts/hot_rows_study.py [--index zipf|uniform] [--sla 1]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import bench
    import workloads as W
    from harness.sla import sla_search
    from paper_2203_07424_b200 import RecModel
    ap = argparse.ArgumentParser()
    ap.add_argument("--index", default="zipf", choices=["zipf", "uniform", "skew2"])
    ap.add_argument("--sla", type=int, default=1)
    ap.add_argument("--profile-items", type=int, default=4096)
    a = ap.parse_args()
    dist_id = {"zipf": W.INDEX_ZIPF, "uniform": W.INDEX_UNIFORM, "skew2": W.INDEX_SKEW2}[a.index]
    cfg = W.RMC1.with_(index_dist=dist_id)
    torch.cuda.set_device(0)
    out = {"workload": cfg.name, "index": a.index, "runs": {}}
    hbm = bench.peaks()[0]
    for tag in ("plain", "remap", "remap0"):
        m = RecModel(cfg, seed=1, max_batch=1024, streams=16)
        if tag != "plain":
            # profiling sample: the indices of profile-items synthetic items (host arrays, G2z)
            segs = W.random_segments(a.profile_items, seed=4242, max_seg=1000)
            big = RecModel(cfg.with_(rows=cfg.rows), seed=1, max_batch=a.profile_items, streams=1)
            ind, off, _ = big.rec_gen_batch(segs)
            big.close()
            rows = m.rec_hot_remap(ind, off, a.profile_items, window_bytes=0 if tag == "remap" else -1)
            out["runs"].setdefault(tag, {})["hot_rows_per_table"] = rows
        clk = bench.ClockSampler(0).__enter__()
        sat = bench.saturation(m, cfg, 1024, 16, 10, 3, 256, 40000, 0, 1, None)
        clk.__exit__(None, None, None)
        nb = 1000
        bseg = sat["tsegs"][:sat["tbstart"][nb]]
        ms = m.rec_bench_sls(bseg, sat["tbstart"][:nb + 1], pdl=True)
        gbs = bench.sls_bytes_per_item(cfg, synth=True) * int(bseg[:, 2].sum()) / (ms * 1e-3) / 1e9
        r = out["runs"].setdefault(tag, {})
        r.update({"saturation_qps": sat["value"], "sls_b2b_gbs": gbs, "sls_b2b_frac": gbs / hbm,
                  "sls_in_step_frac": bench.sls_bytes_per_item(cfg, synth=True) * sat["items"] /
                  (sat["ms_max"] * 1e-3) / 1e9 / hbm, "clocks": clk.summary(sat["t0"], sat["t1"])})
        if a.sla:
            lam, pr = sla_search(m, cfg, 1, 0, None, 8, 1024, 0.5 * sat["value"],
                                 int(max(100000, 1.5 * sat["value"])), cfg.sla_ms)
            r["lambda_star_qps"] = lam
            r["probes"] = pr
        m.close()
        torch.cuda.synchronize()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
