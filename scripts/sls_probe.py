"""Probe what bounds the SLS gather on a B200 (diagnostic, not part of the product).

Times the SLS kernel (CUDA events on its stream, via rec_profile) for RMC1-shaped batches
whose indices are drawn from a restricted row range (footprint sweep: TLB reach / L2
residency) or sorted within each bag (DRAM page locality), for both SLS implementations.
usage: python scripts/sls_probe.py [--batch 1024] [--iters 200]
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
    import workloads as W
    from paper_2203_07424_b200 import RecModel, KERNEL_SLS

    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--iters", type=int, default=200)
    ap.add_argument("--config", default="rmc1")
    ap.add_argument("--pooling", default="", help="with --synth: comma list of fixed pooling L")
    ap.add_argument("--synth", default="", help="comma list of batch sizes: time the in-kernel "
                    "Philox-index SLS (serving path) instead of the footprint sweep")
    a = ap.parse_args()
    if a.synth:
        return synth(a)
    cfg = W.SHORT[a.config]
    B, T, L, D = a.batch, cfg.num_tables, cfg.pooling_lo, cfg.dim
    m = RecModel(cfg, seed=1, max_batch=B, streams=1)
    rng = np.random.default_rng(0)
    dense = torch.zeros((B, cfg.dense_dim), device="cuda")
    off = torch.arange(T * B + 1, dtype=torch.int32, device="cuda") * L
    ctr = torch.zeros(B, device="cuda")
    per_item = T * (L * D * 4 + L * 4 + 4) + T * D * 4
    res = {}
    for name, span, sort in [("full", cfg.rows, False), ("full_sorted_in_bag", cfg.rows, True),
                             ("rows_400k", 400_000, False), ("rows_200k", 200_000, False),
                             ("rows_100k", 100_000, False), ("rows_20k", 20_000, False)]:
        idx = rng.integers(0, span, size=(T * B, L)).astype(np.int32)
        if sort:
            idx.sort(axis=1)
        iv = torch.from_numpy(idx.reshape(-1)).cuda()
        for _ in range(10):
            m.rec_query_async(0, dense, iv, off, T * B * L, B, ctr)
        m.rec_sync(0)
        m.rec_profile(True)
        for _ in range(a.iters):
            m.rec_query_async(0, dense, iv, off, T * B * L, B, ctr)
        ms, n = m.rec_profile_read(KERNEL_SLS)
        m.rec_profile(False)
        us = 1e3 * ms / n
        res[name] = {"us": round(us, 2), "GBps": round(per_item * B / (us * 1e-6) / 1e9, 1),
                     "footprint_MB": round(span * T * D * 4 / 1e6, 1)}
    print(json.dumps({"impl": os.environ.get("REC_SLS_IMPL", "async"), "batch": B, "config": a.config,
                      "results": res}))


def synth(a):
    import torch
    import workloads as W
    from paper_2203_07424_b200 import RecModel, KERNEL_SLS
    res = {}
    pools = [int(x) for x in a.pooling.split(",")] if a.pooling else [None]
    for B, Lp in [(int(x), p) for x in a.synth.split(",") for p in pools]:
        cfg = W.SHORT[a.config]
        if Lp:
            cfg = cfg.with_(pooling_lo=Lp, pooling_hi=Lp)
        per_item = cfg.num_tables * (cfg.pooling_lo * cfg.dim * 4 + cfg.dim * 4)
        m = RecModel(cfg, seed=1, max_batch=B, streams=1)
        segs = np.array([[q, 0, 1] for q in range(B)], np.int32)
        ctr = torch.zeros(B, device="cuda")
        for _ in range(10):
            m.rec_synth_query_async(0, segs, ctr)
        m.rec_sync(0)
        m.rec_profile(True)
        for _ in range(a.iters):
            m.rec_synth_query_async(0, segs, ctr)
        m.rec_sync(0)
        ms, n = m.rec_profile_read(KERNEL_SLS)
        m.rec_profile(False)
        us = 1e3 * ms / n
        bsegs = np.array([[1000 + k, 0, B] for k in range(a.iters)], np.int32)  # distinct rows
        bst = np.arange(a.iters + 1, dtype=np.int64)
        us_b2b = 1e3 * m.rec_bench_sls(bsegs, bst, pdl=False) / a.iters
        us_pdl = 1e3 * m.rec_bench_sls(bsegs, bst, pdl=True) / a.iters
        res[f"B{B}_L{cfg.pooling_lo}"] = {"us": round(us, 2),
                                          "GBps": round(per_item * B / (us * 1e-6) / 1e9, 1),
                                          "b2b_us": round(us_b2b, 2),
                                          "b2b_GBps": round(per_item * B / (us_b2b * 1e-6) / 1e9, 1),
                                          "pdl_us": round(us_pdl, 2),
                                          "pdl_GBps": round(per_item * B / (us_pdl * 1e-6) / 1e9, 1)}
        del m
    print(json.dumps({"mode": "synth", "lib": os.environ.get("REC_LIB_PATH", "default"),
                      "config": a.config, "results": res}))


if __name__ == "__main__":
    main()
