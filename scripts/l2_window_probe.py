"""L2 persisting window over the hot-row prefix (PAPER.md:552-558 hot-embedding
partition, whose B200 residue is an L2 window): SLS throughput for uniform vs skewed index
distributions with and without a persisting window (diagnostic; evidence in profiles/).

Skewed indices (INDEX_SKEW2, DESIGN.md R-index): r = u1 * u2 (product of two uniforms) scaled
to the table, so P(row < x R) = x - x ln x: the lowest 5 % of rows take 20 % of the lookups.
The interleaved arena puts row r of every table at (r T + t) D, so the hot rows of all
tables form ONE contiguous prefix that a single access-policy window covers.
usage: python scripts/l2_window_probe.py [--batch 1024] [--windows 0,32,64,96]"""
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
    from paper_2203_07424_b200 import RecModel
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--batches", type=int, default=400)
    ap.add_argument("--windows", default="0,32,64,96")
    ap.add_argument("--config", default="rmc1")
    ap.add_argument("--dists", default="uniform,skew2")
    a = ap.parse_args()
    base = W.SHORT[a.config]
    props = torch.cuda.get_device_properties(0)
    from cuda.bindings import runtime as rt
    attr = {}
    for nm in ("cudaDevAttrMaxPersistingL2CacheSize", "cudaDevAttrMaxAccessPolicyWindowSize",
               "cudaDevAttrL2CacheSize"):
        err, v = rt.cudaDeviceGetAttribute(getattr(rt.cudaDeviceAttr, nm), 0)
        attr[nm] = v
    out = {"config": base.name, "batch": a.batch, "device": attr, "rows": {}}
    per_item = base.num_tables * (base.pooling_lo * base.dim * 4 + base.dim * 4)
    dmap = {"uniform": W.INDEX_UNIFORM, "skew2": W.INDEX_SKEW2}
    for dist_name, dist in [(x, dmap[x]) for x in a.dists.split(",")]:
        for mb in [int(x) for x in a.windows.split(",")]:
            cfg = base.with_(index_dist=dist)
            m = RecModel(cfg, seed=1, max_batch=a.batch, streams=1, l2_persist_bytes=mb << 20)
            segs = np.array([[2000 + k, 0, a.batch] for k in range(a.batches)], np.int32)
            bst = np.arange(a.batches + 1, dtype=np.int64)
            m.rec_bench_sls(segs[:20], bst[:21], pdl=True)  # warm (and fill the window)
            for pdl in (True, False):
                ms = m.rec_bench_sls(segs, bst, pdl=pdl)
                us = 1e3 * ms / a.batches
                out["rows"][f"{dist_name}_win{mb}MB_{'pdl' if pdl else 'plain'}"] = {
                    "us_per_launch": round(us, 2),
                    "algorithmic_GBps": round(per_item * a.batch / (us * 1e-6) / 1e9, 1)}
            m.close()
            torch.cuda.synchronize()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
