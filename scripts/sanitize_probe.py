"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck) over every
hand-written asynchronous kernel family:
  * k_sls / k_sls_synth (PDL chain of back-to-back launches), k_gen_*, k_interact
  * k_mlp_chain (TMA -> tcgen05 -> TMEM fused stacks, mbarrier rings), bottom and top
  * k_gemm_tc per-layer GEMMs (REC_MLP=layers), MT = 2 weight-sharing tiles (B = 20480, RMC3
    shapes), k_gemm_group (MT-WnD grouped towers)
Each case runs a few batches and checks the CTRs against the CPU oracle (2e-2).
usage: compute-sanitizer --tool <tool> python scripts/sanitize_probe.py [--big 1]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import workloads as W
    from oracle import forward as fw, gen
    from paper_2203_07424_b200 import RecModel
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", type=int, default=1)
    a = ap.parse_args()
    cases = [("tiny_chain", W.TINY, {}, 300),
             ("rmc1_chain", W.small_variant(W.RMC1, 5000), {}, 300),
             ("rmc1_layers", W.small_variant(W.RMC1, 5000), {"REC_MLP": "layers"}, 300),
             ("rmc3_layers", W.small_variant(W.RMC3, 5000), {}, 257),
             ("mtwnd_group", W.small_variant(W.MTWND, 5000), {}, 200),
             ("rmc1_var", W.small_variant(W.RMC1, 5000).with_(pooling_lo=0, pooling_hi=40), {}, 129)]
    if a.big:
        cases.append(("rmc3_mt2", W.small_variant(W.RMC3, 5000), {}, 20480))
    worst = 0.0
    for name, cfg, env, B in cases:
        for k in ("REC_MLP",):
            os.environ.pop(k, None)
        os.environ.update(env)
        m = RecModel(cfg, seed=1, max_batch=B, streams=2)
        segs = W.random_segments(B, seed=3, max_seg=1000 if B > 4096 else 300)
        ind, off, dense = gen.gen_batch(cfg, 1, segs)
        tasks = cfg.tasks
        c = np.zeros(B * tasks, np.float32)
        m.rec_query(dense, ind, off, B, c)                       # eager caller-index path
        cv = torch.zeros(B * tasks, device="cuda")
        for s in range(2):                                        # captured graphs, 2 streams
            m.rec_synth_query_async(s, segs, cv)
        for s in range(2):
            m.rec_sync(s)
        assert np.array_equal(cv.cpu().numpy(), c), name
        if cfg.pooling_fixed and cfg.arch == W.ARCH_DLRM:         # PDL chain of SLS launches
            bst = np.arange(5, dtype=np.int64)
            bsegs = np.array([[7000 + k, 0, min(B, 256)] for k in range(4)], np.int32)
            m.rec_bench_sls(bsegs, bst, pdl=True)
        pick = np.arange(0, B, max(1, B // 24))[:24]
        q, it = gen.expand_segments(segs)
        sub = np.array([[q[k], it[k], 1] for k in pick], np.int32)
        i2, o2, d2 = gen.gen_batch(cfg, 1, sub)
        err = float(np.abs(c.reshape(B, tasks)[pick] - fw.forward(cfg, 1, d2, i2, o2).reshape(len(pick), tasks)).max())
        worst = max(worst, err)
        assert err <= 2e-2, (name, err)
        m.close()
        print(f"{name}: ok (max |ctr - oracle| = {err:.2e})", flush=True)
    print(f"sanitize_probe ok, worst {worst:.2e}")


if __name__ == "__main__":
    main()
