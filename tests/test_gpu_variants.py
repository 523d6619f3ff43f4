"""Every environment-selectable kernel variant of the shipped library gives the default
path's bits (DESIGN.md §10 knob table).  Each variant is a different kernel or schedule for
the same arithmetic: the SLS accumulates every bag in index order (TMA variant: exact with
int8 x 2^e tables in any order, G4), every GEMM output element accumulates over K in the same
order whatever the tiling (batch invariance), so CTRs must be bit-identical to
the default path and within 2e-2 of the oracle.  Both the caller-index path (rec_query) and
the captured-graph path (rec_synth_query_async) are checked.
"""
import numpy as np
import pytest

import workloads as W
from oracle import forward as fw, gen

pytestmark = pytest.mark.gpu

KNOBS = ["REC_SLS", "REC_GEMM_2SM", "REC_GEMM_NARROW", "REC_GEMM_MT1", "REC_FUSE_DENSE",
         "REC_INTERACT_PF", "REC_HOT_POLICY", "REC_MLP", "REC_CHAIN_PDL", "REC_PDL",
         "REC_FUSE_INTERACT", "REC_TOWER_GROUP", "REC_GEMM_STAGES", "REC_INTERACT_WPC",
         "REC_CHAIN_SMEM", "REC_CHAIN_STAGES", "REC_SERVE_DEPTH",
         "REC_SERVE_THREADS", "REC_GREEN_SMS", "REC_PRIO", "REC_GEMM_BN64", "REC_SLS_GRID", "REC_GEMM_MT2", "REC_CHAIN_PERSISTENT", "REC_P2P_FENCE", "REC_INTERACT_BLOCKED", "REC_P2P_LL", "REC_GEMM_2SM_SERVE"]


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__
    __graft_entry__.build()


@pytest.fixture
def clean_env(monkeypatch):
    for k in KNOBS:
        monkeypatch.delenv(k, raising=False)
    return monkeypatch


def _run(cfg, B, segs, l2=0):
    import torch
    from paper_2203_07424_b200 import RecModel
    m = RecModel(cfg, seed=1, max_batch=B, l2_persist_bytes=l2)
    ind, off, dense = gen.gen_batch(cfg, 1, segs)
    # graph path FIRST on a fresh handle: no earlier launch has left this batch's pooled
    # vectors in the workspace, so a kernel that skips bags cannot pass on stale X
    cv = torch.zeros(B * cfg.tasks, device="cuda")
    m.rec_synth_query_async(0, segs, cv)
    m.rec_sync(0)
    graph = cv.cpu().numpy()
    eager = np.zeros(B * cfg.tasks, np.float32)
    m.rec_query(dense, ind, off, B, eager)
    m.close()
    return eager, graph


RMC1 = W.small_variant(W.RMC1, 20000)
RMC3 = W.small_variant(W.RMC3, 20000)
MTWND = W.small_variant(W.MTWND, 20000)
TINY = W.TINY

# (variant id, env, config, batch, l2 persisting bytes)
VARIANTS = [
    ("sls_tma", {"REC_SLS": "tma"}, RMC1, 700, 0),
    ("sls_no_pdl", {"REC_PDL": "0"}, RMC1, 700, 0),
    ("sls_interleaved_grid", {"REC_SLS_GRID": "1"}, RMC1, 1024, 0),
    ("sls_interleaved_grid_rmc2", {"REC_SLS_GRID": "1"}, W.small_variant(W.RMC2, 4096), 1024, 0),
    ("sls_interleaved_grid_rmc1_big", {"REC_SLS_GRID": "1"}, RMC1, 4096, 0),
    ("hot_policy_l2_window", {"REC_HOT_POLICY": "1"}, RMC1.with_(index_dist=W.INDEX_SKEW2), 700, 8 << 20),
    ("l2_window", {}, RMC1, 700, 8 << 20),
    ("fuse_dense", {"REC_FUSE_DENSE": "1"}, RMC1, 700, 0),
    ("fuse_dense_rmc3", {"REC_FUSE_DENSE": "1"}, RMC3, 700, 0),
    ("fuse_dense_tma", {"REC_FUSE_DENSE": "1", "REC_SLS": "tma"}, RMC1, 700, 0),
    ("interact_pf", {"REC_INTERACT_PF": "1"}, RMC1, 700, 0),
    ("interact_wpc2", {"REC_INTERACT_WPC": "2"}, RMC1, 700, 0),
    ("interact_per_pair_rmc2", {"REC_INTERACT_BLOCKED": "0"}, W.small_variant(W.RMC2, 4096), 700, 0),
    ("interact_blocked_rmc1", {"REC_INTERACT_BLOCKED": "4"}, RMC1, 700, 0),
    ("mlp_layers_tiny", {"REC_MLP": "layers"}, TINY, 300, 0),
    ("mlp_layers_rmc1", {"REC_MLP": "layers"}, RMC1, 700, 0),
    ("chain_no_pdl", {"REC_CHAIN_PDL": "0"}, RMC1, 700, 0),
    ("chain_2stage", {"REC_CHAIN_STAGES": "2"}, RMC1, 700, 0),
    ("chain_big_budget", {"REC_CHAIN_SMEM": "227"}, RMC1, 700, 0),
    ("gemm_narrow", {"REC_GEMM_NARROW": "148"}, RMC3, 700, 0),
    ("gemm_bn64_rmc3", {"REC_GEMM_BN64": "1"}, RMC3, 1024, 0),
    ("gemm_mt2_serving_rmc3", {"REC_GEMM_MT2": "1"}, RMC3, 1024, 0),
    ("gemm_bn64_rmc2", {"REC_GEMM_BN64": "1"}, W.small_variant(W.RMC2, 4096), 700, 0),
    ("gemm_stages2", {"REC_GEMM_STAGES": "2"}, RMC3, 700, 0),
    ("gemm_2sm_large", {"REC_GEMM_2SM": "1"}, RMC3, 20480, 0),
    ("gemm_2sm_serving_rmc3", {"REC_GEMM_2SM_SERVE": "2"}, RMC3, 1024, 0),
    ("gemm_2sm_serving_rmc3_odd", {"REC_GEMM_2SM_SERVE": "4"}, RMC3, 700, 0),
    ("gemm_2sm_serving_rmc2", {"REC_GEMM_2SM_SERVE": "2"}, W.small_variant(W.RMC2, 4096), 700, 0),
    ("gemm_mt1_large", {"REC_GEMM_MT1": "1"}, RMC3, 20480, 0),
    ("gemm_narrow_towers", {"REC_GEMM_NARROW": "148"}, MTWND, 700, 0),
    ("towers_per_task", {"REC_TOWER_GROUP": "0"}, MTWND, 700, 0),
    ("prio_dense", {"REC_PRIO": "1"}, RMC1, 700, 0),
]


@pytest.mark.parametrize("vid,env,cfg,B,l2", VARIANTS, ids=[v[0] for v in VARIANTS])
def test_variant_bits_equal_default(vid, env, cfg, B, l2, clean_env):
    segs = W.random_segments(B, seed=77, max_seg=1000 if B > 4096 else 300)
    ref_e, ref_g = _run(cfg, B, segs)                     # default kernels
    assert np.array_equal(ref_e, ref_g)
    for k, v in env.items():
        clean_env.setenv(k, v)
    got_e, got_g = _run(cfg, B, segs, l2)
    assert np.array_equal(got_e, ref_e), vid
    assert np.array_equal(got_g, ref_g), vid
    # and the oracle bar on sampled items
    q, it = gen.expand_segments(segs)
    pick = np.random.default_rng(1).choice(B, size=min(B, 48), replace=False)
    sub = np.array([[q[k], it[k], 1] for k in pick], np.int32)
    i2, o2, d2 = gen.gen_batch(cfg, 1, sub)
    exp = fw.forward(cfg, 1, d2, i2, o2)
    got = got_g.reshape(B, -1)[pick]
    assert np.abs(got - exp.reshape(len(pick), -1)).max() <= 2e-2


@pytest.mark.parametrize("env", [{"REC_SERVE_DEPTH": "2"}, {"REC_SERVE_THREADS": "4"}],
                         ids=["serve_depth2", "serve_threads4"])
def test_serving_variants_same_ctr(env, clean_env):
    """The real-clock serving dispatcher variants (two batches in flight per stream, several
    dispatcher threads) change batching only; every item's CTR bits are batch-invariant, so
    rec_serve's per-item CTRs equal the default dispatcher's."""
    from paper_2203_07424_b200 import RecModel
    cfg = RMC1
    tr = W.poisson_trace(20000.0, 400, seed=5)
    out = {}
    for name, e in (("default", {}), ("variant", env)):
        for k, v in e.items():
            clean_env.setenv(k, v)
        m = RecModel(cfg, seed=1, max_batch=1024, streams=4)
        r = m.rec_serve(tr, 1e9, streams=4, max_batch=1024, want_ctr=True)
        assert r["completed"] == len(tr)
        out[name] = r["ctr"]
        m.close()
    assert np.array_equal(out["default"], out["variant"])
