"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bars (BASELINE.json north_star):
  * synthetic indices / offsets / dense: bit-exact
  * SLS pooled fp32: bit-exact vs the oracle's fp32-sequential order (the kernel
    accumulates each bag in index order), and in int8-exact mode bit-exact vs fp64;
    fp32 value mode additionally within 1e-5 * sum|x| of the fp64 sum
  * CTR: |gpu - oracle| <= 2e-2 absolute, with the oracle's non-vacuity guard
Sizes span several 128-row GEMM tiles with a ragged tail, plus B = 1 and full-size
(1M-row) tables on sampled items.
"""
import numpy as np
import pytest

import workloads as W
from oracle import forward as fw, gen

pytestmark = pytest.mark.gpu

CTR_TOL = 2e-2


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__
    __graft_entry__.build()


def _model(cfg, **kw):
    from paper_2203_07424_b200 import RecModel
    return RecModel(cfg, seed=1, **kw)


def _oracle_pooled_fp32(cfg, ind, off, B):
    shift = gen.emb_shift(cfg.pooling_lo, cfg.pooling_hi)
    f = lambda t, r: gen.table_values(1, t, r, cfg.dim, shift, cfg.value_mode)
    return fw.sls(f, cfg.num_tables, B, cfg.dim, ind, off, fp32_sequential=True)


CASES = [
    ("tiny", W.TINY, 64),
    ("tiny_ragged", W.TINY, 300),
    ("rmc1", W.small_variant(W.RMC1, 20000), 300),
    ("rmc2", W.small_variant(W.RMC2, 4096), 200),
    ("rmc3", W.small_variant(W.RMC3, 20000), 257),
    ("rmc1_var", W.small_variant(W.RMC1, 20000).with_(pooling_lo=20, pooling_hi=160), 129),
    ("rmc1_skew", W.small_variant(W.RMC1, 20000).with_(index_dist=W.INDEX_SKEW2), 64),
    ("rmc1_zipf", W.small_variant(W.RMC1, 20000).with_(index_dist=W.INDEX_ZIPF), 129),
    ("rmc1_zipf_var", W.small_variant(W.RMC1, 20000).with_(index_dist=W.INDEX_ZIPF, pooling_lo=20,
                                                          pooling_hi=160), 65),
    ("rmc1_fp32", W.small_variant(W.RMC1, 20000).with_(value_mode=W.REC_VALUES_FP32), 150),
    ("one_hot", W.small_variant(W.TINY, 5000).with_(pooling_lo=1, pooling_hi=1), 77),
]


@pytest.mark.parametrize("name,cfg,B", CASES, ids=[c[0] for c in CASES])
def test_gen_batch_bit_exact(name, cfg, B):
    m = _model(cfg, max_batch=B)
    segs = W.random_segments(B, seed=21)
    ind, off, dense = gen.gen_batch(cfg, 1, segs)
    gi, go, gd = m.rec_gen_batch(segs)
    assert np.array_equal(go, off)
    assert np.array_equal(gi, ind)
    assert np.array_equal(gd, dense)


@pytest.mark.parametrize("name,cfg,B", CASES, ids=[c[0] for c in CASES])
def test_forward_parity(name, cfg, B):
    m = _model(cfg, max_batch=B)
    segs = W.random_segments(B, seed=22)
    ind, off, dense = gen.gen_batch(cfg, 1, segs)
    ctr = np.zeros(B, np.float32)
    pooled = np.zeros((B, cfg.num_tables, cfg.dim), np.float32)
    logit = np.zeros(B, np.float32)
    m.rec_query_debug(dense, ind, off, B, ctr, pooled=pooled, logits=logit)
    exp = fw.forward(cfg, 1, dense, ind, off, return_all=True)
    # SLS: bit-exact against the fp32-sequential definition
    assert np.array_equal(pooled, _oracle_pooled_fp32(cfg, ind, off, B))
    if cfg.value_mode == W.REC_VALUES_INT8_EXACT:
        assert np.array_equal(pooled.astype(np.float64), exp["pooled"])
    else:
        shift = gen.emb_shift(cfg.pooling_lo, cfg.pooling_hi)
        absum = fw.sls(lambda t, r: np.abs(gen.table_values(1, t, r, cfg.dim, shift, 1)),
                       cfg.num_tables, B, cfg.dim, ind, off)
        assert np.all(np.abs(pooled - exp["pooled"]) <= 1e-5 * absum + 1e-30)
    # CTR within 2e-2, non-vacuous
    err = np.abs(ctr.astype(np.float64) - exp["ctr"])
    assert err.max() <= CTR_TOL, (err.max(), np.argmax(err))
    assert exp["logit"].std() > 0.5
    # logits agree too (looser: bf16 hidden activations)
    assert np.abs(logit - exp["logit"]).max() < 0.15


def test_batch_one_and_batch_invariance():
    cfg = W.small_variant(W.RMC1, 20000)
    m = _model(cfg, max_batch=1024)
    segs = W.random_segments(1024, seed=5)
    ind, off, dense = gen.gen_batch(cfg, 1, segs)
    full = np.zeros(1024, np.float32)
    m.rec_query(dense, ind, off, 1024, full)
    # the same items in batches of 1, 7 and 1024 produce identical CTR bits
    q, it = gen.expand_segments(segs)
    for d in (1, 7, 333):
        for start in (0, 500, 1024 - d):
            sub = np.array([[q[k], it[k], 1] for k in range(start, start + d)], np.int32)
            i2, o2, d2 = gen.gen_batch(cfg, 1, sub)
            c2 = np.zeros(d, np.float32)
            m.rec_query(d2, i2, o2, d, c2)
            assert np.array_equal(c2, full[start:start + d]), (d, start)


def test_device_pointers_match_host():
    import torch
    cfg = W.small_variant(W.RMC2, 4096)
    B = 130
    m = _model(cfg, max_batch=B)
    ind, off, dense = gen.gen_batch(cfg, 1, W.random_segments(B, seed=8))
    c_host = np.zeros(B, np.float32)
    m.rec_query(dense, ind, off, B, c_host)
    dv = torch.from_numpy(dense).cuda()
    iv = torch.from_numpy(ind).cuda()
    ov = torch.from_numpy(off).cuda()
    cv = torch.zeros(B, device="cuda")
    m.rec_query(dv, iv, ov, B, cv)
    assert np.array_equal(cv.cpu().numpy(), c_host)
    # async path on a second stream slot gives the same bits
    m2 = _model(cfg, max_batch=B, streams=2)
    cv2 = torch.zeros(B, device="cuda")
    m2.rec_query_async(1, dv, iv, ov, int(off[-1]), B, cv2)
    m2.rec_sync(1)
    assert np.array_equal(cv2.cpu().numpy(), c_host)
    # async path with HOST inputs/outputs (pinned and pageable): same bits
    pin = [torch.from_numpy(x).pin_memory() for x in (dense, ind, off)]
    cp = torch.zeros(B).pin_memory()
    m2.rec_query_async(0, pin[0], pin[1], pin[2], int(off[-1]), B, cp)
    c_np = np.zeros(B, np.float32)
    m2.rec_query_async(1, dense, ind, off, int(off[-1]), B, c_np)
    m2.rec_sync(0)
    m2.rec_sync(1)
    assert np.array_equal(cp.numpy(), c_host)
    assert np.array_equal(c_np, c_host)


def test_synth_query_matches_host_inputs():
    import torch
    cfg = W.small_variant(W.RMC3, 20000)
    B = 300
    m = _model(cfg, max_batch=B)
    segs = W.random_segments(B, seed=9)
    ind, off, dense = gen.gen_batch(cfg, 1, segs)
    c_host = np.zeros(B, np.float32)
    m.rec_query(dense, ind, off, B, c_host)
    cv = torch.zeros(B, device="cuda")
    m.rec_synth_query_async(0, segs, cv)
    m.rec_sync(0)
    assert np.array_equal(cv.cpu().numpy(), c_host)


def test_edge_cases_empty_bags_duplicates_errors():
    from paper_2203_07424_b200 import RecError
    cfg = W.small_variant(W.TINY, 1000)
    T, B, D = cfg.num_tables, 5, cfg.dim
    m = _model(cfg, max_batch=8)
    rng = np.random.default_rng(0)
    lens = np.array([0, 3, 0, 1, 5] * T)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    ind = rng.integers(0, 1000, size=off[-1]).astype(np.int32)
    ind[1:3] = ind[0] if off[-1] > 3 else ind[1:3]               # duplicates
    dense = (rng.integers(-128, 128, size=(B, cfg.dense_dim)) / 128.0).astype(np.float32)
    ctr = np.zeros(B, np.float32)
    pooled = np.zeros((B, T, D), np.float32)
    m.rec_query_debug(dense, ind, off, B, ctr, pooled=pooled)
    exp = fw.forward(cfg, 1, dense, ind, off, return_all=True)
    assert np.array_equal(pooled.astype(np.float64), exp["pooled"])
    assert np.all(pooled[0] == 0) and np.all(pooled[2] == 0)
    assert np.abs(ctr - exp["ctr"]).max() <= CTR_TOL
    bad = ind.copy()
    bad[2] = 1000                                                 # == rows: out of range
    with pytest.raises(RecError) as ei:
        m.rec_query(dense, bad, off, B, ctr)
    assert ei.value.status == -2
    bad[2] = -1
    with pytest.raises(RecError) as ei:
        m.rec_query(dense, bad, off, B, ctr)
    assert ei.value.status == -2
    boff = off.copy()
    boff[3] = boff[2] - 1
    with pytest.raises(RecError) as ei:
        m.rec_query(dense, ind, boff, B, ctr)
    assert ei.value.status == -3
    with pytest.raises(RecError) as ei:
        m.rec_query(dense, ind, off, 9, np.zeros(9, np.float32))   # > max_batch
    assert ei.value.status == -1
    # the model still works after errors
    m.rec_query(dense, ind, off, B, ctr)


def test_device_offsets_validation():
    import torch
    from paper_2203_07424_b200 import RecError
    cfg = W.small_variant(W.TINY, 1000)
    m = _model(cfg, max_batch=16)
    ind, off, dense = gen.gen_batch(cfg, 1, W.random_segments(16, seed=3))
    boff = off.copy()
    boff[5] = boff[4] - 1
    with pytest.raises(RecError) as ei:
        m.rec_query(torch.from_numpy(dense).cuda(), torch.from_numpy(ind).cuda(),
                    torch.from_numpy(boff).cuda(), 16, torch.zeros(16, device="cuda"))
    assert ei.value.status == -3


@pytest.mark.parametrize("name", ["rmc1", "rmc2", "rmc3", "mtwnd"])
def test_full_size_sampled(name):
    """BASELINE sizes (1M rows/table, B = 1024, the bench launch configuration): sampled items."""
    import torch
    cfg = W.SHORT[name]
    B = 1024
    N = max(cfg.tasks, 1)
    m = _model(cfg, max_batch=B)
    segs = W.random_segments(B, seed=31)
    cv = torch.zeros(B * N, device="cuda")
    m.rec_synth_query_async(0, segs, cv)
    m.rec_sync(0)
    ctr = cv.cpu().numpy().reshape(B, N) if N > 1 else cv.cpu().numpy()
    q, it = gen.expand_segments(segs)
    pick = np.random.default_rng(0).choice(B, size=24 if name == "rmc2" else 48, replace=False)
    sub = np.array([[q[k], it[k], 1] for k in pick], np.int32)
    i2, o2, d2 = gen.gen_batch(cfg, 1, sub)
    exp = fw.forward(cfg, 1, d2, i2, o2)
    assert np.abs(ctr[pick] - exp).max() <= CTR_TOL


def test_large_batch_weight_sharing_gemm_invariance():
    """B = 20480 on RMC3 shapes routes the 2560x512 bottom layer through the 2-M-tile
    (weight-sharing) tcgen05 GEMM; every item's CTR must equal the small-batch result bit for
    bit (batch invariance) and the oracle within 2e-2 on sampled items."""
    import torch
    cfg = W.small_variant(W.RMC3, 20000)
    B = 20480
    m = _model(cfg, max_batch=B)
    segs = W.random_segments(B, seed=41, max_seg=1000)
    cv = torch.zeros(B, device="cuda")
    m.rec_synth_query_async(0, segs, cv)
    m.rec_sync(0)
    big = cv.cpu().numpy()
    q, it = gen.expand_segments(segs)
    pick = np.random.default_rng(3).choice(B, size=40, replace=False)
    sub = np.array([[q[k], it[k], 1] for k in pick], np.int32)
    small = _model(cfg, max_batch=64)
    cs = torch.zeros(40, device="cuda")
    small.rec_synth_query_async(0, sub, cs)
    small.rec_sync(0)
    assert np.array_equal(cs.cpu().numpy(), big[pick])
    i2, o2, d2 = gen.gen_batch(cfg, 1, sub)
    exp = fw.forward(cfg, 1, d2, i2, o2)
    assert np.abs(big[pick] - exp).max() <= CTR_TOL


def test_mtwnd_parity_and_invariance():
    """MT-WnD (R26-R29): one-hot lookups bit-exact, per-task CTRs within 2e-2
    of the oracle, identical bits whatever the batch, device-synth == host inputs."""
    import torch
    cfg = W.small_variant(W.MTWND, 20000)
    N = cfg.tasks
    m = _model(cfg, max_batch=300)
    for B in (1, 300):
        segs = W.random_segments(B, seed=50 + B)
        ind, off, dense = gen.gen_batch(cfg, 1, segs)
        assert dense.shape == (B, 0)
        gi, go, gd = m.rec_gen_batch(segs)
        assert np.array_equal(gi, ind) and np.array_equal(go, off)
        ctr = np.zeros((B, N), np.float32)
        pooled = np.zeros((B, cfg.num_tables, cfg.dim), np.float32)
        logit = np.zeros((B, N), np.float32)
        m.rec_query_debug(dense, ind, off, B, ctr, pooled=pooled, logits=logit)
        exp = fw.forward(cfg, 1, dense, ind, off, return_all=True)
        assert np.array_equal(pooled.astype(np.float64), exp["pooled"])
        assert np.abs(ctr - exp["ctr"]).max() <= CTR_TOL
        assert np.abs(logit - exp["logit"]).max() < 0.15
        if B == 300:
            assert np.all(exp["logit"].std(axis=0) > 0.5)
            # batch invariance on a sub-batch, device-synthesised path
            q, it = gen.expand_segments(segs)
            sub = np.array([[q[k], it[k], 1] for k in range(40, 77)], np.int32)
            cs = torch.zeros(37 * N, device="cuda")
            m.rec_synth_query_async(0, sub, cs)
            m.rec_sync(0)
            assert np.array_equal(cs.cpu().numpy().reshape(37, N), ctr[40:77])


def test_bench_sls_measurement_call():
    """rec_bench_sls (the roofline measurement) launches the production SLS kernel over a
    batch sequence with and without PDL, returns positive times, rejects bad arguments and
    leaves the model serving identical bits afterwards."""
    import torch
    from paper_2203_07424_b200 import RecError
    cfg = W.small_variant(W.RMC1, 20000)
    m = _model(cfg, max_batch=256)
    segs = W.random_segments(200, seed=61)
    before = torch.zeros(200, device="cuda")
    m.rec_synth_query_async(0, segs, before)
    m.rec_sync(0)
    bsegs = np.array([[5000 + k, 0, 256] for k in range(8)], np.int32)
    bst = np.arange(9, dtype=np.int64)
    assert m.rec_bench_sls(bsegs, bst, pdl=True) > 0
    assert m.rec_bench_sls(bsegs, bst, pdl=False) > 0
    with pytest.raises(RecError):
        m.rec_bench_sls(np.array([[1, 0, 300]], np.int32), np.array([0, 1], np.int64))  # > max_batch
    after = torch.zeros(200, device="cuda")
    m.rec_synth_query_async(0, segs, after)
    m.rec_sync(0)
    assert np.array_equal(after.cpu().numpy(), before.cpu().numpy())


@pytest.mark.parametrize("name,cfg,B", [("tiny", W.TINY, 300),
                                        ("rmc1", W.small_variant(W.RMC1, 20000), 300),
                                        ("rmc3", W.small_variant(W.RMC3, 20000), 1),
                                        ("rmc1_fp32", W.small_variant(W.RMC1, 20000).with_(
                                            value_mode=W.REC_VALUES_FP32), 257)])
def test_fused_interaction_bit_identical(name, cfg, B, monkeypatch):
    """The dot interaction computed inside the top chain (REC_FUSE_INTERACT=1) gives the same CTR and
    logit bits as the separate k_interact kernel + TMA-loaded A (REC_FUSE_INTERACT=0), and
    both stay within the oracle bar."""
    import torch
    segs = W.random_segments(B, seed=31)
    ind, off, dense = gen.gen_batch(cfg, 1, segs)
    out = {}
    for fuse in ("1", "0"):
        monkeypatch.setenv("REC_FUSE_INTERACT", fuse)
        m = _model(cfg, max_batch=max(B, 64))
        ctr = np.zeros(B, np.float32)
        logit = np.zeros(B, np.float32)
        m.rec_query_debug(dense, ind, off, B, ctr, logits=logit)   # eager caller-index path
        cv = torch.zeros(B, device="cuda")
        m.rec_synth_query_async(0, segs, cv)                         # the captured-graph path
        m.rec_sync(0)
        out[fuse] = (ctr, logit, cv.cpu().numpy())
        del m
    assert np.array_equal(out["1"][0], out["0"][0])
    assert np.array_equal(out["1"][1], out["0"][1])
    assert np.array_equal(out["1"][2], out["0"][2])
    assert np.array_equal(out["1"][2], out["1"][0])
    exp = fw.forward(cfg, 1, dense, ind, off, return_all=True)
    assert np.abs(out["1"][0].astype(np.float64) - exp["ctr"]).max() <= CTR_TOL


def test_sm_partition_same_bits(monkeypatch):
    """REC_GREEN_SMS=24: dense stages on a 24-SM green context, the SLS on the other SMs
    (captured graphs updated through the driver with the partition's context) — the CTR bits
    equal the shared-SM default on the graph path."""
    cfg = W.small_variant(W.RMC1, 20000)
    segs = W.random_segments(700, seed=41)
    import torch
    out = {}
    for g in ("0", "24"):
        monkeypatch.setenv("REC_GREEN_SMS", g)
        m = _model(cfg, max_batch=1024)
        ctr = torch.zeros(700, dtype=torch.float32, device="cuda")
        for _ in range(3):  # several launches of the same slot graph (node updates)
            m.rec_synth_query_async(0, segs, ctr)
            m.rec_sync(0)
        out[g] = ctr.cpu().numpy()
        del m
    assert np.array_equal(out["0"], out["24"])
    ind, off, dense = gen.gen_batch(cfg, 1, segs)
    exp = fw.forward(cfg, 1, dense, ind, off)
    assert np.abs(out["24"].astype(np.float64) - exp).max() <= CTR_TOL


def test_negative_control_perturbations_fail():
    """SURVEY §8(c) CTR pin / §4 tier 6: the parity checks have teeth on the GPU path.  A
    one-weight perturbation of the oracle's model must break the 2e-2 CTR bar against the
    GPU's CTRs, and one changed index must break the bit-exact pooled check."""
    cfg = W.small_variant(W.RMC1, 20000)
    B = 256
    m = _model(cfg, max_batch=B)
    segs = W.random_segments(B, seed=23)
    ind, off, dense = gen.gen_batch(cfg, 1, segs)
    ctr = np.zeros(B, np.float32)
    pooled = np.zeros((B, cfg.num_tables, cfg.dim), np.float32)
    m.rec_query_debug(dense, ind, off, B, ctr, pooled=pooled)
    exp = fw.forward(cfg, 1, dense, ind, off, return_all=True)
    assert np.abs(ctr - exp["ctr"]).max() <= CTR_TOL                 # the real check passes
    bottom, top = gen.model_params(cfg, 1)
    W0, b0 = top[-1]
    W0 = W0.copy()
    hidden = fw.mlp(exp["v"], top[:-1], relu_last=True)
    W0[0, int(np.argmax(hidden.mean(0)))] += 1.0                      # one weight
    bad = fw.forward(cfg, 1, dense, ind, off, params=(bottom, top[:-1] + [(W0, b0)]))
    assert np.abs(ctr - bad).max() > CTR_TOL
    ind2 = ind.copy()
    ind2[5] = (ind2[5] + 1) % cfg.rows                                # one index
    exp2 = fw.forward(cfg, 1, dense, ind2, off, return_all=True)
    assert not np.array_equal(pooled.astype(np.float64), exp2["pooled"])


def test_async_offsets_validation():
    """rec_query_async: host offsets are checked before enqueueing, including
    offsets[T*B] == nnz; device offsets inconsistent with nnz are flagged at rec_sync and the
    SLS never reads past nnz indices."""
    import torch
    from paper_2203_07424_b200 import RecError
    cfg = W.small_variant(W.TINY, 1000)
    B = 16
    m = _model(cfg, max_batch=B, streams=2)
    ind, off, dense = gen.gen_batch(cfg, 1, W.random_segments(B, seed=3))
    nnz = int(off[-1])
    ctr = np.zeros(B, np.float32)
    with pytest.raises(RecError) as ei:                               # host: nnz mismatch
        m.rec_query_async(0, dense, ind, off, nnz - 1, B, ctr)
    assert ei.value.status == -3
    boff = off.copy()
    boff[3] = boff[2] - 1
    with pytest.raises(RecError) as ei:                               # host: decreasing
        m.rec_query_async(0, dense, ind, boff, nnz, B, ctr)
    assert ei.value.status == -3
    # device offsets whose end exceeds nnz: flagged, and the read is clamped to nnz indices
    dv, iv = torch.from_numpy(dense).cuda(), torch.from_numpy(ind[:nnz - 7].copy()).cuda()
    ov = torch.from_numpy(off).cuda()
    cv = torch.zeros(B, device="cuda")
    m.rec_query_async(1, dv, iv, ov, nnz - 7, B, cv)
    with pytest.raises(RecError) as ei:
        m.rec_sync(1)
    assert ei.value.status == -3
    # a consistent call afterwards works and matches the synchronous path
    m.rec_query_async(1, dv, torch.from_numpy(ind).cuda(), ov, nnz, B, cv)
    m.rec_sync(1)
    ref = np.zeros(B, np.float32)
    m.rec_query(dense, ind, off, B, ref)
    assert np.array_equal(cv.cpu().numpy(), ref)


def test_persistent_chain_large_batch_invariance(monkeypatch):
    """B = 40960 on RMC1 shapes: the fused bottom / top chains run as one wave of persistent
    CTAs walking 320 tiles (the ring streams across tiles); every item's CTR equals the
    small-batch (one CTA per tile) result bit for bit and the oracle within 2e-2, and equals the
    non-persistent launch (REC_CHAIN_PERSISTENT=0)."""
    import torch
    monkeypatch.delenv("REC_CHAIN_PERSISTENT", raising=False)
    cfg = W.small_variant(W.RMC1, 20000)
    B = 40960
    segs = W.random_segments(B, seed=43, max_seg=1000)
    out = {}
    for pers in ("1", "0"):
        monkeypatch.setenv("REC_CHAIN_PERSISTENT", pers)
        m = _model(cfg, max_batch=B)
        cv = torch.zeros(B, device="cuda")
        m.rec_synth_query_async(0, segs, cv)
        m.rec_sync(0)
        out[pers] = cv.cpu().numpy()
        m.close()
    assert np.array_equal(out["1"], out["0"])
    monkeypatch.delenv("REC_CHAIN_PERSISTENT", raising=False)
    q, it = gen.expand_segments(segs)
    pick = np.random.default_rng(4).choice(B, size=40, replace=False)
    sub = np.array([[q[k], it[k], 1] for k in pick], np.int32)
    small = _model(cfg, max_batch=64)
    cs = torch.zeros(40, device="cuda")
    small.rec_synth_query_async(0, sub, cs)
    small.rec_sync(0)
    assert np.array_equal(cs.cpu().numpy(), out["1"][pick])
    i2, o2, d2 = gen.gen_batch(cfg, 1, sub)
    assert np.abs(out["1"][pick] - fw.forward(cfg, 1, d2, i2, o2)).max() <= CTR_TOL
