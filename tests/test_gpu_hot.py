"""Locality-aware hot-row partition on the GPU.

rec_hot_remap profiles the access frequency of a Zipf(0.9) sample (G2z: hot rows scattered
over the table by a fixed bijection, so only the profile can find them), permutes the
embedding arena so the hot rows of all tables form one contiguous prefix, remaps every index
to its arena row and covers the prefix with a persisting L2 window sized capacity /
co-located models.  The result must not change: pooled vectors bit-exact vs the
oracle on the ORIGINAL (un-remapped) model, CTR bits identical to an un-remapped handle on
both the caller-index and the device-synthesised paths."""
import numpy as np
import pytest

import workloads as W
from oracle import forward as fw, gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__
    __graft_entry__.build()


CFG = W.small_variant(W.RMC1, 20000).with_(index_dist=W.INDEX_ZIPF)


def _profile(cfg, n=2048):
    segs = W.random_segments(n, seed=900)
    ind, off, _ = gen.gen_batch(cfg, 1, segs)
    return ind, off, n


@pytest.mark.parametrize("window", [0, 1 << 20, -1], ids=["auto", "1MB", "none"])
def test_hot_remap_same_bits(window):
    import torch
    from paper_2203_07424_b200 import RecModel
    plain = RecModel(CFG, seed=1, max_batch=1024, streams=2)
    hot = RecModel(CFG, seed=1, max_batch=1024, streams=2)
    pind, poff, pn = _profile(CFG)
    rows = hot.rec_hot_remap(pind, poff, pn, window_bytes=window)
    if window < 0:
        assert rows == 0
    else:
        assert rows > 0
    for B in (1, 700):
        segs = W.random_segments(B, seed=40 + B)
        ind, off, dense = gen.gen_batch(CFG, 1, segs)
        c_hot = np.zeros(B, np.float32)
        pooled = np.zeros((B, CFG.num_tables, CFG.dim), np.float32)
        hot.rec_query_debug(dense, ind, off, B, c_hot, pooled=pooled)
        exp = fw.forward(CFG, 1, dense, ind, off, return_all=True)
        assert np.array_equal(pooled.astype(np.float64), exp["pooled"])      # oracle, original ids
        assert np.abs(c_hot - exp["ctr"]).max() <= 2e-2
        c_plain = np.zeros(B, np.float32)
        plain.rec_query(dense, ind, off, B, c_plain)
        assert np.array_equal(c_hot, c_plain)
        g_hot, g_plain = (torch.zeros(B, device="cuda") for _ in range(2))
        hot.rec_synth_query_async(1, segs, g_hot)                           # graph path
        plain.rec_synth_query_async(1, segs, g_plain)
        hot.rec_sync(1)
        plain.rec_sync(1)
        assert torch.equal(g_hot, g_plain)
        assert np.array_equal(g_hot.cpu().numpy(), c_hot)
    # out-of-range caller indices are still reported (the remap kernel checks them)
    from paper_2203_07424_b200 import RecError
    segs = W.random_segments(16, seed=3)
    ind, off, dense = gen.gen_batch(CFG, 1, segs)
    ind[4] = CFG.rows
    with pytest.raises(RecError) as ei:
        hot.rec_query(dense, ind, off, 16, np.zeros(16, np.float32))
    assert ei.value.status == -2
    hot.close()
    plain.close()


def test_hot_remap_profile_orders_rows_by_frequency():
    """A remap built from a profile of the very batch that is then served (every profiled row
    moved) keeps that batch's CTRs within the oracle bar."""
    from paper_2203_07424_b200 import RecModel
    cfg = CFG.with_(rows=3000)
    m = RecModel(cfg, seed=1, max_batch=512)
    pind, poff, pn = _profile(cfg, 512)
    m.rec_hot_remap(pind, poff, pn, window_bytes=-1)
    # CTRs of the profile batch itself unchanged vs the oracle
    ind, off, dense = gen.gen_batch(cfg, 1, W.random_segments(512, seed=900))
    c = np.zeros(512, np.float32)
    m.rec_query(dense, ind, off, 512, c)
    assert np.abs(c - fw.forward(cfg, 1, dense, ind, off)).max() <= 2e-2
    m.close()
