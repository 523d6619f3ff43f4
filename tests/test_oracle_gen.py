"""Oracle pins for the synthetic generators (G2-G5)."""
import numpy as np
import pytest

import workloads as W
from oracle import gen, philox as ph


def _bf16_exact(x):
    x32 = np.asarray(x, dtype=np.float32)
    bits = x32.view(np.uint32)
    return np.all((bits & np.uint32(0xFFFF)) == 0)


def test_index_power_of_two_rows_is_top_bits():
    # closed form: with R = 2^k rows, floor(r*R/2^64) = r >> (64-k)
    cfg = W.TINY.with_(rows=1 << 12)
    segs = W.random_segments(50, seed=3)
    q, it = gen.expand_segments(segs)
    lens = gen.bag_lengths(11, cfg, q, it)
    for t in (0, 5):
        idx = gen.bag_indices(11, cfg, t, q, it, lens[t], 1 << 12)
        # rebuild r for each slot from the scalar (KAT-pinned) generator
        k0, k1 = ph.seed_key(11)
        pos = 0
        for b in range(q.size):
            for j in range(int(lens[t, b])):
                w = ph.philox_scalar([j, int(it[b]), (t << 8) | 1, int(q[b])], [k0, k1])
                r = (w[1] << 32) | w[0]
                assert idx[pos] == r >> (64 - 12)
                pos += 1


def test_index_range_and_rough_uniformity():
    cfg = W.RMC1.with_(rows=1000)
    segs = W.random_segments(400, seed=5)
    ind, off, _ = gen.gen_batch(cfg, 1, segs)
    assert ind.min() >= 0 and ind.max() < 1000
    h = np.bincount(ind, minlength=1000)
    # 320000 draws into 1000 bins: mean 320, Poisson sd ~17.9
    assert abs(h.mean() - 320) < 1e-9 and 14.0 < h.std() < 22.0


def test_offsets_closed_form_fixed_pooling():
    cfg = W.RMC1.with_(rows=5000)
    segs = W.random_segments(77, seed=9)
    ind, off, dense = gen.gen_batch(cfg, 1, segs)
    T, L, B = cfg.num_tables, cfg.pooling_lo, 77
    assert np.array_equal(off, np.arange(T * B + 1) * L)
    assert ind.size == T * B * L
    assert dense.shape == (B, cfg.dense_dim)


def test_variable_pooling_bounds_and_degenerate():
    cfg = W.RMC1.with_(rows=5000, pooling_lo=20, pooling_hi=160)
    segs = W.random_segments(300, seed=2)
    q, it = gen.expand_segments(segs)
    lens = gen.bag_lengths(1, cfg, q, it)
    assert lens.min() >= 20 and lens.max() <= 160
    assert lens.min() < 40 and lens.max() > 140          # spans the range
    # lo == hi reduces to the fixed case
    cfg2 = cfg.with_(pooling_lo=33, pooling_hi=33)
    assert np.all(gen.bag_lengths(1, cfg2, q, it) == 33)


def test_batch_invariance_of_inputs():
    # an item's indices / dense row depend on (qid, item) only, not on its batch
    cfg = W.TINY
    a = np.array([[7, 0, 5], [3, 10, 4]])
    b = np.array([[3, 12, 2], [9, 1, 1], [7, 2, 3]])
    ia, oa, da = gen.gen_batch(cfg, 1, a)
    ib, ob, db = gen.gen_batch(cfg, 1, b)
    # item (3, 12) is row 7 of batch a (5 + 2) and row 0 of batch b
    assert np.array_equal(da[7], db[0])
    T, L = cfg.num_tables, cfg.pooling_lo
    for t in range(T):
        ga, gb = t * 9 + 7, t * 6 + 0
        assert np.array_equal(ia[oa[ga]:oa[ga + 1]], ib[ob[gb]:ob[gb + 1]])


def test_values_exact_in_bf16_and_ranges():
    for mode in (0,):
        v = gen.table_values(1, 3, np.arange(100), 32, 2, mode)
        assert _bf16_exact(v) and np.abs(v).max() <= 2.0 ** -2
        assert np.all(v * 2 ** 9 == np.round(v * 2 ** 9))
    v = gen.table_values(1, 3, np.arange(100), 64, 1, 1)        # fp32 mode: 24-bit fixed point
    assert np.all(v.astype(np.float32).astype(np.float64) == v)
    assert v.min() >= -0.5 and v.max() < 0.5
    W_, b_ = gen.layer_params(1, 0, 256, 128)
    assert _bf16_exact(W_) and _bf16_exact(b_)
    d = gen.dense_features(1, 13, np.array([1, 2]), np.array([0, 1]))
    assert _bf16_exact(d) and d.min() >= -1 and d.max() < 1


def test_weight_scale_variance():
    # a_l = 2^round(log2 sqrt(3/fan_in)) -> Var(W) within a factor sqrt(2) of 1/fan_in
    for fan_in in (16, 87, 256, 884, 2560):
        W_, _ = gen.layer_params(7, 1, fan_in, 256)
        r = W_.var() * fan_in
        assert 0.5 < r < 2.1, (fan_in, r)


def test_domains_disjoint():
    W0, _ = gen.layer_params(1, 0, 64, 64)
    W64, _ = gen.layer_params(1, 64, 64, 64)
    assert not np.array_equal(W0, W64)
    e0 = gen.table_values(1, 0, np.arange(8), 32, 0, 0)
    e1 = gen.table_values(1, 1, np.arange(8), 32, 0, 0)
    assert not np.array_equal(e0, e1)


def test_skewed_indices_are_skewed():
    cfg = W.RMC1.with_(rows=1000, index_dist=W.INDEX_SKEW2)
    ind, _, _ = gen.gen_batch(cfg, 1, W.random_segments(300, seed=4))
    h = np.sort(np.bincount(ind, minlength=1000))[::-1]
    top10 = h[:100].sum() / h.sum()
    # product of two uniforms: P(u < 0.1) = 0.1 (1 + ln 10) = 0.330
    assert 0.30 < top10 < 0.36
    assert (ind < 100).mean() > 0.30


def test_emb_shift_values():
    assert gen.emb_shift(80, 80) == 2 and gen.emb_shift(20, 20) == 1 and gen.emb_shift(120, 120) == 3


# ----------------------------------------------------------------- Zipf(0.9) rows (G2z)
def test_zipf_pow10_and_bisection_constant():
    # pow10 is x^10 up to the rounding of four multiplications; c is the largest double with
    # pow10(c) <= R (the next double up exceeds R), so every rank is < R
    for R in (7, 1000, 20000, 1_000_000, (1 << 31) - 1):
        c = gen.zipf_c(R)
        assert gen.pow10(c) <= R < gen.pow10(np.nextafter(c, np.inf))
        assert abs(c - R ** 0.1) <= 1e-12 * R ** 0.1
    x = np.linspace(1.0, 8.0, 1001)
    assert np.allclose(gen.pow10(x), x ** 10, rtol=1e-15, atol=0)


def test_zipf_rank_cdf_closed_form():
    # P(rank <= k - 1) = P(x^10 < k + 1) = ((k + 1)^0.1 - 1) / (c - 1): a Zipf law with
    # exponent 0.9 (density of y = x^10 is proportional to y^-0.9); 2e5 draws, 5-sigma bounds
    R = 1_000_000
    rng = np.random.default_rng(4)
    r = rng.integers(0, 1 << 63, size=200_000, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, size=200_000, dtype=np.uint64)
    rank = gen.zipf_rank(r, R)
    assert rank.min() >= 0 and rank.max() <= R - 1
    c = gen.zipf_c(R)
    for k in (1, 10, 100, 10_000, 100_000, 999_999):
        p = min(1.0, ((k + 1) ** 0.1 - 1.0) / (c - 1.0))
        emp = np.mean(rank <= k - 1)
        assert abs(emp - p) <= 5 * np.sqrt(p * (1 - p) / r.size) + 1e-12, (k, emp, p)
    # the hottest 10 % of rows take ~72 % of the accesses (closed form 0.7247)
    assert abs(np.mean(rank < R // 10) - ((R // 10) ** 0.1 - 1) / (c - 1)) < 0.01


def test_zipf_rows_bijection_and_generator_counters():
    R = 1000
    ranks = np.arange(R, dtype=np.uint64)
    for t in (0, 3):
        rows = ((ranks * np.uint64(gen.ZIPF_MULT) + np.uint64(gen.ZIPF_T_OFF * t)) % np.uint64(R))
        assert np.unique(rows).size == R                      # a permutation of the rows
    # bag_indices with index_dist 3 follows G2's counters, then the G2z map (scalar rebuild)
    cfg = W.TINY.with_(rows=5000, index_dist=W.INDEX_ZIPF)
    segs = W.random_segments(20, seed=8)
    q, it = gen.expand_segments(segs)
    lens = gen.bag_lengths(11, cfg, q, it)
    k0, k1 = ph.seed_key(11)
    c = gen.zipf_c(5000)
    for t in (0, 6):
        idx = gen.bag_indices(11, cfg, t, q, it, lens[t], 5000)
        pos = 0
        for b in range(q.size):
            for j in range(int(lens[t, b])):
                w = ph.philox_scalar([j, int(it[b]), (t << 8) | 1, int(q[b])], [k0, k1])
                r = (w[1] << 32) | w[0]
                u = float(r >> 11) * 2.0 ** -53
                rank = min(int(np.floor((1.0 + u * (c - 1.0)) ** 10)) - 1, 4999)  # pow: +-1 ulp
                rk = int(gen.zipf_rank(np.array([r], np.uint64), 5000)[0])
                assert abs(rk - rank) <= 1
                assert idx[pos] == (rk * gen.ZIPF_MULT + gen.ZIPF_T_OFF * t) % 5000
                pos += 1


def test_dense_features_byte_layout_scalar_rebuild():
    """G4 dense features: feature f of (q, item) = int8 of byte f mod 16 of the little-endian
    16-byte Philox output of counter (f // 16, item, 3, q), times 2^-7 (scalar rebuild from the
    KAT-pinned scalar generator, bytes extracted by hand)."""
    q, it, F = np.array([5, 900]), np.array([3, 77]), 45
    d = gen.dense_features(9, F, q, it)
    k0, k1 = ph.seed_key(9)
    for b in range(2):
        for f in range(F):
            w = ph.philox_scalar([f // 16, int(it[b]), 3, int(q[b])], [k0, k1])
            raw = b"".join(int(x).to_bytes(4, "little") for x in w)[f % 16]
            val = raw - 256 if raw >= 128 else raw
            assert d[b, f] == val * 2.0 ** -7
