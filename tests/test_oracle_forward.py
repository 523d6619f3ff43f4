"""Oracle pins for the forward path (F1-F4).

Each test pins the oracle to something other than itself: brute-force loops on
tiny tables, one-hot lookups returning the exact row,
linearity of pooling, interaction symmetry / ordering / metamorphic table swap,
textbook special cases of the MLP, and the non-vacuity guard of the CTR check.
"""
import itertools
import math

import numpy as np
import pytest

import workloads as W
from oracle import forward as fw, gen


def _tiny_table(T, R, D, seed=0):
    rng = np.random.default_rng(seed)
    return rng.integers(-128, 128, size=(T, R, D)).astype(np.float64) / 128.0


def test_sls_bruteforce_all_small_bags():
    # R = 4 rows, every multiset bag of size 0..3, two tables
    T, R, D = 2, 4, 8
    E = _tiny_table(T, R, D)
    bags = [()] + [c for k in (1, 2, 3) for c in itertools.combinations_with_replacement(range(R), k)]
    B = len(bags)
    idx, off = [], [0]
    for t in range(T):
        for bag in bags:
            idx.extend(bag)
            off.append(len(idx))
    idx, off = np.array(idx), np.array(off)
    out = fw.sls(lambda t, r: E[t][r], T, B, D, idx, off)
    for t in range(T):
        for b, bag in enumerate(bags):
            exp = np.zeros(D)
            for r in bag:                              # plain loop definition
                for k in range(D):
                    exp[k] += E[t][r][k]
            assert np.array_equal(out[b, t], exp)


def test_sls_one_hot_returns_exact_row():
    # pooling 1: "the dummy SLS ... setting the pooling factor to 1"
    cfg = W.TINY.with_(pooling_lo=1, pooling_hi=1, rows=1000)
    segs = W.random_segments(40, seed=1)
    ind, off, _ = gen.gen_batch(cfg, 1, segs)
    rows_fn = lambda t, r: gen.table_values(1, t, r, cfg.dim, 0, 0)
    out = fw.sls(rows_fn, cfg.num_tables, 40, cfg.dim, ind, off)
    for t in range(cfg.num_tables):
        for b in range(40):
            assert np.array_equal(out[b, t], rows_fn(t, np.array([ind[t * 40 + b]]))[0])


def test_sls_linearity_and_bag_concatenation():
    T, R, D = 3, 50, 16
    E = _tiny_table(T, R, D, seed=2)
    rng = np.random.default_rng(3)
    B = 20
    lens = rng.integers(0, 9, size=T * B)
    off = np.concatenate([[0], np.cumsum(lens)])
    idx = rng.integers(0, R, size=off[-1])
    f = lambda t, r: E[t][r]
    base = fw.sls(f, T, B, D, idx, off)
    # SLS(a E) = a SLS(E)
    assert np.allclose(fw.sls(lambda t, r: 0.25 * E[t][r], T, B, D, idx, off), 0.25 * base, rtol=0, atol=0)
    # SLS(bag1 ++ bag2) = SLS(bag1) + SLS(bag2): merge bags of pairs (2b, 2b+1)
    idx2, off2 = [], [0]
    for t in range(T):
        for b in range(0, B, 2):
            g = t * B + b
            idx2.extend(idx[off[g]:off[g + 2]])
            off2.append(len(idx2))
    merged = fw.sls(f, T, B // 2, D, np.array(idx2), np.array(off2))
    assert np.allclose(merged, base[0::2] + base[1::2], rtol=0, atol=1e-12)


def test_sls_empty_and_duplicates():
    E = _tiny_table(1, 5, 4, seed=4)
    out = fw.sls(lambda t, r: E[t][r], 1, 3, 4, np.array([2, 2, 2, 1]), np.array([0, 0, 3, 4]))
    assert np.array_equal(out[0, 0], np.zeros(4))
    assert np.array_equal(out[1, 0], 3 * E[0][2])
    assert np.array_equal(out[2, 0], E[0][1])


def test_sls_fp32_sequential_equals_exact_in_int8_mode():
    # int8 * 2^-e sums of < 2^24/127 terms are exact in fp32 in ANY order (G4)
    cfg = W.small_variant(W.RMC1, 3000)
    segs = W.random_segments(64, seed=6)
    ind, off, _ = gen.gen_batch(cfg, 1, segs)
    f = lambda t, r: gen.table_values(1, t, r, cfg.dim, 2, 0)
    a = fw.sls(f, cfg.num_tables, 64, cfg.dim, ind, off)
    b = fw.sls(f, cfg.num_tables, 64, cfg.dim, ind, off, fp32_sequential=True)
    assert np.array_equal(a, b.astype(np.float64))


def test_mlp_identity_and_zero_special_cases():
    rng = np.random.default_rng(5)
    x = rng.standard_normal((7, 6))
    I = [(np.eye(6), np.zeros(6))]
    assert np.array_equal(fw.mlp(x, I, relu_last=True), np.maximum(x, 0))
    assert np.array_equal(fw.mlp(x, I, relu_last=False), x)
    # zero weights => ctr = sigmoid(b_last)
    layers = [(np.zeros((4, 6)), rng.standard_normal(4)), (np.zeros((1, 4)), np.array([0.7]))]
    out = fw.mlp(x, layers, relu_last=False)
    assert np.allclose(out, 0.7) and np.allclose(fw.sigmoid(out), 1 / (1 + np.exp(-0.7)))


def test_mlp_against_loops():
    rng = np.random.default_rng(8)
    x = rng.standard_normal((3, 5))
    W1, b1 = rng.standard_normal((4, 5)), rng.standard_normal(4)
    W2, b2 = rng.standard_normal((2, 4)), rng.standard_normal(2)
    out = fw.mlp(x, [(W1, b1), (W2, b2)], relu_last=False)
    for n in range(3):
        h = [max(0.0, sum(W1[o][i] * x[n][i] for i in range(5)) + b1[o]) for o in range(4)]
        y = [sum(W2[o][i] * h[i] for i in range(4)) + b2[o] for o in range(2)]
        assert np.allclose(out[n], y, rtol=1e-12, atol=1e-12)


def test_interaction_order_and_symmetry():
    B, T, D = 2, 3, 4
    rng = np.random.default_rng(9)
    x = rng.standard_normal((B, D))
    p = rng.standard_normal((B, T, D))
    v = fw.interaction(x, p)
    assert v.shape == (B, D + T * (T + 1) // 2)
    X = np.concatenate([x[:, None], p], axis=1)
    for b in range(B):
        exp = list(x[b])
        for i in range(1, T + 1):            # row-major strict lower triangle
            for j in range(i):
                exp.append(sum(X[b, i, k] * X[b, j, k] for k in range(D)))
        assert np.allclose(v[b], exp, rtol=1e-13, atol=1e-13)
        Z = X[b] @ X[b].T
        assert np.allclose(Z, Z.T) and np.all(np.diag(Z) >= 0)


def test_interaction_one_hot_basis():
    D, T = 8, 4
    x = np.eye(D)[0][None]
    p = np.eye(D)[1:T + 1][None]                     # X = first T+1 basis vectors
    v = fw.interaction(x, p)
    assert np.array_equal(v[0, D:], np.zeros(T * (T + 1) // 2))
    p2 = np.repeat(np.eye(D)[0][None, None], T, axis=1)  # all rows equal e0
    v2 = fw.interaction(x, p2)
    assert np.array_equal(v2[0, D:], np.ones(T * (T + 1) // 2))


def test_interaction_table_swap_metamorphic():
    B, T, D = 3, 4, 5
    rng = np.random.default_rng(10)
    x, p = rng.standard_normal((B, D)), rng.standard_normal((B, T, D))
    perm = [2, 0, 3, 1]                               # table t' = perm[t]
    v = fw.interaction(x, p)
    vp = fw.interaction(x, p[:, perm])
    pos = {}
    k = 0
    for i in range(1, T + 1):
        for j in range(i):
            pos[(i, j)] = k
            k += 1
    slot = [0] + [1 + q for q in perm]                # X row of permuted position
    for i in range(1, T + 1):
        for j in range(i):
            a, b = max(slot[i], slot[j]), min(slot[i], slot[j])
            assert np.isclose(vp[:, D + pos[(i, j)]], v[:, D + pos[(a, b)]]).all()


@pytest.mark.parametrize("name", ["tiny", "rmc1", "rmc2", "rmc3"])
def test_ctr_non_vacuity_guard(name):
    # logit spread in [0.5, 4] and < 5% of CTRs outside [0.02, 0.98] (SURVEY §8(c) CTR pin)
    cfg = W.small_variant(W.SHORT[name], 20000 if name != "rmc2" else 4096)
    B = 256 if name != "rmc2" else 96
    segs = W.random_segments(B, seed=12)
    ind, off, dense = gen.gen_batch(cfg, 1, segs)
    out = fw.forward(cfg, 1, dense, ind, off, return_all=True)
    s = out["logit"].std()
    assert 0.5 <= s <= 4.0, s
    c = out["ctr"]
    assert np.mean((c < 0.02) | (c > 0.98)) < 0.05
    # a one-weight perturbation must move CTRs by more than the 2e-2 parity tolerance
    bottom, top = gen.model_params(cfg, 1)
    W0, b0 = top[-1]
    W0 = W0.copy()
    hidden = fw.mlp(out["v"], top[:-1], relu_last=True)          # input of the last layer
    j = int(np.argmax(hidden.mean(0)))                            # most active unit
    W0[0, j] += 1.0
    c2 = fw.forward(cfg, 1, dense, ind, off, params=(bottom, top[:-1] + [(W0, b0)]))
    assert np.max(np.abs(c2 - c)) > 2e-2


def _dlrm_brute(cfg, seed, dense, ind, off, B):
    """The DLRM query forward written out as explicit loops (DESIGN.md
    R1, R2, R8, R24): every sum, product, ReLU and the interaction's pair order by hand.
    Parameters come from the seeded parameter scheme (G4/G5, pinned in test_oracle_gen.py);
    the embedding scale s = round(log2(0.577 sqrt(mean L))) is restated here (G4)."""
    T, D = cfg.num_tables, cfg.dim
    bottom, top = gen.model_params(cfg, seed)
    s = int(round(math.log2(0.577 * math.sqrt(0.5 * (cfg.pooling_lo + cfg.pooling_hi)))))
    out = []
    for b in range(B):
        # F1 SLS: p_t = sum of the bag's rows, in index order (R8 sum)
        p = []
        for t in range(T):
            acc = [0.0] * D
            for j in range(int(off[t * B + b]), int(off[t * B + b + 1])):
                row = gen.table_values(seed, t, np.array([ind[j]]), D, s, cfg.value_mode)[0]
                for k in range(D):
                    acc[k] += float(row[k])
            p.append(acc)
        # F2 bottom: ReLU after EVERY layer, including the last (R2)
        h = [float(v) for v in dense[b]]
        for Wm, bv in bottom:
            h = [max(0.0, float(bv[o]) + sum(float(Wm[o, i]) * h[i] for i in range(len(h))))
                 for o in range(Wm.shape[0])]
        x = h
        # F3 interaction: X = [x; p_0; ...; p_{T-1}]; pairs (i, j), i = 1..T, j < i (R1)
        X = [x] + p
        v = list(x)
        for i in range(1, T + 1):
            for j in range(i):
                v.append(sum(X[i][k] * X[j][k] for k in range(D)))
        # F4 top: ReLU on hidden layers, the width-1 last layer linear, then sigmoid (R2)
        h = v
        for li, (Wm, bv) in enumerate(top):
            z = [float(bv[o]) + sum(float(Wm[o, i]) * h[i] for i in range(len(h)))
                 for o in range(Wm.shape[0])]
            h = z if li == len(top) - 1 else [max(0.0, q) for q in z]
        out.append(1.0 / (1.0 + math.exp(-h[0])))
    return np.array(out)


@pytest.mark.parametrize("lo,hi,vm", [(3, 3, 0), (0, 4, 0), (2, 5, 1)])
def test_forward_dlrm_bruteforce_tiny(lo, hi, vm):
    """oracle.forward.forward (the composition of F1-F4) equals the loop definition on a
    T = 3, D = 4 DLRM: catches a bottom without the last ReLU, [pooled; x] order, a transposed
    pair index, a wrong embedding scale, or the sigmoid on the wrong value."""
    cfg = W.ModelConfig("dlrm-brute", 3, 40, 4, lo, hi, (5, 6, 4), (7, 3, 1), 0, 8, 1.0,
                        value_mode=vm)
    B = 9
    segs = W.random_segments(B, seed=17, max_seg=4)
    ind, off, dense = gen.gen_batch(cfg, 1, segs)
    if lo == 0:
        assert np.any(np.diff(off) == 0)              # the case has empty bags
    got = fw.forward(cfg, 1, dense, ind, off)
    exp = _dlrm_brute(cfg, 1, dense, ind, off, B)
    assert np.allclose(got, exp, rtol=0, atol=1e-12)
    assert exp.std() > 1e-3                            # not a constant (non-vacuous)


def test_forward_dlrm_bruteforce_detects_plausible_slips():
    """Negative control of the pin above: each plausible slip in the composition moves the
    CTRs far beyond 1e-12 on the same inputs."""
    cfg = W.ModelConfig("dlrm-brute", 3, 40, 4, 3, 3, (5, 6, 4), (7, 3, 1), 0, 8, 1.0)
    B = 9
    ind, off, dense = gen.gen_batch(cfg, 1, W.random_segments(B, seed=17, max_seg=4))
    exp = _dlrm_brute(cfg, 1, dense, ind, off, B)
    bottom, top = gen.model_params(cfg, 1)
    shift = gen.emb_shift(3, 3)
    rows_fn = lambda t, r, s=shift: gen.table_values(1, t, r, 4, s, 0)
    pooled = fw.sls(rows_fn, 3, B, 4, ind, off)
    x = fw.mlp(dense.astype(np.float64), bottom, relu_last=True)
    slips = {
        "no last bottom ReLU": (fw.mlp(dense.astype(np.float64), bottom, relu_last=False), pooled),
        "wrong emb shift": (x, fw.sls(lambda t, r: gen.table_values(1, t, r, 4, shift + 1, 0),
                                      3, B, 4, ind, off)),
    }
    for name, (xx, pp) in slips.items():
        c = fw.sigmoid(fw.mlp(fw.interaction(xx, pp), top, relu_last=False)[:, 0])
        assert np.max(np.abs(c - exp)) > 1e-6, name
    # [pooled; x] order instead of [x; pooled]
    Xs = np.concatenate([pooled, x[:, None]], axis=1)
    ii, jj = np.tril_indices(4, k=-1)
    Z = np.einsum("bid,bjd->bij", Xs, Xs)
    c = fw.sigmoid(fw.mlp(np.concatenate([x, Z[:, ii, jj]], 1), top, relu_last=False)[:, 0])
    assert np.max(np.abs(c - exp)) > 1e-6
