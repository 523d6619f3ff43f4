"""Oracle pins for the MT-WnD forward (Table I row MT-WnD, PAPER.md:191;
DESIGN.md readings R26-R29): one-hot lookups, concatenation, N task towers + wide part.

Pinned by brute-force Python loops on a tiny model (every multiply written out), task
independence (a task's CTR does not move when another task's parameters change), the
one-hot property (the concatenated vector holds the exact table rows) and the shared
parameter scheme (task 0's tower is the DLRM top stack of the same widths)."""
import math

import numpy as np

import workloads as W
from oracle import forward as fw, gen

TINY_WND = W.ModelConfig("wnd-tiny", 3, 50, 4, 1, 1, (), (8, 4, 1), 0, 16, 100.0,
                         arch=W.ARCH_MTWND, tasks=2)


def _brute(cfg, seed, ind, off, B):
    towers, wide = gen.model_params(cfg, seed)[1]
    shift = gen.emb_shift(cfg.pooling_lo, cfg.pooling_hi)
    T, D = cfg.num_tables, cfg.dim
    out = np.zeros((B, cfg.tasks))
    for b in range(B):
        u = []
        for t in range(T):
            acc = [0.0] * D
            for j in range(off[t * B + b], off[t * B + b + 1]):
                row = gen.table_values(seed, t, np.array([ind[j]]), D, shift, cfg.value_mode)[0]
                for d in range(D):
                    acc[d] += float(row[d])
            u.extend(acc)
        for k in range(cfg.tasks):
            h = u
            for li, (Wm, bv) in enumerate(towers[k]):
                nxt = []
                for o in range(Wm.shape[0]):
                    s = float(bv[o])
                    for i in range(Wm.shape[1]):
                        s += float(Wm[o, i]) * h[i]
                    nxt.append(max(s, 0.0) if li < len(towers[k]) - 1 else s)
                h = nxt
            logit = h[0] + sum(float(wide[k][i]) * u[i] for i in range(len(u)))
            out[b, k] = 1.0 / (1.0 + math.exp(-logit))
    return out


def test_mtwnd_bruteforce_tiny():
    segs = W.random_segments(7, seed=2)
    ind, off, dense = gen.gen_batch(TINY_WND, 1, segs)
    assert dense.shape == (7, 0)
    assert np.all(np.diff(off) == 1)                # one-hot: one lookup per (table, item)
    got = fw.forward(TINY_WND, 1, dense, ind, off)
    exp = _brute(TINY_WND, 1, ind, off, 7)
    assert got.shape == (7, 2)
    assert np.allclose(got, exp, rtol=0, atol=1e-12)


def test_mtwnd_one_hot_concat_is_exact_rows():
    cfg = W.small_variant(W.MTWND, 500)
    segs = W.random_segments(5, seed=4)
    ind, off, dense = gen.gen_batch(cfg, 1, segs)
    out = fw.forward(cfg, 1, dense, ind, off, return_all=True)
    shift = gen.emb_shift(1, 1)
    B, T, D = 5, cfg.num_tables, cfg.dim
    for b in range(B):
        for t in range(T):
            row = gen.table_values(1, t, np.array([ind[off[t * B + b]]]), D, shift, cfg.value_mode)[0]
            assert np.array_equal(out["v"][b, t * D:(t + 1) * D], row)


def test_mtwnd_tasks_are_independent():
    cfg = TINY_WND
    segs = W.random_segments(9, seed=6)
    ind, off, dense = gen.gen_batch(cfg, 1, segs)
    bottom, (towers, wide) = gen.model_params(cfg, 1)
    base = fw.forward(cfg, 1, dense, ind, off, params=(bottom, (towers, wide)))
    towers2 = [towers[0], [(W_ * 0.5, b_ - 1.0) for W_, b_ in towers[1]]]
    wide2 = [wide[0], -wide[1]]
    alt = fw.forward(cfg, 1, dense, ind, off, params=(bottom, (towers2, wide2)))
    assert np.array_equal(alt[:, 0], base[:, 0])    # task 0 untouched
    assert not np.allclose(alt[:, 1], base[:, 1])   # task 1 moved


def test_mtwnd_task0_tower_is_the_dlrm_top_stack():
    # the parameter scheme gives task 0 the ids of a DLRM top stack of the same widths
    cfg = TINY_WND
    tower0 = gen.model_params(cfg, 1)[1][0][0]
    dl = W.ModelConfig("x", 3, 50, 4, 1, 1, (2, 4), (8, 4, 1), 0, 16, 1.0)
    top = gen.model_params(dl, 1)[1]
    assert tower0[0][0].shape[1] == cfg.top_in == 12 and top[0][0].shape[1] == dl.top_in == 10
    for (Wa, ba), (Wb, bb) in zip(tower0[1:], top[1:]):   # same fan-in -> identical layers
        assert np.array_equal(Wa, Wb) and np.array_equal(ba, bb)


def test_mtwnd_full_shape_nonvacuous():
    cfg = W.small_variant(W.MTWND, 20000)
    segs = W.random_segments(256, seed=3)
    ind, off, dense = gen.gen_batch(cfg, 1, segs)
    out = fw.forward(cfg, 1, dense, ind, off, return_all=True)
    assert out["ctr"].shape == (256, 2)
    assert np.all(out["logit"].std(axis=0) > 0.5)   # CTR checks at 2e-2 are not vacuous
