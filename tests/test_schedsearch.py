"""Alg. 1: oracle pins and harness parity (CPU only).

Pins: on unimodal (concave-along-rays) QPS surfaces the gradient search lands on the
brute-force argmax (SPEC.md oracle equivalence); candidate moves are the three
directions; single-point grid; all-infeasible grid -> origin with 0; evaluations stay
well below the grid size on large grids (SPEC.md: <= 15 % of 20 x 8)."""
import itertools

import numpy as np
import pytest

from oracle import serving as sv
from harness import schedsearch as hs


def test_candidate_moves_three_directions():
    assert sorted(sv.candidate_moves(0, 0, 4, 4)) == [(0, 1), (1, 0), (1, 1)]
    assert sv.candidate_moves(3, 0, 4, 4) == [(3, 1)]
    assert sv.candidate_moves(3, 3, 4, 4) == []


def _surfaces(seed):
    rng = np.random.default_rng(seed)
    for _ in range(50):
        nm, nd = rng.integers(1, 9), rng.integers(1, 9)
        pm, pd = rng.integers(0, nm), rng.integers(0, nd)
        am, ad = rng.uniform(0.5, 3), rng.uniform(0.5, 3)
        base = rng.uniform(10, 100)
        ms = list(range(1, nm + 1))
        ds = [16 * 2 ** k for k in range(nd)]

        def f(m, d, pm=pm, pd=pd, am=am, ad=ad, base=base, ms=ms, ds=ds):
            i, j = ms.index(m), ds.index(d)
            # strictly positive, unimodal along every axis (no zero plateau to stall on)
            return base * float(np.exp(-0.1 * (am * (i - pm) ** 2 + ad * (j - pd) ** 2)))
        yield f, ms, ds


def test_oracle_gradient_equals_brute_force_on_unimodal():
    for f, ms, ds in _surfaces(0):
        g = sv.gradient_search(f, ms, ds)
        b = sv.brute_force_search(f, ms, ds)
        assert (g["m"], g["d"], g["qps"]) == (b["m"], b["d"], b["qps"])
        assert g["evals"] <= len(ms) * len(ds)


def test_harness_matches_oracle():
    for f, ms, ds in _surfaces(1):
        h = hs.gradient_search(f, ms, ds)
        o = sv.gradient_search(f, ms, ds)
        assert (h["m"], h["d"], h["qps"], h["path"]) == (o["m"], o["d"], o["qps"], o["path"])


def test_degenerate_grids():
    assert sv.gradient_search(lambda m, d: 5.0, [1], [64])["qps"] == 5.0
    r = hs.gradient_search(lambda m, d: 0.0, [1, 2, 4], [64, 128])
    assert (r["m"], r["d"], r["qps"]) == (1, 64, 0.0)


def test_evaluations_small_fraction_of_large_grid():
    ms, ds = list(range(1, 21)), [16 * 2 ** k for k in range(8)]
    f = lambda m, d: 100 - (m - 6) ** 2 - 4 * (np.log2(d / 16) - 3) ** 2
    r = hs.gradient_search(f, ms, ds)
    assert (r["m"], r["d"]) == (6, 128)
    assert r["evals"] <= 0.15 * len(ms) * len(ds)
