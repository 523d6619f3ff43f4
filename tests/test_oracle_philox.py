"""Oracle pins: Philox4x32-10 against the Random123 KATs; exact 64-bit mul-high."""
import os

import numpy as np

from oracle import philox as ph

GOLD = os.path.join(os.path.dirname(__file__), "golden", "philox4x32_10_kat.txt")


def _kats():
    for line in open(GOLD):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        v = [int(x, 16) for x in line.split()]
        yield v[0:4], v[4:6], v[6:10]


def test_kat_scalar():
    n = 0
    for ctr, key, out in _kats():
        assert list(ph.philox_scalar(ctr, key)) == out
        n += 1
    assert n == 3


def test_kat_vectorised():
    for ctr, key, out in _kats():
        got = ph.philox(*[np.uint64(c) for c in ctr], np.uint64(key[0]), np.uint64(key[1]))
        assert [int(g) for g in got] == out


def test_vectorised_matches_scalar_random():
    rng = np.random.default_rng(0)
    c = rng.integers(0, 2**32, size=(4, 200), dtype=np.uint64)
    k = rng.integers(0, 2**32, size=(2,), dtype=np.uint64)
    got = ph.philox(c[0], c[1], c[2], c[3], k[0], k[1])
    for i in range(200):
        exp = ph.philox_scalar([int(c[j, i]) for j in range(4)], [int(k[0]), int(k[1])])
        assert tuple(int(g[i]) for g in got) == exp


def test_mulhi64_bruteforce():
    rng = np.random.default_rng(1)
    a = rng.integers(0, 2**63, size=2000, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, size=2000, dtype=np.uint64)
    b = rng.integers(0, 2**63, size=2000, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, size=2000, dtype=np.uint64)
    got = ph.mulhi64(a, b)
    for x, y, g in zip(a, b, got):
        assert int(g) == (int(x) * int(y)) >> 64
    # edge values
    for x, y in [(2**64 - 1, 2**64 - 1), (2**64 - 1, 1), (2**32, 2**32), (0, 5)]:
        assert int(ph.mulhi64(np.uint64(x), np.uint64(y))) == (x * y) >> 64


def test_seed_key():
    assert ph.seed_key(1) == (1, 0)
    assert ph.seed_key((7 << 32) | 9) == (9, 7)
