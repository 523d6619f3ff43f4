"""Philox4x32-10 (Salmon et al., SC'11 "Parallel random numbers: as easy as 1, 2, 3").

TEST INFRASTRUCTURE (see oracle/__init__.py).

DESIGN.md G1.  The paper fixes no generator; every random quantity of the synthetic
workload is a pure function of a counter through Philox so that the oracle and
the CUDA kernels can derive identical bits independently.

Round (Random123 philox4x32round):
    (c0,c1,c2,c3) <- (hi(M1*c2) ^ c1 ^ k0, lo(M1*c2), hi(M0*c0) ^ c3 ^ k1, lo(M0*c0))
and the key is bumped by (W0, W1) before every round after the first; 10 rounds.
Pinned by the Random123 known-answer tests in tests/test_oracle_philox.py.
"""
from __future__ import annotations

import numpy as np

M0 = 0xD2511F53
M1 = 0xCD9E8D57
W0 = 0x9E3779B9
W1 = 0xBB67AE85
MASK32 = 0xFFFFFFFF


def philox_scalar(ctr, key):
    """Pure-Python-int Philox4x32-10 on one counter (4 x u32) and key (2 x u32)."""
    c0, c1, c2, c3 = (int(x) & MASK32 for x in ctr)
    k0, k1 = (int(x) & MASK32 for x in key)
    for r in range(10):
        if r:
            k0 = (k0 + W0) & MASK32
            k1 = (k1 + W1) & MASK32
        p0 = M0 * c0
        p1 = M1 * c2
        c0, c1, c2, c3 = ((p1 >> 32) ^ c1 ^ k0, p1 & MASK32, (p0 >> 32) ^ c3 ^ k1, p0 & MASK32)
    return c0, c1, c2, c3


def philox(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32-10.  Inputs broadcast; returns four uint64 arrays of u32."""
    u = np.uint64
    m = u(MASK32)
    c0, c1, c2, c3 = (np.asarray(x, dtype=np.uint64) & m for x in (c0, c1, c2, c3))
    k0 = np.asarray(k0, dtype=np.uint64) & m
    k1 = np.asarray(k1, dtype=np.uint64) & m
    c0, c1, c2, c3 = np.broadcast_arrays(c0, c1, c2, c3)
    for r in range(10):
        if r:
            k0 = (k0 + u(W0)) & m
            k1 = (k1 + u(W1)) & m
        p0 = u(M0) * c0          # < 2^64: exact in uint64
        p1 = u(M1) * c2
        c0, c1, c2, c3 = ((p1 >> u(32)) ^ c1 ^ k0, p1 & m, (p0 >> u(32)) ^ c3 ^ k1, p0 & m)
    return c0, c1, c2, c3


def seed_key(seed: int):
    """Key = (seed mod 2^32, seed >> 32)  (G1)."""
    seed = int(seed) & ((1 << 64) - 1)
    return seed & MASK32, seed >> 32


def mulhi64(a, b):
    """floor(a*b / 2^64) for uint64 arrays, exactly, via 32-bit limbs."""
    u = np.uint64
    m = u(MASK32)
    a = np.asarray(a, dtype=np.uint64)
    b = np.asarray(b, dtype=np.uint64)
    a_lo, a_hi = a & m, a >> u(32)
    b_lo, b_hi = b & m, b >> u(32)
    ll = a_lo * b_lo
    lh = a_lo * b_hi
    hl = a_hi * b_lo
    hh = a_hi * b_hi
    # carry of the middle column: (ll>>32) + lo(lh) + lo(hl) < 3*2^32
    mid = (ll >> u(32)) + (lh & m) + (hl & m)
    return hh + (lh >> u(32)) + (hl >> u(32)) + (mid >> u(32))
