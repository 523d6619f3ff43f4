"""Synthetic model parameters and query inputs as pure functions of counters.

TEST INFRASTRUCTURE (see oracle/__init__.py).

The paper publishes no data, no weights and no traces (PAPER.md:782 only says the
load generator follows "the query arrival characteristics observed in
production").  DESIGN.md G2-G5 define every synthetic value as Philox4x32-10 of a
counter (ctr0, ctr1, ctr2 = (table<<8)|domain, ctr3) under key = seed:

  domain 1  index   E-table row of (query q, item i, table t, slot j): ctr (j, i, t<<8|1, q)
  domain 2  length  pooling factor of (q, i, t) when pooling varies:  ctr (0, i, t<<8|2, q)
  domain 3  dense   dense features 16f'..16f'+15 of (q, i):             ctr (f', i, 3, q)
                    (feature f = byte f mod 16 of the 16-byte output, round 2)
  domain 4  table   E_t[r][k]:                                         ctr (k, r, t<<8|4, 0)
  domain 5  weight  layer l, W[o][i]:                                  ctr (i, o, l<<8|5, 0)
  domain 6  bias    layer l, b[o]:                                     ctr (o, 0, l<<8|6, 0)

Bottom layers are numbered l = 0, 1, ...; top layers l = 64, 65, ... (disjoint domains).
All values are int8 * 2^e (or 24-bit fixed point in fp32 mode): exactly representable
in fp32 AND bf16, so oracle and GPU start from identical parameters.
"""
from __future__ import annotations

import math
from typing import Sequence

import numpy as np

from .philox import philox, seed_key, mulhi64

TOP_LAYER_BASE = 64


def _int8_low_byte(w0: np.ndarray) -> np.ndarray:
    b = (w0 & np.uint64(0xFF)).astype(np.int64)
    return np.where(b >= 128, b - 256, b)


def _u64(w_lo: np.ndarray, w_hi: np.ndarray) -> np.ndarray:
    return (w_hi << np.uint64(32)) | w_lo


def emb_shift(pooling_lo: int, pooling_hi: int) -> int:
    """s = round(log2(0.577 * sqrt(L))) with L the mean pooling (G4)."""
    L = 0.5 * (pooling_lo + pooling_hi)
    return int(round(math.log2(0.577 * math.sqrt(L))))


def weight_exp(fan_in: int) -> int:
    """a_l = 2^round(log2 sqrt(3 / fan_in)) (G5): Var(W) ~ 1/fan_in."""
    return int(round(math.log2(math.sqrt(3.0 / fan_in))))


# ------------------------------------------------------------------ parameters (G4, G5)
def table_values(seed: int, t: int, rows_idx, dim: int, shift: int, value_mode: int) -> np.ndarray:
    """E_t[rows_idx][0:dim] in float64 (exact values), shape [len(rows_idx), dim]."""
    k0, k1 = seed_key(seed)
    r = np.asarray(rows_idx, dtype=np.uint64).reshape(-1, 1)
    k = np.arange(dim, dtype=np.uint64).reshape(1, -1)
    w0, _, _, _ = philox(k, r, np.uint64((t << 8) | 4), np.uint64(0), k0, k1)
    if value_mode == 0:                     # REC_VALUES_INT8_EXACT
        return _int8_low_byte(w0).astype(np.float64) * 2.0 ** -(7 + shift)
    v = (w0 >> np.uint64(8)).astype(np.int64) - (1 << 23)   # REC_VALUES_FP32
    return v.astype(np.float64) * 2.0 ** -(23 + shift)


def layer_params(seed: int, layer: int, fan_in: int, fan_out: int, extra_shift: int = 0):
    """(W [fan_out][fan_in], b [fan_out]) in float64, exact int8 * 2^e values."""
    k0, k1 = seed_key(seed)
    e = -7 + weight_exp(fan_in) - extra_shift
    i = np.arange(fan_in, dtype=np.uint64).reshape(1, -1)
    o = np.arange(fan_out, dtype=np.uint64).reshape(-1, 1)
    w0, _, _, _ = philox(i, o, np.uint64((layer << 8) | 5), np.uint64(0), k0, k1)
    W = _int8_low_byte(w0).astype(np.float64) * 2.0 ** e
    ob = np.arange(fan_out, dtype=np.uint64)
    b0, _, _, _ = philox(ob, np.uint64(0), np.uint64((layer << 8) | 6), np.uint64(0), k0, k1)
    b = _int8_low_byte(b0).astype(np.float64) * 2.0 ** e
    return W, b


TASK_LAYER_STRIDE = 16   # MT-WnD: tower k's layer l has id TOP_LAYER_BASE + 16 k + l (R29)
WIDE_LAYER = 15          # ... and its wide vector id TOP_LAYER_BASE + 16 k + 15


def model_params(cfg, seed: int):
    """All MLP parameters of a config.

    DLRM: (bottom [(W,b)...], top [(W,b)...]).
    MT-WnD (R26-R29): (bottom = [], (towers [[(W,b)...] per task], wide [v_k [T*D]])) — tower k
    uses layer ids TOP_LAYER_BASE + 16 k + l, its wide vector the id TOP_LAYER_BASE + 16 k + 15
    (the W row of a fan_out = 1 layer; no bias); task 0's tower equals a DLRM top stack over
    the same input width."""
    bottom = []
    for l in range(len(cfg.bottom) - 1):
        bottom.append(layer_params(seed, l, cfg.bottom[l], cfg.bottom[l + 1]))
    widths = [cfg.top_in] + list(cfg.top)
    towers = []
    for k in range(cfg.tasks):
        tw = []
        for l in range(len(cfg.top)):
            tw.append(layer_params(seed, TOP_LAYER_BASE + TASK_LAYER_STRIDE * k + l, widths[l],
                                   widths[l + 1], cfg.top_shift if l == 0 else 0))
        towers.append(tw)
    if getattr(cfg, "arch", 0) == 0:
        return bottom, towers[0]
    wide = [layer_params(seed, TOP_LAYER_BASE + TASK_LAYER_STRIDE * k + WIDE_LAYER, cfg.top_in, 1,
                         cfg.top_shift)[0][0] for k in range(cfg.tasks)]
    return bottom, (towers, wide)


# ------------------------------------------------------------------ query inputs (G2, G3)
def expand_segments(segs) -> tuple:
    """Batch rows b -> (qid, item) from a segment list [(qid, start, len)...] in order."""
    segs = np.asarray(segs, dtype=np.int64).reshape(-1, 3)
    q = np.concatenate([np.full(s[2], s[0], dtype=np.int64) for s in segs]) if len(segs) else np.zeros(0, np.int64)
    it = np.concatenate([np.arange(s[1], s[1] + s[2], dtype=np.int64) for s in segs]) if len(segs) else np.zeros(0, np.int64)
    return q, it


def bag_lengths(seed: int, cfg, q: np.ndarray, it: np.ndarray) -> np.ndarray:
    """lengths [T][B] (G3)."""
    T = cfg.num_tables
    B = q.size
    if cfg.pooling_lo == cfg.pooling_hi:
        return np.full((T, B), cfg.pooling_lo, dtype=np.int64)
    k0, k1 = seed_key(seed)
    span = np.uint64(cfg.pooling_hi - cfg.pooling_lo + 1)
    out = np.empty((T, B), dtype=np.int64)
    for t in range(T):
        w0, w1, _, _ = philox(np.uint64(0), it.astype(np.uint64), np.uint64((t << 8) | 2),
                              q.astype(np.uint64), k0, k1)
        out[t] = cfg.pooling_lo + mulhi64(_u64(w0, w1), span).astype(np.int64)
    return out


def bag_indices(seed: int, cfg, t: int, q: np.ndarray, it: np.ndarray, lengths_t: np.ndarray,
                rows_t: int) -> np.ndarray:
    """Concatenated indices of the bags (t, b) for b = 0..B-1, slot order (G2)."""
    k0, k1 = seed_key(seed)
    nnz = int(lengths_t.sum())
    bq = np.repeat(q, lengths_t).astype(np.uint64)
    bi = np.repeat(it, lengths_t).astype(np.uint64)
    starts = np.repeat(np.cumsum(lengths_t) - lengths_t, lengths_t)
    j = (np.arange(nnz, dtype=np.int64) - starts).astype(np.uint64)
    w0, w1, w2, w3 = philox(j, bi, np.uint64((t << 8) | 1), bq, k0, k1)
    r = _u64(w0, w1)
    if cfg.index_dist == 3:                  # Zipf(0.9), scattered (G2z)
        return zipf_rows(r, rows_t, t)
    if cfg.index_dist == 2:                  # skewed: product of two uniforms (G2)
        r = mulhi64(r, _u64(w2, w3))
    return mulhi64(r, np.uint64(rows_t)).astype(np.int64)


# ------------------------------------------------------------------ Zipf(0.9) indices (G2z)
# SPEC.md:279 draws embedding rows from a Zipf law with exponent 0.9 ("hot" rows, the locality
# the hot-embedding partition exploits).  G2z is the continuous inverse-CDF
# form of that law, written so that every step is an exactly rounded IEEE fp64 operation (no
# pow, no fused multiply-add), hence bit-identical wherever it is evaluated:
#   c     = the largest double in [1, 16] with pow10(c) <= R, by 60 bisection steps
#   u     = (r >> 11) * 2^-53                      (53-bit uniform in [0, 1))
#   x     = 1 + u * (c - 1)                        (x uniform in [1, c))
#   y     = pow10(x) = ((x^2)^2)^2 * x^2           (y = x^10 has density prop. to y^-0.9)
#   rank  = min(floor(y) - 1, R - 1)               (0 = hottest)
#   row   = (rank * 2654435761 + 7919 t) mod R    (a bijection: 2654435761 is prime > R, so
#                                                  hot rows are scattered over the table and
#                                                  only a frequency profile finds them)
ZIPF_MULT = 2654435761
ZIPF_T_OFF = 7919


def pow10(x):
    """x^10 as four exactly rounded multiplications (x2 = x*x, x4, x8, x8*x2)."""
    x2 = x * x
    x4 = x2 * x2
    x8 = x4 * x4
    return x8 * x2


def zipf_c(R: int) -> float:
    lo, hi = 1.0, 16.0
    for _ in range(60):
        mid = (lo + hi) * 0.5
        if pow10(mid) <= float(R):
            lo = mid
        else:
            hi = mid
    return lo


def zipf_rank(r: np.ndarray, R: int) -> np.ndarray:
    c = zipf_c(R)
    u = (np.asarray(r, dtype=np.uint64) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    x = 1.0 + u * (c - 1.0)
    y = pow10(x)
    return np.minimum(np.floor(y).astype(np.int64) - 1, R - 1)


def zipf_rows(r: np.ndarray, R: int, t: int) -> np.ndarray:
    rank = zipf_rank(r, R).astype(np.uint64)
    return ((rank * np.uint64(ZIPF_MULT) + np.uint64(ZIPF_T_OFF * t)) % np.uint64(R)).astype(np.int64)


def dense_features(seed: int, F: int, q: np.ndarray, it: np.ndarray) -> np.ndarray:
    """dense [B][F] in float64 (exact int8 * 2^-7 values) (G4, round 2): feature f
    of (q, item) is byte f mod 16 of the 16-byte little-endian output (w0, w1, w2, w3) of
    philox((f // 16, item, 3, q)), read as int8, times 2^-7."""
    k0, k1 = seed_key(seed)
    nblk = (F + 15) // 16
    blk = np.arange(nblk, dtype=np.uint64).reshape(1, -1)
    w = philox(blk, it.astype(np.uint64).reshape(-1, 1), np.uint64(3),
               q.astype(np.uint64).reshape(-1, 1), k0, k1)            # 4 x [B][nblk]
    B = np.asarray(it).size
    out = np.empty((B, nblk * 16), dtype=np.float64)
    for j in range(16):                                                # byte j of the block
        word = w[j // 4]
        out[:, j::16] = _int8_low_byte(word >> np.uint64(8 * (j % 4))).astype(np.float64)
    return out[:, :F] * 2.0 ** -7


def gen_batch(cfg, seed: int, segs, rows: Sequence[int] = None):
    """(indices int32 [nnz], offsets int32 [T*B+1], dense float32 [B][F]) for a batch.

    Table-major CSR: bag g = t*B + b, offsets = exclusive prefix sum of lengths
    over g, offsets[T*B] = nnz (G3).
    """
    q, it = expand_segments(segs)
    T = cfg.num_tables
    rows = [cfg.rows] * T if rows is None else list(rows)
    lens = bag_lengths(seed, cfg, q, it)
    idx = [bag_indices(seed, cfg, t, q, it, lens[t], rows[t]) for t in range(T)]
    indices = np.concatenate(idx) if idx else np.zeros(0, np.int64)
    offsets = np.zeros(T * q.size + 1, dtype=np.int64)
    offsets[1:] = np.cumsum(lens.reshape(-1))
    dense = dense_features(seed, cfg.dense_dim, q, it)
    return indices.astype(np.int32), offsets.astype(np.int32), dense.astype(np.float32)
