"""The batched DLRM query forward, written out from its definition, in float64.

TEST INFRASTRUCTURE (see oracle/__init__.py).

PAPER.md:140-141 — a recommendation model is "a SparseNet with memory-intensive
sparse operations on embeddings and a DenseNet with compute-intensive
operations"; Table I gives, per model, the embedding tables
with multi-hot lookups and pooling, a Bottom-FC and a Predict-FC stack.  The
interaction between them is not written in the paper (only Fig. rec_char(a),
PAPER.md:127, and the DLRM citation); reading R1 takes
DLRM's pairwise dot interaction without self-pairs.

  F1 SLS      p[b][t] = sum_{j in bag(t,b)} E_t[idx_j]
  F2 bottom   h_{l+1} = ReLU(W_l h_l + b_l) for every layer          (Table I Bottom-FC; R2)
  F3 interact Z = X X^T, X = [x; p_0; ...; p_{T-1}];
              v = [x, Z(1,0), Z(2,0), Z(2,1), ..., Z(T,T-1)]         (R1)
  F4 top      ReLU hidden layers, last (width 1) linear -> logit,
              ctr = 1 / (1 + exp(-logit))                            (Table I Predict-FC; R2)

MT-WnD (Table I row 4; readings R26-R29): one-hot lookups (F1 with bags of one
index), no Bottom-FC, u = [p_0, ..., p_{T-1}] (concatenation, T*D), and per task k
  logit_k = tower_k(u) + <v_k, u>,  ctr_k = sigmoid(logit_k)      (deep tower + wide part)
"""
from __future__ import annotations

import numpy as np

from . import gen


def sls(table_rows_fn, T: int, B: int, D: int, indices: np.ndarray, offsets: np.ndarray,
        fp32_sequential: bool = False) -> np.ndarray:
    """F1: pooled [B][T][D].

    table_rows_fn(t, rows) -> float64 [len(rows)][D] gives E_t rows.  Bag g = t*B + b
    spans indices[offsets[g]:offsets[g+1]] (table-major CSR).  Empty bag -> zero
    vector; duplicate indices count with multiplicity (reading R9).

    fp32_sequential=True sums each bag in float32 strictly in index order
    (np.cumsum, not the pairwise np.add.reduce) for bit-exact comparison with a
    kernel that accumulates sequentially in fp32.
    """
    out = np.zeros((B, T, D), dtype=np.float32 if fp32_sequential else np.float64)
    for t in range(T):
        lo, hi = int(offsets[t * B]), int(offsets[(t + 1) * B])
        seg = indices[lo:hi]
        if seg.size == 0:
            continue
        uniq, inv = np.unique(seg, return_inverse=True)
        vals = table_rows_fn(t, uniq)[inv]                       # [n][D] float64
        for b in range(B):
            s, e = int(offsets[t * B + b]) - lo, int(offsets[t * B + b + 1]) - lo
            if e <= s:
                continue
            if fp32_sequential:
                out[b, t] = np.cumsum(vals[s:e].astype(np.float32), axis=0, dtype=np.float32)[-1]
            else:
                out[b, t] = vals[s:e].sum(axis=0)
    return out


def mlp(h: np.ndarray, layers, relu_last: bool) -> np.ndarray:
    """Chained FC layers h <- act(h W^T + b) in float64 (F2 / F4)."""
    n = len(layers)
    for l, (W, b) in enumerate(layers):
        h = h @ W.T + b
        if l < n - 1 or relu_last:
            h = np.maximum(h, 0.0)
    return h


def interaction(x: np.ndarray, pooled: np.ndarray) -> np.ndarray:
    """F3: v [B][D + T(T+1)/2], strict lower triangle of X X^T, row-major over i, j < i."""
    B, T, D = pooled.shape
    X = np.concatenate([x.reshape(B, 1, D), pooled], axis=1)    # [B][T+1][D]
    Z = np.einsum("bid,bjd->bij", X, X)
    ii, jj = np.tril_indices(T + 1, k=-1)                       # row-major: (1,0),(2,0),(2,1),...
    return np.concatenate([x, Z[:, ii, jj]], axis=1)


def sigmoid(z: np.ndarray) -> np.ndarray:
    return 1.0 / (1.0 + np.exp(-z))


def forward(cfg, seed: int, dense: np.ndarray, indices: np.ndarray, offsets: np.ndarray,
            params=None, rows=None, return_all: bool = False):
    """F1-F4 for one batch: CTR [B] (float64).  `params` from gen.model_params."""
    T, D = cfg.num_tables, cfg.dim
    B = dense.shape[0]
    if params is None:
        params = gen.model_params(cfg, seed)
    bottom, top = params
    shift = gen.emb_shift(cfg.pooling_lo, cfg.pooling_hi)
    rows_fn = lambda t, r: gen.table_values(seed, t, r, D, shift, cfg.value_mode)
    pooled = sls(rows_fn, T, B, D, np.asarray(indices), np.asarray(offsets))
    if getattr(cfg, "arch", 0) == 1:
        return forward_mtwnd(pooled, top, return_all)
    x = mlp(np.asarray(dense, dtype=np.float64), bottom, relu_last=True)
    v = interaction(x, pooled)
    logit = mlp(v, top, relu_last=False)[:, 0]
    ctr = sigmoid(logit)
    if return_all:
        return dict(pooled=pooled, x=x, v=v, logit=logit, ctr=ctr)
    return ctr


def forward_mtwnd(pooled: np.ndarray, towers_wide, return_all: bool = False):
    """MT-WnD: CTR [B][N] (float64) from pooled [B][T][D] and (towers, wide) (R26-R28)."""
    towers, wide = towers_wide
    B = pooled.shape[0]
    u = pooled.reshape(B, -1)
    logit = np.stack([mlp(u, tw, relu_last=False)[:, 0] + u @ v for tw, v in zip(towers, wide)],
                     axis=1)
    ctr = sigmoid(logit)
    if return_all:
        return dict(pooled=pooled, x=np.zeros((B, 0)), v=u, logit=logit, ctr=ctr)
    return ctr
