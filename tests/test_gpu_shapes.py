"""GPU parity over the shape space the C ABI accepts (include/rec.h: D a multiple of 4 up to
128, any T >= 1, ragged bags including empty ones, any 1 <= B <= max_batch).

Each case runs the caller-index path (rec_query_inspect: host indices/offsets -> k_sls,
bottom MLP, k_interact, top MLP) and the captured-graph path (rec_synth_query_async: inputs
materialised on the device) on the same items and checks, against the CPU oracle:
  * pooled X slots 1..T bit-exact (int8-exact tables, SURVEY §8(c) SLS pin);
  * the bottom output x = X slot 0 within the bf16-MLP tolerance of the fp64 oracle;
  * the interaction row A_top element-wise (a5; R1, R10): the x part is bf16-RN(x) bit-exact,
    every pair Z(i, j) (strict lower triangle, row-major) within 1 bf16 ulp of the fp64 dot
    product of the GPU's own fp32 X rows (plus the fp32 accumulation slack), padding zero;
  * CTR within 2e-2 of the oracle (BASELINE north_star) with a non-vacuous logit spread;
  * both paths give identical CTR bits.
Shapes: D in {4, 16, 48, 96, 128} (LANES 8 / 16 / 32 SLS paths, partially active lane groups,
32/64/128-wide GEMM tiles) x T in {1, 3, 26}; B in {1, 129, 1024} (one row, a ragged tail over
two 128-row tiles, eight tiles).
"""
import numpy as np
import pytest

import workloads as W
from oracle import forward as fw, gen

pytestmark = pytest.mark.gpu

CTR_TOL = 2e-2
# first-top-layer scale per (D, T) (reading R21: a per-config power of two that keeps the
# logit spread in [0.5, 4] so the CTR check is non-vacuous; chosen with the oracle alone)
TOP_SHIFT = {(4, 1): -1, (16, 1): -2, (48, 1): -2, (96, 1): -2, (128, 1): -2,
             (4, 3): 0, (16, 3): 0, (48, 3): 0, (96, 3): 0, (128, 3): 0,
             (4, 26): 0, (16, 26): 1, (48, 26): 1, (96, 26): 2, (128, 26): 2}
DIMS = (4, 16, 48, 96, 128)
TABLES = (1, 3, 26)
ROWS = 3000


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__
    __graft_entry__.build()


def _cfg(D, T):
    # ragged bags: lengths U[0, 6] (G3), so empty bags occur in every batch
    return W.ModelConfig(f"sweep-D{D}-T{T}", T, ROWS, D, 0, 6, (13, 64, D), (64, 16, 1),
                         TOP_SHIFT[(D, T)], 1024, 20.0)


def bf16_rn_bits(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 round-to-nearest-even, as bit patterns (plain definition, no NaNs here)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


def bf16_value(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def check_interaction(X: np.ndarray, A: np.ndarray, T: int, D: int):
    """A_top rows against the fp64 interaction of the GPU's own X (a5 element-wise)."""
    B = X.shape[0]
    K = D + T * (T + 1) // 2
    assert np.array_equal(A[:, :D], bf16_rn_bits(X[:, 0, :]))           # x part, bit-exact
    assert np.all(A[:, K:] == 0)                                         # zero padding
    X64 = X.astype(np.float64)
    ii, jj = np.tril_indices(T + 1, k=-1)                                # (1,0),(2,0),(2,1),...
    ref = np.einsum("bpd,bpd->bp", X64[:, ii, :], X64[:, jj, :])         # exact-ish fp64 dots
    mag = np.einsum("bpd,bpd->bp", np.abs(X64[:, ii, :]), np.abs(X64[:, jj, :]))
    got = bf16_value(A[:, D:K])
    ulp = np.exp2(np.floor(np.log2(np.maximum(np.abs(ref), 1e-30))) - 7)  # 1 bf16 ulp of ref
    bound = ulp + D * 2.0 ** -23 * mag                                    # + fp32 FMA-chain slack
    err = np.abs(got - ref)
    assert np.all(err <= bound), (float(err.max()), np.unravel_index(np.argmax(err - bound), err.shape))
    return ref


@pytest.mark.parametrize("T", TABLES)
@pytest.mark.parametrize("D", DIMS)
def test_shape_sweep(D, T):
    import torch
    from paper_2203_07424_b200 import RecModel
    cfg = _cfg(D, T)
    m = RecModel(cfg, seed=1, max_batch=1024)
    for B in (1, 129, 1024):
        segs = W.random_segments(B, seed=1000 * D + 10 * T + B % 7, max_seg=97)
        ind, off, dense = gen.gen_batch(cfg, 1, segs)
        if B >= 129:
            assert np.any(np.diff(off) == 0)                             # empty bags present
        # captured-graph path first (device-materialised inputs), then the eager path
        cv = torch.zeros(B, device="cuda")
        m.rec_synth_query_async(0, segs, cv)
        m.rec_sync(0)
        ctr, X, A = m.rec_query_inspect(dense, ind, off, B)
        exp = fw.forward(cfg, 1, dense, ind, off, return_all=True)
        # a3: pooled bit-exact
        assert np.array_equal(X[:, 1:, :].astype(np.float64), exp["pooled"]), "pooled"
        # a4: bottom output vs the fp64 oracle (bf16 operands, fp32 accumulate)
        xs = np.maximum(1.0, np.abs(exp["x"]).max(axis=1, keepdims=True))
        assert np.all(np.abs(X[:, 0, :] - exp["x"]) <= 1e-2 * xs), "bottom MLP"
        # a5: interaction row element-wise
        check_interaction(X, A, T, D)
        # a6: CTR
        err = np.abs(ctr.astype(np.float64) - exp["ctr"])
        assert err.max() <= CTR_TOL, (B, float(err.max()))
        if B == 1024:
            s = exp["logit"].std()
            assert 0.5 <= s <= 4.0, s                                    # non-vacuous
        assert np.array_equal(cv.cpu().numpy(), ctr), "graph path != eager path"
    m.close()


def test_interaction_check_has_teeth():
    """Negative control for check_interaction: a one-ulp-scale corruption of one pair, a
    swapped pair order, or a dropped x part each fail it."""
    cfg = _cfg(16, 3)
    from paper_2203_07424_b200 import RecModel
    m = RecModel(cfg, seed=1, max_batch=256)
    segs = W.random_segments(200, seed=3)
    ind, off, dense = gen.gen_batch(cfg, 1, segs)
    _, X, A = m.rec_query_inspect(dense, ind, off, 200)
    ref = check_interaction(X, A, 3, 16)
    D = 16
    b, p = np.unravel_index(np.argmax(np.abs(ref)), ref.shape)
    bad = A.copy()
    bad[b, D + p] = bad[b, D + p] ^ np.uint16(0x0002)                   # 2 ulps off
    with pytest.raises(AssertionError):
        check_interaction(X, bad, 3, D)
    bad = A.copy()
    bad[:, [D + 1, D + 2]] = bad[:, [D + 2, D + 1]]                     # Z(2,0) <-> Z(2,1)
    with pytest.raises(AssertionError):
        check_interaction(X, bad, 3, D)
    bad = A.copy()
    bad[:, :D] = 0
    with pytest.raises(AssertionError):
        check_interaction(X, bad, 3, D)
    m.close()
