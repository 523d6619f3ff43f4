"""Seeded synthetic workload definitions shared by the oracle, the tests and bench.py.

This module holds NONE of the method's arithmetic (no Philox, no SLS, no MLP,
no split/fuse).  It only states

* the model shapes of the paper's DLRM configurations (Table I, PAPER.md:188-190,
  as fixed by BASELINE.json ``configs`` and the readings in DESIGN.md §3), and
* seeded generators of *inputs*: query traces (Poisson arrivals, heavy-tailed
  sizes) and item-segment lists for parity batches.

Both ``oracle/`` and the CUDA path consume these values as plain inputs.
"""
from __future__ import annotations

from dataclasses import dataclass, field, asdict
from typing import List, Tuple

import numpy as np

REC_VALUES_INT8_EXACT = 0
REC_VALUES_FP32 = 1

INDEX_UNIFORM = 0
INDEX_SKEW2 = 2
INDEX_ZIPF = 3   # Zipf(0.9) rows scattered by a fixed bijection (G2z)

ARCH_DLRM = 0    # SLS -> bottom MLP -> dot interaction -> top MLP (Table I rows 1-3)
ARCH_MTWND = 1   # one-hot lookups -> concat -> N task towers + wide part (Table I row 4; R26-R29)


@dataclass(frozen=True)
class ModelConfig:
    """One DLRM configuration (Table I).

    bottom: layer widths INCLUDING the dense-input width, e.g. [256, 128, 32]
            (reading R3).
    top:    layer widths EXCLUDING the interaction width, ending in 1
            (reading R3).
    top_shift: extra power-of-two down-scaling of the first top layer's weights,
            a per-config spec constant (reading R21) that keeps the
            logit spread in the non-vacuous range.
    """
    name: str
    num_tables: int
    rows: int
    dim: int
    pooling_lo: int
    pooling_hi: int
    bottom: Tuple[int, ...]
    top: Tuple[int, ...]
    top_shift: int
    batch: int
    sla_ms: float
    value_mode: int = REC_VALUES_INT8_EXACT
    index_dist: int = INDEX_UNIFORM
    arch: int = ARCH_DLRM
    tasks: int = 1            # MT-WnD: number of task towers N (reading R27)

    @property
    def dense_dim(self) -> int:
        return self.bottom[0] if self.bottom else 0

    @property
    def top_in(self) -> int:
        """Width of the first top / tower layer's input: the interaction vector (DLRM) or
        the concatenated embeddings (MT-WnD, reading R26)."""
        T, D = self.num_tables, self.dim
        return T * D if self.arch == ARCH_MTWND else D + T * (T + 1) // 2

    @property
    def pooling_fixed(self) -> bool:
        return self.pooling_lo == self.pooling_hi

    def with_(self, **kw) -> "ModelConfig":
        d = asdict(self)
        d.update(kw)
        d["bottom"] = tuple(d["bottom"])
        d["top"] = tuple(d["top"])
        return ModelConfig(**d)


# BASELINE.json configs[0]: "DLRM-tiny: 8 tables x 10k rows x dim 32, pooling 20,
# bottom MLP 13-64-32, top MLP 64-1, batch 64"
TINY = ModelConfig("DLRM-tiny", 8, 10_000, 32, 20, 20, (13, 64, 32), (64, 1), 2, 64, 20.0)
# BASELINE.json configs[1] + Table I row RMC1; SLA 20 ms
RMC1 = ModelConfig("DLRM-RMC1", 10, 1_000_000, 32, 80, 80, (256, 128, 32), (256, 64, 1), 2, 1024, 20.0)
# BASELINE.json configs[2] + Table I row RMC2; bottom ends in 64 = dim
# (reading R4); SLA 50 ms
RMC2 = ModelConfig("DLRM-RMC2", 40, 1_000_000, 64, 120, 120, (256, 128, 64), (512, 128, 1), 0, 1024, 50.0)
# BASELINE.json configs[3] + Table I row RMC3; pooling 20 (reading R5);
# SLA 50 ms
RMC3 = ModelConfig("DLRM-RMC3", 10, 1_000_000, 32, 20, 20, (2560, 512, 32), (512, 128, 1), 1, 1024, 50.0)

# SURVEY §8(f) 4 / Table I row MT-WnD: 26 tables, one-hot lookups (pooling
# 1, no Gather-Reduce), no Bottom-FC, Predict-FC N x (1024-512-256); SLA 100 ms.
# dim 32 and N = 2 tasks are readings R26/R27; top_shift keeps the logits non-vacuous (R21).
MTWND = ModelConfig("MT-WnD", 26, 1_000_000, 32, 1, 1, (), (1024, 512, 256, 1), 0, 1024, 100.0,
                    arch=ARCH_MTWND, tasks=2)

CONFIGS = {c.name: c for c in (TINY, RMC1, RMC2, RMC3, MTWND)}
SHORT = {"tiny": TINY, "rmc1": RMC1, "rmc2": RMC2, "rmc3": RMC3, "mtwnd": MTWND}


def small_variant(cfg: ModelConfig, rows: int = 4096) -> ModelConfig:
    """Same layer shapes, fewer rows per table (for oracle-fast parity tests)."""
    return cfg.with_(rows=rows)


# ----------------------------------------------------------------------------------
# Query traces (inputs to rec_serve).  PAPER.md:78 "the query arrival pattern follows
# the Poisson distribution ... heavy-tail distribution of query sizes"
# sizes "typically varying between 10 and 1000".  Reading R13: lognormal
# (mu = ln 100, sigma = 1) truncated to [1, 1000] by resampling.
# ----------------------------------------------------------------------------------
TRACE_DTYPE = np.dtype([("arrival_s", "<f8"), ("size", "<i4"), ("qid", "<i4")])


def query_sizes(n: int, seed: int, lo: int = 1, hi: int = 1000,
                mu: float = float(np.log(100.0)), sigma: float = 1.0) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    out = np.empty(n, dtype=np.int64)
    filled = 0
    while filled < n:
        draw = np.floor(rng.lognormal(mu, sigma, size=max(2 * (n - filled), 64)))
        draw = draw[(draw >= lo) & (draw <= hi)]
        take = min(n - filled, draw.size)
        out[filled:filled + take] = draw[:take]
        filled += take
    return out.astype(np.int32)


def poisson_trace(rate_qps: float, n: int, seed: int, **size_kw) -> np.ndarray:
    """n queries with exponential inter-arrivals (mean 1/rate) and lognormal sizes."""
    rng = np.random.Generator(np.random.PCG64(seed ^ 0x5EED))
    gaps = rng.exponential(1.0 / rate_qps, size=n)
    tr = np.zeros(n, dtype=TRACE_DTYPE)
    tr["arrival_s"] = np.cumsum(gaps) - gaps[0]
    tr["size"] = query_sizes(n, seed, **size_kw)
    tr["qid"] = np.arange(n, dtype=np.int32)
    return tr


def burst_trace(n: int, seed: int, **size_kw) -> np.ndarray:
    """All queries present at t=0 (saturation / throughput workload)."""
    tr = np.zeros(n, dtype=TRACE_DTYPE)
    tr["size"] = query_sizes(n, seed, **size_kw)
    tr["qid"] = np.arange(n, dtype=np.int32)
    return tr


def random_segments(batch: int, seed: int, max_qid: int = 1 << 20,
                    max_seg: int = 300) -> np.ndarray:
    """A list of (qid, start, len) item segments totalling exactly `batch` items.

    Pure input generation: which (query, item) pairs make up a parity batch.
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    segs: List[Tuple[int, int, int]] = []
    left = batch
    while left > 0:
        ln = int(min(left, rng.integers(1, max_seg + 1)))
        segs.append((int(rng.integers(0, max_qid)), int(rng.integers(0, 1000)), ln))
        left -= ln
    return np.asarray(segs, dtype=np.int32).reshape(-1, 3)


__all__ = [
    "ModelConfig", "TINY", "RMC1", "RMC2", "RMC3", "MTWND", "CONFIGS", "SHORT", "small_variant",
    "ARCH_DLRM", "ARCH_MTWND",
    "TRACE_DTYPE", "query_sizes", "poisson_trace", "burst_trace", "random_segments",
    "REC_VALUES_INT8_EXACT", "REC_VALUES_FP32", "INDEX_UNIFORM", "INDEX_SKEW2", "INDEX_ZIPF",
]
