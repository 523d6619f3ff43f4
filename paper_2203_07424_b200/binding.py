"""ctypes binding of include/rec.h (argument marshalling only).

Every computation happens inside libhercules_rec.so (sm_100a kernels + C++ runtime).
There is no Python or CPU fallback: if the library is missing this module raises at
import-use time, and without a B200 rec_model_create returns REC_E_CUDA.

Arrays may be NumPy arrays (host memory) or torch CUDA tensors (device memory); raw
integer addresses are passed through unchanged.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("REC_LIB_PATH") or os.path.join(HERE, "libhercules_rec.so")

REC_OK = 0
STATUS = {0: "REC_OK", -1: "REC_E_INVALID_ARG", -2: "REC_E_INDEX_OOB", -3: "REC_E_OFFSETS",
          -4: "REC_E_OOM", -5: "REC_E_CUDA", -6: "REC_E_NCCL", -7: "REC_E_UNSUPPORTED"}
REC_VALUES_INT8_EXACT, REC_VALUES_FP32 = 0, 1
REC_INDEX_UNIFORM, REC_INDEX_SKEW2, REC_INDEX_ZIPF = 0, 2, 3
REC_SHARD_REPLICA, REC_SHARD_TABLE, REC_SHARD_ROW = 0, 1, 2
REC_INPUT_DEVICE_SYNTH, REC_INPUT_HOST = 0, 1
REC_CLOCK_REAL, REC_CLOCK_VIRTUAL = 0, 1
KERNEL_SLS, KERNEL_GEMM, KERNEL_INTERACT, KERNEL_GEN = 0, 1, 2, 3

EXPORTS = ["rec_model_create", "rec_model_destroy", "rec_query", "rec_query_debug",
           "rec_query_async", "rec_synth_query_async", "rec_sync", "rec_stream_handle",
           "rec_gen_batch", "rec_profile", "rec_profile_read", "rec_serve", "rec_last_error",
           "rec_nccl_unique_id_size", "rec_nccl_get_unique_id", "rec_version", "rec_split_fuse",
           "rec_synth_query_batches", "rec_shard_plan", "rec_bench_mlp", "rec_bench_sls", "rec_set_pipeline", "rec_synth_query_pipeline",
           "rec_debug_chain_timeline", "rec_query_inspect", "rec_hot_remap",
           "rec_bench_sls_caller", "rec_global_batches"]


class rec_model_desc(C.Structure):
    _fields_ = [("num_tables", C.c_int32), ("rows", C.POINTER(C.c_int64)), ("dim", C.c_int32),
                ("pooling_lo", C.c_int32), ("pooling_hi", C.c_int32),
                ("bottom_widths", C.POINTER(C.c_int32)), ("n_bottom", C.c_int32),
                ("top_widths", C.POINTER(C.c_int32)), ("n_top", C.c_int32),
                ("top_shift", C.c_int32), ("seed", C.c_uint64), ("value_mode", C.c_int32),
                ("index_dist", C.c_int32), ("max_batch", C.c_int32), ("streams", C.c_int32),
                ("device", C.c_int32), ("shard", C.c_int32), ("rank", C.c_int32),
                ("world", C.c_int32), ("nccl_id", C.c_void_p), ("l2_persist_bytes", C.c_int64),
                ("arch", C.c_int32), ("n_tasks", C.c_int32)]


class rec_serve_policy(C.Structure):
    _fields_ = [("streams", C.c_int32), ("max_batch", C.c_int32), ("fusion_timeout_ms", C.c_double),
                ("input_mode", C.c_int32), ("clock", C.c_int32), ("alpha_ns", C.c_double),
                ("beta_ns", C.c_double), ("warmup_frac", C.c_double)]


class rec_serve_report(C.Structure):
    _fields_ = [("offered_qps", C.c_double), ("achieved_qps", C.c_double), ("mean_ms", C.c_double),
                ("p50_ms", C.c_double), ("p95_ms", C.c_double), ("p99_ms", C.c_double),
                ("breakdown_ms", C.c_double * 4), ("completed", C.c_int64), ("dropped", C.c_int64),
                ("batches", C.c_int64), ("mean_batch", C.c_double), ("sla_met", C.c_int32),
                ("stable", C.c_int32), ("ranks", C.c_int32)]

    def as_dict(self) -> dict:
        d = {k: getattr(self, k) for k, _ in self._fields_ if k != "breakdown_ms"}
        d["breakdown_ms"] = list(self.breakdown_ms)
        return d


_LIB = None


def lib() -> C.CDLL:
    """Load libhercules_rec.so (fail loudly if it was not built)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                               "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
        L.rec_model_create.argtypes = [C.POINTER(rec_model_desc), C.POINTER(vp)]
        L.rec_model_destroy.argtypes = [vp]
        L.rec_model_destroy.restype = None
        L.rec_query.argtypes = [vp, vp, vp, vp, i32, vp]
        L.rec_query_debug.argtypes = [vp, vp, vp, vp, i32, vp, vp, vp]
        L.rec_query_async.argtypes = [vp, i32, vp, vp, vp, i64, i32, vp]
        L.rec_synth_query_async.argtypes = [vp, i32, vp, i32, vp]
        L.rec_sync.argtypes = [vp, i32]
        L.rec_stream_handle.argtypes = [vp, i32]
        L.rec_stream_handle.restype = vp
        L.rec_gen_batch.argtypes = [vp, vp, i32, vp, vp, vp]
        L.rec_profile.argtypes = [vp, i32]
        L.rec_profile_read.argtypes = [vp, i32, C.POINTER(C.c_double), C.POINTER(i64)]
        L.rec_serve.argtypes = [vp, vp, i64, C.c_double, C.POINTER(rec_serve_policy),
                                C.POINTER(rec_serve_report), vp, vp, i64, C.POINTER(i64), vp]
        L.rec_last_error.restype = C.c_char_p
        L.rec_nccl_unique_id_size.restype = i32
        L.rec_nccl_get_unique_id.argtypes = [vp]
        L.rec_version.restype = i32
        L.rec_split_fuse.argtypes = [vp, i64, i32, vp, i64, vp, i64, C.POINTER(i64), C.POINTER(i64)]
        L.rec_split_fuse.restype = i32
        L.rec_synth_query_batches.argtypes = [vp, vp, vp, i64, i32]
        L.rec_synth_query_batches.restype = i32
        L.rec_shard_plan.argtypes = [i32, vp, i32, i32, i32, i32, vp]
        L.rec_shard_plan.restype = i32
        L.rec_bench_mlp.argtypes = [vp, i32, i32, i32, C.POINTER(C.c_double)]
        L.rec_bench_mlp.restype = i32
        L.rec_bench_sls.argtypes = [vp, vp, vp, i32, i32, C.POINTER(C.c_double)]
        L.rec_bench_sls.restype = i32
        L.rec_set_pipeline.argtypes = [vp, i32]
        L.rec_set_pipeline.restype = i32
        L.rec_synth_query_pipeline.argtypes = [vp, vp, vp, C.c_int64, vp]
        L.rec_synth_query_pipeline.restype = i32
        L.rec_debug_chain_timeline.argtypes = [vp, i32, i32, vp]
        L.rec_debug_chain_timeline.restype = i32
        L.rec_query_inspect.argtypes = [vp, vp, vp, vp, i32, vp, vp, vp, C.POINTER(i32)]
        L.rec_query_inspect.restype = i32
        L.rec_hot_remap.argtypes = [vp, vp, vp, i32, i64, C.POINTER(i64)]
        L.rec_hot_remap.restype = i32
        L.rec_bench_sls_caller.argtypes = [vp, vp, vp, i32, i32, i64, C.POINTER(C.c_double)]
        L.rec_bench_sls_caller.restype = i32
        L.rec_global_batches.argtypes = [vp, i64, i32, C.c_double, vp, i64, vp, vp, i64,
                                         C.POINTER(i64), C.POINTER(i64)]
        L.rec_global_batches.restype = i32
        for f in ("rec_model_create", "rec_query", "rec_query_debug", "rec_query_async",
                  "rec_synth_query_async", "rec_sync", "rec_gen_batch", "rec_profile",
                  "rec_profile_read", "rec_serve", "rec_nccl_get_unique_id"):
            getattr(L, f).restype = i32
        _LIB = L
    return _LIB


class RecError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def _check(st: int):
    if st != REC_OK:
        raise RecError(st, lib().rec_last_error().decode())


def _ptr(x) -> Optional[int]:
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if isinstance(x, np.ndarray):
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("arrays must be C-contiguous")
        return x.ctypes.data
    if hasattr(x, "data_ptr"):
        if not x.is_contiguous():
            raise ValueError("tensors must be contiguous")
        return x.data_ptr()
    raise TypeError(f"cannot pass {type(x)} as a pointer")


class RecModel:
    """Owning wrapper of a rec_model_t handle (methods mirror the C ABI names)."""

    def __init__(self, cfg, seed: int = 1, max_batch: Optional[int] = None, streams: int = 1,
                 device: int = 0, shard: int = REC_SHARD_REPLICA, rank: int = 0, world: int = 1,
                 nccl_id: Optional[bytes] = None, l2_persist_bytes: int = 0,
                 rows: Optional[list] = None):
        self.cfg = cfg
        T = cfg.num_tables
        self._rows = (C.c_int64 * T)(*([cfg.rows] * T if rows is None else rows))
        self._bottom = (C.c_int32 * len(cfg.bottom))(*cfg.bottom)
        self._top = (C.c_int32 * len(cfg.top))(*cfg.top)
        self._nccl = C.create_string_buffer(nccl_id, len(nccl_id)) if nccl_id else None
        d = rec_model_desc()
        d.num_tables = T
        d.rows = self._rows
        d.dim = cfg.dim
        d.pooling_lo, d.pooling_hi = cfg.pooling_lo, cfg.pooling_hi
        d.bottom_widths, d.n_bottom = self._bottom, len(cfg.bottom)
        d.top_widths, d.n_top = self._top, len(cfg.top)
        d.top_shift = cfg.top_shift
        d.seed = seed
        d.value_mode = cfg.value_mode
        d.index_dist = cfg.index_dist
        d.max_batch = max_batch if max_batch is not None else cfg.batch
        d.streams = streams
        d.device = device
        d.shard, d.rank, d.world = shard, rank, world
        d.nccl_id = C.cast(self._nccl, C.c_void_p) if self._nccl is not None else None
        d.l2_persist_bytes = l2_persist_bytes
        d.arch = getattr(cfg, "arch", 0)
        d.n_tasks = getattr(cfg, "tasks", 1)
        self.desc = d
        self.max_batch = d.max_batch
        self.streams = streams
        h = C.c_void_p()
        _check(lib().rec_model_create(C.byref(d), C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().rec_model_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------- queries
    def rec_query(self, dense, indices, offsets, batch: int, ctr):
        _check(lib().rec_query(self.h, _ptr(dense), _ptr(indices), _ptr(offsets), batch, _ptr(ctr)))

    def rec_query_debug(self, dense, indices, offsets, batch: int, ctr, pooled=None, logits=None):
        _check(lib().rec_query_debug(self.h, _ptr(dense), _ptr(indices), _ptr(offsets), batch,
                                     _ptr(ctr), _ptr(pooled), _ptr(logits)))

    def rec_query_inspect(self, dense, indices, offsets, batch: int):
        """(ctr [B(,N)], X [B][T+1][D] fp32, A_top [B][ld] as uint16 bf16 bit patterns)."""
        cfg = self.cfg
        tasks = getattr(cfg, "tasks", 1)
        ctr = np.zeros((batch, tasks) if tasks > 1 else batch, dtype=np.float32)
        x = np.zeros((batch, cfg.num_tables + 1, cfg.dim), dtype=np.float32)
        ld = C.c_int32()
        a = np.zeros((batch, ((cfg.top_in + 7) // 8) * 8), dtype=np.uint16)
        _check(lib().rec_query_inspect(self.h, _ptr(dense), _ptr(indices), _ptr(offsets), batch,
                                       _ptr(ctr), _ptr(x), _ptr(a), C.byref(ld)))
        assert ld.value == a.shape[1]
        return ctr, x, a

    def rec_hot_remap(self, indices, offsets, batch: int, window_bytes: int = 0) -> int:
        """Hot-row partition from a profiling sample; returns rows per table in the L2 window."""
        h = C.c_int64()
        _check(lib().rec_hot_remap(self.h, _ptr(indices), _ptr(offsets), batch, window_bytes, C.byref(h)))
        return h.value

    def rec_query_async(self, slot: int, dense, indices, offsets, nnz: int, batch: int, ctr):
        _check(lib().rec_query_async(self.h, slot, _ptr(dense), _ptr(indices), _ptr(offsets),
                                     nnz, batch, _ptr(ctr)))

    def rec_synth_query_async(self, slot: int, segs: np.ndarray, ctr):
        segs = np.ascontiguousarray(segs, dtype=np.int32).reshape(-1, 3)
        _check(lib().rec_synth_query_async(self.h, slot, _ptr(segs), segs.shape[0], _ptr(ctr)))

    def rec_synth_query_batches(self, segs: np.ndarray, batch_start: np.ndarray, first_slot: int = 0):
        segs = np.ascontiguousarray(segs, dtype=np.int32).reshape(-1, 3)
        bs = np.ascontiguousarray(batch_start, dtype=np.int64)
        _check(lib().rec_synth_query_batches(self.h, _ptr(segs), _ptr(bs), len(bs) - 1, first_slot))

    def rec_set_pipeline(self, lanes: int):
        _check(lib().rec_set_pipeline(self.h, lanes))

    def rec_synth_query_pipeline(self, segs: np.ndarray, batch_start: np.ndarray, ctr=None):
        segs = np.ascontiguousarray(segs, dtype=np.int32).reshape(-1, 3)
        bs = np.ascontiguousarray(batch_start, dtype=np.int64)
        _check(lib().rec_synth_query_pipeline(self.h, _ptr(segs), _ptr(bs), len(bs) - 1,
                                              _ptr(ctr) if ctr is not None else None))

    def rec_sync(self, slot: int = 0):
        _check(lib().rec_sync(self.h, slot))

    def rec_stream_handle(self, slot: int = 0) -> int:
        return lib().rec_stream_handle(self.h, slot)

    def rec_gen_batch(self, segs: np.ndarray):
        segs = np.ascontiguousarray(segs, dtype=np.int32).reshape(-1, 3)
        cfg = self.cfg
        B = int(segs[:, 2].sum())
        ind = np.zeros(cfg.num_tables * B * max(cfg.pooling_hi, 1), dtype=np.int32)
        off = np.zeros(cfg.num_tables * B + 1, dtype=np.int32)
        dense = np.zeros((B, cfg.dense_dim), dtype=np.float32)
        _check(lib().rec_gen_batch(self.h, _ptr(segs), segs.shape[0], _ptr(ind), _ptr(off), _ptr(dense)))
        return ind[:off[-1]].copy(), off, dense

    def rec_bench_mlp(self, which: int, batch: int, iters: int = 50) -> float:
        ms = C.c_double()
        _check(lib().rec_bench_mlp(self.h, which, batch, iters, C.byref(ms)))
        return ms.value

    def rec_bench_sls(self, segs: np.ndarray, batch_start: np.ndarray, pdl: bool = True) -> float:
        """Total CUDA-event ms of one SLS launch per batch, back to back (see rec.h)."""
        segs = np.ascontiguousarray(segs, dtype=np.int32).reshape(-1, 3)
        bs = np.ascontiguousarray(batch_start, dtype=np.int64)
        ms = C.c_double()
        _check(lib().rec_bench_sls(self.h, _ptr(segs), _ptr(bs), len(bs) - 1, int(pdl), C.byref(ms)))
        return ms.value

    def rec_bench_sls_caller(self, indices, offsets, batch: int, nbatches: int, idx_stride: int) -> float:
        """Total CUDA-event ms of nbatches caller-index SLS launches (device arrays, rec.h)."""
        ms = C.c_double()
        _check(lib().rec_bench_sls_caller(self.h, _ptr(indices), _ptr(offsets), batch, nbatches,
                                          idx_stride, C.byref(ms)))
        return ms.value

    def rec_debug_chain_timeline(self, which: int, batch: int):
        out = np.zeros(16, dtype=np.int64)
        _check(lib().rec_debug_chain_timeline(self.h, which, batch, _ptr(out)))
        return out

    def rec_profile(self, enable: bool):
        _check(lib().rec_profile(self.h, 1 if enable else 0))

    def rec_profile_read(self, kernel: int):
        ms, n = C.c_double(), C.c_int64()
        _check(lib().rec_profile_read(self.h, kernel, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    # ---------------------------------------------------------------- serving
    def rec_serve(self, trace: np.ndarray, sla_ms: float, streams: int, max_batch: int,
                  fusion_timeout_ms: float = 0.0, input_mode: int = REC_INPUT_DEVICE_SYNTH,
                  clock: int = REC_CLOCK_REAL, alpha_ns: float = 0.0, beta_ns: float = 0.0,
                  warmup_frac: float = 0.1, want_latency: bool = True, log_cap: int = 0,
                  want_ctr: bool = False):
        trace = np.ascontiguousarray(trace)
        n = len(trace)
        pol = rec_serve_policy(streams, max_batch, fusion_timeout_ms, input_mode, clock, alpha_ns,
                               beta_ns, warmup_frac)
        rep = rec_serve_report()
        lat = np.zeros(n, dtype=np.float64) if want_latency else None
        log = np.zeros((max(log_cap, 0), 5), dtype=np.int32) if log_cap > 0 else None
        rows = C.c_int64(0)
        tasks = getattr(self.cfg, "tasks", 1)
        ctr = (np.zeros(int(trace["size"].astype(np.int64).sum()) * tasks, dtype=np.float32)
               if want_ctr else None)
        _check(lib().rec_serve(self.h, _ptr(trace), n, sla_ms, C.byref(pol), C.byref(rep), _ptr(lat),
                               _ptr(log), log_cap, C.byref(rows), _ptr(ctr)))
        out = rep.as_dict()
        out["latency_ms"] = lat
        out["batch_log"] = log[:rows.value] if log is not None else None
        out["ctr"] = ctr.reshape(-1, tasks) if ctr is not None and tasks > 1 else ctr
        return out


def rec_split_fuse(trace: np.ndarray, max_batch: int):
    """S1+S2 for a burst of pending queries (host-only C++).  Returns (segs [n][3], batch_start)."""
    trace = np.ascontiguousarray(trace)
    n = len(trace)
    cap = int(sum(-(-int(s) // max_batch) for s in trace["size"])) if n and max_batch > 0 else 0
    segs = np.zeros((max(cap, 1), 3), dtype=np.int32)
    bstart = np.zeros(cap + 2, dtype=np.int64)
    nb, ns = C.c_int64(), C.c_int64()
    _check(lib().rec_split_fuse(_ptr(trace), n, max_batch, _ptr(segs), cap, _ptr(bstart), cap + 1,
                                C.byref(nb), C.byref(ns)))
    return segs[:ns.value], bstart[:nb.value + 1]


def rec_global_batches(trace: np.ndarray, max_batch: int, tau_ms: float):
    """R31 deterministic global batch cut (host-only C++): (segs [n][3], batch_start, close_s)."""
    trace = np.ascontiguousarray(trace)
    n = len(trace)
    cap = int(sum(-(-int(s) // max_batch) for s in trace["size"])) if n and max_batch > 0 else 0
    segs = np.zeros((max(cap, 1), 3), dtype=np.int32)
    bstart = np.zeros(cap + 2, dtype=np.int64)
    close = np.zeros(cap + 1, dtype=np.float64)
    nb, ns = C.c_int64(), C.c_int64()
    _check(lib().rec_global_batches(_ptr(trace), n, max_batch, tau_ms, _ptr(segs), cap, _ptr(bstart),
                                    _ptr(close), cap + 1, C.byref(nb), C.byref(ns)))
    return segs[:ns.value], bstart[:nb.value + 1], close[:nb.value]


def rec_shard_plan(rows, world: int, rank: int, shard: int, batch: int) -> dict:
    """Host-only shard plan of `rank` (first/count of local tables, local row range, item block)."""
    r = np.ascontiguousarray(rows, dtype=np.int64)
    out = np.zeros(6, dtype=np.int64)
    _check(lib().rec_shard_plan(len(r), _ptr(r), world, rank, shard, batch, _ptr(out)))
    return dict(t0=int(out[0]), t_local=int(out[1]), row_lo=int(out[2]), row_hi=int(out[3]),
                item0=int(out[4]), items=int(out[5]))


def nccl_unique_id() -> bytes:
    n = lib().rec_nccl_unique_id_size()
    buf = C.create_string_buffer(n)
    _check(lib().rec_nccl_get_unique_id(buf))
    return buf.raw
