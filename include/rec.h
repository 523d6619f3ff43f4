/*
 * rec.h — C ABI of the B200-native DLRM query hot path under Hercules-style
 * recommendation inference serving (arXiv 2203.07424, "Hercules").
 *
 * Citations: P:n = line n of the paper text; DESIGN.md §n / Rn = this
 * repo's design notes and readings.  Library: libhercules_rec.so (sm_100a).
 *
 * Conventions for every call
 *   - Every function returns rec_status (REC_OK = 0) unless declared otherwise.
 *   - All array arguments are borrowed for the duration of the call; the library
 *     never retains a caller pointer.  Unless stated, a pointer may be host or
 *     device memory (detected with cudaPointerGetAttributes); host data is staged
 *     through library-owned pinned buffers.
 *   - Outputs are written only when the call returns REC_OK (for *_async calls:
 *     when the matching rec_sync returns REC_OK).
 *   - A model handle is not safe for concurrent calls from several host threads.
 *   - On error, rec_last_error() returns a thread-local message naming the field
 *     or the failing CUDA/NCCL call.  There is no CPU fallback: without a usable
 *     sm_100 device rec_model_create returns REC_E_CUDA.
 */
#ifndef HERCULES_REC_H
#define HERCULES_REC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  REC_OK = 0,
  REC_E_INVALID_ARG = -1,  /* null pointer, inconsistent widths, batch <= 0, bad policy   */
  REC_E_INDEX_OOB = -2,    /* an index outside [0, rows_t) (R9: no clamping)              */
  REC_E_OFFSETS = -3,      /* offsets[0] != 0, decreasing, or offsets[T*B] != nnz bound   */
  REC_E_OOM = -4,          /* device or pinned allocation failed                          */
  REC_E_CUDA = -5,         /* CUDA runtime/driver error (incl. no sm_100 device)          */
  REC_E_NCCL = -6,         /* NCCL error in a sharded model                               */
  REC_E_UNSUPPORTED = -7   /* D % 4 != 0, D > 128, rows >= 2^31, widths > limits          */
} rec_status;

enum { REC_VALUES_INT8_EXACT = 0, REC_VALUES_FP32 = 1 };           /* DESIGN.md G4        */
enum { REC_INDEX_UNIFORM = 0, REC_INDEX_SKEW2 = 2,                 /* DESIGN.md G2, R17   */
       REC_INDEX_ZIPF = 3 };   /* Zipf(0.9) rows scattered by a bijection (G2z) */
enum { REC_SHARD_REPLICA = 0, REC_SHARD_TABLE = 1, REC_SHARD_ROW = 2 };
enum { REC_INPUT_DEVICE_SYNTH = 0, REC_INPUT_HOST = 1 };
enum { REC_CLOCK_REAL = 0, REC_CLOCK_VIRTUAL = 1 };                 /* DESIGN.md S4        */

typedef struct rec_model_s* rec_model_t;   /* opaque; owns all device memory it allocated */

/*
 * Model description — "a recommendation model in the form of a computation graph
 * G_m" restricted to the DLRM class of Table I: T embedding
 * tables with multi-hot pooled lookups (SparseNet), a Bottom-FC and a Predict-FC
 * stack (DenseNet), joined by the dot interaction (R1).
 */
typedef struct {
  int32_t num_tables;             /* T >= 1                                                */
  const int64_t* rows;            /* [T] rows per table, each in [1, 2^31)                 */
  int32_t dim;                    /* D: multiple of 4, <= 128; == bottom_widths[n_bottom-1] */
  int32_t pooling_lo, pooling_hi; /* lookups per bag for synthetic inputs (G3); lo == hi =>
                                     fixed; lo = hi = 1 is the one-hot case     */
  const int32_t* bottom_widths;   /* [n_bottom] INCLUDING the dense input width (R3),
                                     e.g. {256,128,32}; n_bottom >= 2                       */
  int32_t n_bottom;
  const int32_t* top_widths;      /* [n_top] EXCLUDING the interaction width, last == 1 (R3),
                                     e.g. {256,64,1}; n_top >= 2; top_widths[n_top-2] <= 256 */
  int32_t n_top;
  int32_t top_shift;              /* extra 2^-top_shift on the first top layer (R21)        */
  uint64_t seed;                  /* tables, weights and synthetic inputs = f(seed) (G1-G5) */
  int32_t value_mode;             /* REC_VALUES_INT8_EXACT | REC_VALUES_FP32                */
  int32_t index_dist;             /* REC_INDEX_UNIFORM | REC_INDEX_SKEW2 | REC_INDEX_ZIPF    */
  int32_t max_batch;              /* workspace capacity in items per call/batch (>= 1)      */
  int32_t streams;                /* co-located streams m, workspaces, >= 1     */
  int32_t device;                 /* CUDA device ordinal used by this handle                */
  int32_t shard;                  /* REC_SHARD_REPLICA | REC_SHARD_TABLE | REC_SHARD_ROW    */
  int32_t rank, world;            /* this process's rank and the number of GPUs (1 => local) */
  const void* nccl_id;            /* 128-byte ncclUniqueId shared by all ranks (world > 1;
                                     sharded: required; replicas: optional, enables rec_serve's
                                     global percentiles)                                   */
  int64_t l2_persist_bytes;       /* > 0: L2 persisting window over the hot row prefix of
                                     every table (A10/D2 residue), 0 = off       */
  int32_t arch;                   /* REC_ARCH_DLRM (0) | REC_ARCH_MTWND (1), SURVEY 8(f)4:
                                     MT-WnD (Table I; R26-R29) has no bottom MLP
                                     (n_bottom = 0, no dense input), concatenates the T
                                     looked-up vectors (top input T*D) and runs n_tasks
                                     towers top_widths, each plus a wide linear part       */
  int32_t n_tasks;                /* MT-WnD task towers N in [1, 8]; DLRM: 0 or 1          */
} rec_model_desc;

#define REC_ARCH_DLRM 0
#define REC_ARCH_MTWND 1

/* Build the model: validate, allocate the fp32 table arena and the bf16 weights,
 * generate all parameters on the device from `seed` (G4/G5), encode TMA tensor maps,
 * create `streams` CUDA streams with per-stream workspaces, and (world > 1)
 * bootstrap NCCL.  Errors: INVALID_ARG (names the field), UNSUPPORTED, OOM, CUDA, NCCL. */
rec_status rec_model_create(const rec_model_desc* desc, rec_model_t* out);
void rec_model_destroy(rec_model_t m);                       /* NULL-safe; frees everything */

/* One batched query forward: the SparseNet's SparseLengthsSum over the multi-hot embedding
 * lookups ("memory-intensive sparse operations on embeddings"; "pooling" of the
 * lookups per table; "Gather-Reduce") -> the DenseNet's Bottom-FC ->
 * dot interaction (R1: P:127) -> Predict-FC -> sigmoid, with the layer widths of
 * Table I (MT-WnD: lookups -> concat -> towers + wide, ctr [B][n_tasks]
 * item-major, dense unused and may be NULL).  dense [B][F] fp32 row-major (F = bottom_widths[0]);
 * indices [nnz] int32 and offsets [T*B+1] int32 in table-major CSR (bag g = t*B + b
 * spans indices[offsets[g] .. offsets[g+1])); ctr [B] fp32 out.  Host or device
 * pointers.  Synchronous.  Errors: INVALID_ARG (batch <= 0 or > max_batch),
 * OFFSETS, INDEX_OOB (device-detected), CUDA. */
rec_status rec_query(rec_model_t m, const float* dense, const int32_t* indices,
                     const int32_t* offsets, int32_t batch, float* ctr);

/* rec_query plus diagnostics: pooled [B][T][D] fp32 (SLS output) and logits [B]
 * (pre-sigmoid), each optional (NULL).  Used by the parity tests. */
rec_status rec_query_debug(rec_model_t m, const float* dense, const int32_t* indices,
                           const int32_t* offsets, int32_t batch, float* ctr,
                           float* pooled, float* logits);

/* rec_query plus the interaction stage's operands and result, for the element-wise checks of
 * a5 (dot interaction, readings R1/R10): x [B][T+1][D] fp32 is the interaction
 * input X_b = [bottom-MLP output x_b; pooled p_b,0 .. p_b,T-1] exactly as the kernels hold it;
 * a_top [B][ld] are the bf16 bit patterns of the first top layer's A operand
 * [x_b, Z(1,0), Z(2,0), Z(2,1), ..., Z(T,T-1), 0-pad] (MT-WnD: the concatenated lookups),
 * ld = *a_top_ld = Ktop padded to a multiple of 8.  Each output optional (NULL); host or
 * device pointers.  Synchronous.  Errors: as rec_query; UNSUPPORTED for sharded models and,
 * for a_top, when the interaction is fused into the top chain (A built in shared memory). */
rec_status rec_query_inspect(rec_model_t m, const float* dense, const int32_t* indices,
                             const int32_t* offsets, int32_t batch, float* ctr, float* x,
                             uint16_t* a_top, int32_t* a_top_ld);

/* Enqueue rec_query on stream slot `slot` (0 <= slot < streams) without waiting.
 * Device or host pointers: host inputs are copied into the slot's device buffers on its
 * stream and host ctr is filled by a device-to-host copy there (pinned host memory keeps
 * the call asynchronous; the caller must not modify host inputs or read ctr before
 * rec_sync(m, slot)).  `nnz` = offsets[T*B] = the number of readable indices (host
 * indices: <= T * max_batch * pooling_hi).  Host offsets are validated before anything is
 * enqueued (OFFSETS: offsets[0] != 0, decreasing, or offsets[T*B] != nnz); device offsets
 * are validated on the device for the same conditions (the error is returned by
 * rec_sync(m, slot)) and every bag is clamped to [0, nnz), so inconsistent offsets never
 * read outside the indices.  Completion is collected by rec_sync(m, slot).
 * Table-wise sharded models (shard = REC_SHARD_TABLE, peer access between all GPUs): every
 * rank enqueues the same GLOBAL batch (all T tables' indices, all B items' dense rows) on the
 * same slot in the same order; the all-to-all of pooled vectors and the CTR all-gather run
 * inside the slot's chain over peer memory, and ctr receives all B CTRs on
 * every rank.  Every cross-GPU wait of the chain is bounded by REC_P2P_TIMEOUT_S (default
 * 60 s): a peer that never joins the batch makes rec_sync(m, slot) return REC_E_NCCL (the CTRs
 * of that batch are then undefined; the CUDA context stays usable, the model should be
 * closed).  Row-wise or NCCL-exchange sharded models: REC_E_UNSUPPORTED (use rec_query). */
rec_status rec_query_async(rec_model_t m, int32_t slot, const float* dense,
                           const int32_t* indices, const int32_t* offsets, int64_t nnz,
                           int32_t batch, float* ctr);

/* Device-synthesised batch (serving input mode REC_INPUT_DEVICE_SYNTH):
 * the batch is the concatenation of item segments segs[nseg][3] = (qid, start, len)
 * (host memory); its inputs are generated on the device (G2-G4) and the forward runs on
 * stream slot `slot`.  ctr [sum len] fp32 DEVICE pointer, or NULL (the CTRs stay in the
 * stream's workspace).  Async.  Table-wise sharded models: as rec_query_async (the same
 * global batch on the same slot on every rank; fixed pooling), REC_E_UNSUPPORTED otherwise. */
rec_status rec_synth_query_async(rec_model_t m, int32_t slot, const int32_t* segs,
                                 int32_t nseg, float* ctr);

/* Submit nbatches device-synthesised batches (as rec_synth_query_async with ctr = NULL:
 * CTRs stay in each stream's workspace), batch b = segments segs[batch_start[b] ..
 * batch_start[b+1]) on stream slot (first_slot + b) % streams — model co-location
 * round-robin without a host round trip per batch.  Async. */
rec_status rec_synth_query_batches(rec_model_t m, const int32_t* segs, const int64_t* batch_start,
                                   int64_t nbatches, int32_t first_slot);

/* S-D pipeline (SparseNet and DenseNet stages of consecutive
 * batches overlap).  lanes > 0 splits the model's `streams` workspaces into `lanes` groups
 * of N = streams / lanes (2 <= N <= 64); each lane is one captured graph that runs N batches:
 * their SLS kernels back to back on the lane stream with programmatic dependent launch,
 * each batch's dense features + bottom MLP and its interaction + top MLP on that batch's
 * own streams.  While lanes exist, rec_synth_query_batches submits groups of N batches per
 * lane launch (lanes alternate; a remainder < N uses the slot graphs).  lanes = 0 removes
 * the lanes.  Needs fixed pooling and an unsharded model (REC_E_UNSUPPORTED); streams not
 * divisible into groups of 2..64 -> REC_E_INVALID_ARG.  Synchronises the device. */
rec_status rec_set_pipeline(rec_model_t m, int32_t lanes);
/* rec_synth_query_batches through the lanes, also returning the CTRs: ctr_out (DEVICE,
 * fp32, or NULL) receives every batch's CTRs concatenated in batch order (sum of items).
 * Bit-identical to submitting the same batches with rec_synth_query_async.  Async; needs
 * rec_set_pipeline(m, > 0) first (REC_E_INVALID_ARG otherwise). */
rec_status rec_synth_query_pipeline(rec_model_t m, const int32_t* segs, const int64_t* batch_start,
                                    int64_t nbatches, float* ctr_out);

/* Wait for stream slot `slot`; returns INDEX_OOB / OFFSETS if a kernel flagged it. */
rec_status rec_sync(rec_model_t m, int32_t slot);

/* cudaStream_t of stream slot `slot` (for event timing by the caller), or NULL. */
void* rec_stream_handle(rec_model_t m, int32_t slot);

/* Test/diagnostic export: the synthetic inputs of a segment batch (G2-G4), bit-exact
 * with the oracle.  indices [T*B*pooling_hi] capacity, offsets [T*B+1], dense [B][F];
 * host or device pointers. */
rec_status rec_gen_batch(rec_model_t m, const int32_t* segs, int32_t nseg,
                         int32_t* indices, int32_t* offsets, float* dense);

/* Per-kernel device time accumulated while profiling is on (CUDA events recorded on
 * the launching stream around every launch).  kernel: 0 = SLS, 1 = GEMM (all layers),
 * 2 = interaction, 3 = input generation; kernel = 4 returns in *launches the number of
 * kernels this handle has launched so far (all streams; *total_ms = 0); kernels 5..8 return
 * host time of the synthetic submit path (5 graph-parameter updates, 6 graph launches,
 * 7 slot waits, 8 total).
 * enable != 0 turns recording on and resets the times. */
rec_status rec_profile(rec_model_t m, int32_t enable);
/* Diagnostic: time `iters` back-to-back launches of one dense stage on stream slot 0 at
 * `batch` rows (which: 0 = bottom MLP, 1 = interaction + top MLP, 2 = interaction only)
 * over whatever the workspace holds; *ms_per_iter = CUDA-event time per iteration.  Used to
 * report tensor-pipe utilisation at large batches (north_star "MLP TC util"). */
rec_status rec_bench_mlp(rec_model_t m, int32_t which, int32_t batch, int32_t iters, double* ms_per_iter);
/* Time back-to-back launches of the synthetic-index SLS kernel (a2+a3 fused) on stream
 * slot 0, one launch per batch of a batch sequence in the rec_synth_query_batches format
 * (segs[][3] = (qid, first item, items); batch k = segs[batch_start[k] .. batch_start[k+1])),
 * each batch once, so no launch re-reads rows a previous one left in L2 (distinct query ids
 * draw distinct rows).  *ms_total = CUDA-event time on the launching stream over all
 * nbatches launches.  pdl = 0: plain launches (each starts after the previous one retired;
 * launch gap, ramp and drain included); pdl = 1: programmatic dependent launch (a launch's
 * gathers overlap the previous launch's drain, its writes wait for it).  Needs fixed pooling
 * and an unsharded model (REC_E_UNSUPPORTED otherwise); writes the workspace's X only.
 * bench.py uses it for the SLS roofline line. */
rec_status rec_bench_sls(rec_model_t m, const int32_t* segs, const int64_t* batch_start,
                         int32_t nbatches, int32_t pdl, double* ms_total);
/* Time back-to-back launches of the caller-index SLS kernel (k_sls: indices and offsets
 * read from memory, rec_query / rec_query_async / e2e path) on stream slot 0: nbatches batches
 * of `batch` items, batch k's offsets at offsets + k * (T * batch + 1) and its indices at
 * indices + k * idx_stride (DEVICE pointers, table-major CSR per batch; idx_stride = readable
 * indices per batch).  *ms_total = CUDA-event time of the nbatches launches.  Writes the
 * workspace's X only.  Errors: INVALID_ARG (host pointers, sizes), UNSUPPORTED (sharded),
 * INDEX_OOB / OFFSETS (device flags of the launches). */
rec_status rec_bench_sls_caller(rec_model_t m, const int32_t* indices, const int32_t* offsets,
                                int32_t batch, int32_t nbatches, int64_t idx_stride, double* ms_total);
/* Diagnostic: %globaltimer stamps (ns) of CTA 0 of one fused-MLP launch (which: 0 bottom,
 * 1 top): [0] entry [1] TMEM+barriers ready [2] first TMA issued [3] first stage landed
 * [4+l] layer l MMAs committed [8+2l]/[9+2l] epilogue l start/end [15] exit; [14] = CUDA-event
 * time of the launch in ns.  Zero = stage not reached. */
rec_status rec_debug_chain_timeline(rec_model_t m, int32_t which, int32_t batch, int64_t* out16);
rec_status rec_profile_read(rec_model_t m, int32_t kernel, double* total_ms, int64_t* launches);

/* Locality-aware hot-row partition ("hot" embeddings placed in
 * the fastest memory, the partition sized by "memory capacity / model co-location").
 * indices / offsets [T*batch+1]: a profiling sample of queries (table-major CSR, original row
 * ids, host or device).  The library counts accesses per (table, row), orders every table's
 * rows by descending count (ties by row id), physically permutes the embedding arena so the
 * hot rows of all tables form one contiguous prefix (interleaved arena), and from then on
 * maps every index (caller or device-synthesised) to its arena row before the gather; CTRs
 * are unchanged (the same rows are summed in the same order).  A persisting L2 access-policy
 * window then covers the first window_bytes of the arena: window_bytes = 0 -> the device's
 * persisting-L2 capacity / the number of models co-located on the device, < 0 -> no window.
 * *hot_rows (optional) = rows per table inside the window.  Synchronises the device and
 * re-captures the model's graphs.  Errors: INVALID_ARG, UNSUPPORTED (sharded models, unequal
 * rows), OFFSETS, INDEX_OOB (profile index out of range), OOM, CUDA. */
rec_status rec_hot_remap(rec_model_t m, const int32_t* indices, const int32_t* offsets, int32_t batch,
                         int64_t window_bytes, int64_t* hot_rows);

/* ---------------------------------------------------------------- serving (a1, a7) */
typedef struct { double arrival_s; int32_t size; int32_t qid; } rec_trace_row;

typedef struct {
  int32_t streams;            /* m co-located streams used (<= model streams) */
  int32_t max_batch;          /* d: split chunk and fused-batch cap (<= model max_batch)  */
  double fusion_timeout_ms;   /* tau: 0 = work-conserving (R15)                           */
  int32_t input_mode;         /* REC_INPUT_DEVICE_SYNTH | REC_INPUT_HOST                  */
  int32_t clock;              /* REC_CLOCK_REAL | REC_CLOCK_VIRTUAL                       */
  double alpha_ns, beta_ns;   /* virtual clock: service = alpha + beta * items (S4)       */
  double warmup_frac;         /* fraction of the trace span excluded from percentiles     */
} rec_serve_policy;

typedef struct {
  double offered_qps, achieved_qps, mean_ms, p50_ms, p95_ms, p99_ms;
  double breakdown_ms[4];     /* mean per query: queue (arrival -> dispatch of its last
                                 sub-query), input (H2D + host packing; 0 for device-synth),
                                 sparse (SLS), dense (rest of the chain's device time) of the
                                 batch completing the query - [1..3] only while profiling is on
                                 (rec_profile(m, 1): stage-event graphs, slower); otherwise
                                 [2] = dispatch -> observed completion and [1], [3] = 0        */
  int64_t completed, dropped, batches;
  double mean_batch;
  int32_t sla_met;            /* p95 <= SLA, all completed, achieved >= 0.98 offered (R23) */
  int32_t stable;
  int32_t ranks;              /* ranks the percentiles cover: 1, or world for replica models
                                 created with world > 1 and an nccl_id (every rank serves its
                                 share of the trace, e.g. q mod G; latencies are all-gathered
                                 (C4) so every rank reports the GLOBAL mean / p50 / p95 / p99,
                                 stable = all ranks stable, offered / achieved = sums)        */
} rec_serve_report;

/* Query splitting + fusion (S1, S2) for queries that are all pending
 * (a burst, FIFO in trace order): split each query into chunks of max_batch items
 * (remainder last), then fuse FIFO chunks into batches with cumulative size <= max_batch
 * (at least one chunk each).  Host-only (no device needed).
 * segs_out [seg_cap][3] = (qid, start, len); batch_start [bcap+1]: batch b spans
 * segs_out[batch_start[b] .. batch_start[b+1]).  *nbatches, *nsegs are set.
 * Errors: INVALID_ARG (max_batch < 1, size < 1, capacity too small). */
rec_status rec_split_fuse(const rec_trace_row* trace, int64_t n, int32_t max_batch,
                          int32_t* segs_out, int64_t seg_cap, int64_t* batch_start,
                          int64_t bcap, int64_t* nbatches, int64_t* nsegs);

/* The deterministic global dispatcher of sharded serving (R31; host-only): split
 * every query into sub-queries of <= max_batch items (S1), then cut the FIFO into batches of
 * whole sub-queries with cumulative size <= max_batch; a batch closes when it is full (the
 * next sub-query does not fit, or it holds exactly max_batch items: close = that arrival) or
 * tau_ms after its first sub-query arrived, whichever comes first; close times are made
 * non-decreasing.  Output as rec_split_fuse plus close_s[b] (trace time, seconds).
 * Errors: INVALID_ARG (tau_ms <= 0, bad trace, capacity). */
rec_status rec_global_batches(const rec_trace_row* trace, int64_t n, int32_t max_batch, double tau_ms,
                              int32_t* segs_out, int64_t seg_cap, int64_t* batch_start, double* close_s,
                              int64_t bcap, int64_t* nbatches, int64_t* nsegs);

/* Serve a query trace (rows sorted by arrival_s, qid unique) on this GPU under the
 * policy: split each query into chunks of d (S1), fuse FIFO chunks with
 * cumulative size <= d (S2) onto the lowest idle of m streams (S3), run the
 * forward per batch, timestamp completions, and report latency percentiles against
 * `sla_ms` (S5).  Real clock: arrivals are released open-loop at
 * arrival_s; the batch list depends on timing (invariants only).  Virtual clock:
 * the dispatcher advances a simulated clock (S4) and the batch list is unique and
 * bit-exact with the oracle replay; the kernels still run.
 * latency_ms [n] (optional, per trace row) and batch_log (optional, flattened rows
 * (batch, stream, qid, start, len), capacity log_cap rows; the number of rows written
 * is returned in report->batches' companion, see rec_serve_log_rows).
 * ctr_out [sum sizes][n_tasks] (optional, host): CTR(s) of every item, query-major in
 * trace order.  Errors: INVALID_ARG (bad policy, before any work), CUDA.
 * Table-wise sharded models (every rank calls rec_serve with the same trace): batches are cut
 * by a deterministic global dispatcher from the trace alone (R31: a batch closes
 * when full or tau = fusion_timeout_ms (default SLA / 50) after its first sub-query arrived;
 * batch k on slot k mod m), so every rank runs the same batches; ranks align their clocks
 * with an NCCL barrier; real clock and REC_INPUT_DEVICE_SYNTH only (else UNSUPPORTED). */
rec_status rec_serve(rec_model_t m, const rec_trace_row* trace, int64_t n, double sla_ms,
                     const rec_serve_policy* pol, rec_serve_report* out,
                     double* latency_ms, int32_t* batch_log, int64_t log_cap,
                     int64_t* log_rows, float* ctr_out);

/* Shard plan of a rank (host-only): out[6] = {first local table, local table
 * count, first local row, end local row (row-wise; else 0 / INT32_MAX), first item of this
 * rank's block, items in the block} for a global batch of `batch` items (contiguous blocks
 * of ceil(batch / world), reading R22).  Errors: INVALID_ARG, UNSUPPORTED (table-wise needs
 * num_tables % world == 0, row-wise needs equal rows). */
rec_status rec_shard_plan(int32_t num_tables, const int64_t* rows, int32_t world, int32_t rank,
                          int32_t shard, int32_t batch, int64_t* out);

/* --------------------------------------------------------------------- utilities */
const char* rec_last_error(void);             /* thread-local; valid until the next call */
int32_t rec_nccl_unique_id_size(void);        /* bytes of an ncclUniqueId (128)          */
rec_status rec_nccl_get_unique_id(void* out); /* rank 0 creates, caller broadcasts       */
int32_t rec_version(void);

#ifdef __cplusplus
}
#endif

#endif /* HERCULES_REC_H */
