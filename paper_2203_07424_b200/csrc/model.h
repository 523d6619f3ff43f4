// model.h — internal host-side model state behind the C ABI (include/rec.h).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/rec.h"
#include "kernels.h"

namespace rec {

void set_error(const char* fmt, ...);
rec_status cuda_fail(cudaError_t e, const char* what);

#define REC_CUDA(call)                                   \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) return cuda_fail(_e, #call);  \
  } while (0)

struct Layer {
  int K = 0, Kpad = 0, N = 0, Npad = 0, bn = 0;  // true fan-in, padded fan-in, fan-out
  int layer_id = 0, exp = 0;
  __nv_bfloat16* W = nullptr;                    // [N][Kpad] bf16
  float* bias = nullptr;                         // [N]
  CUtensorMap tmap_w;
  CUtensorMap tmap_w128;                         // box rows min(bn, 128) (fused MLP, 128-row chunks)
  CUtensorMap tmap_w64;                          // box rows min(bn, 64) (64-wide serving tiles)
};

// A staging slot of device-synthesised batches: the batch descriptor (kernel parameters of
// the chain's first kernel) and the CUDA graph of the whole a2-a6 chain.  Several slots per
// stream let the host run ahead of the GPU while profiling events stay per launch.
struct SynthSlot {
  SegBatch* sb = nullptr;            // host copy of the first kernel's by-value parameter
  SegBatch* sb_local = nullptr;      // sharded: this rank's item block of the batch (dense part)
  GenArgs ga{};
  SlsSynthArgs sa{};
  cudaEvent_t free = nullptr;        // the last launch that used this slot completed
  struct Variant {                   // [0] kernels only (production), [1] + stage events
    cudaGraph_t graph = nullptr;     // kept alive: the node handles belong to it
    cudaGraphExec_t exec = nullptr;
    cudaGraphNode_t gen_node = nullptr;    // first kernel of the main stream (SLS or inputs)
    cudaGraphNode_t dense_node = nullptr;  // fused path: dense-feature kernel on the branch
  } var[2];
  cudaGraphNode_t* cap_gen = nullptr;  // capture target for the node handles
  cudaGraphNode_t* cap_dense = nullptr;
  cudaEvent_t ev[8] = {};            // stage boundaries inside the graph (timing)
  bool prof_pending = false;
};

// One per co-located stream: the buffers a batch needs on that stream.
struct Workspace {
  cudaStream_t stream = nullptr;
  cudaStream_t stream_b = nullptr;   // parallel branch: bottom MLP runs concurrently with SLS
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaStream_t stream_c = nullptr;   // pipeline lanes: interaction + top of this workspace's batch
  cudaEvent_t ev_sls = nullptr, ev_done = nullptr;  // pipeline capture edges
  cudaEvent_t ev_g1 = nullptr, ev_g2 = nullptr;     // SM-partition (green context) edges
  int* dB = nullptr;                 // device batch size of the in-flight synthetic batch
  int4* gsegs = nullptr;             // device segments for batches with > kParamSegs segments
  int cap = 0;                       // max items
  int64_t idx_cap = 0;               // max indices
  int* indices = nullptr;            // [idx_cap]
  int* offsets = nullptr;            // [T*cap+1]
  int4* segs = nullptr;              // [cap] device segment list
  int* rowq = nullptr;               // [cap]
  int* rowi = nullptr;               // [cap]
  float* dense_f32 = nullptr;        // [cap][F] (caller dense staging / gen output)
  __nv_bfloat16* dense_bf = nullptr; // [cap][Fpad]
  float* X = nullptr;                // [cap][T+1][D]
  __nv_bfloat16* A_top = nullptr;    // [cap][Ktop_pad]
  __nv_bfloat16* h[2] = {nullptr, nullptr};  // hidden ping-pong [cap][hmax]
  float* ctr = nullptr;              // [cap][n_tasks]
  float* logit = nullptr;            // [cap][n_tasks]
  float* wide = nullptr;             // MT-WnD: [cap][n_tasks] wide-part logits
  std::vector<__nv_bfloat16*> th;    // MT-WnD: hidden ping-pong of towers 1..N-1 (2 per task)
  std::vector<std::vector<CUtensorMap>> tmap_a_task;  // [task][layer] A maps (task >= 1)
  std::vector<std::vector<void*>> out_task;           // [task][layer] hidden outputs
  int* flag = nullptr;               // device error flags (bit0 OOB, bit1 offsets)
  int* flag_host = nullptr;          // pinned mirror
  uint8_t* pin = nullptr;            // pinned staging
  size_t pin_bytes = 0;
  cudaEvent_t pin_free = nullptr;    // last H2D out of `pin` completed
  std::vector<CUtensorMap> tmap_a_bottom, tmap_a_top;  // A operand per GEMM layer
  std::vector<void*> out_bottom, out_top;              // output buffer per GEMM layer
  ChainMaps chain_bottom{}, chain_top{};                // fused-MLP tensor maps (k_mlp.cu)
  std::vector<SynthSlot> slots;                        // synthetic-batch staging ring
  int next_slot = 0;
  int graph_kernels = 0;                               // kernels per graph launch
  double host_ns[4] = {0, 0, 0, 0};  // host time in synth_submit (param update, graph launch,
                                     // slot wait, total) — per stream: dispatch threads
  // table-wise sharded slot exchange (dist.cu p2p_slots_init): this workspace's X lives in the
  // model's IPC-exported exchange arena (x_external: not freed separately); the P2P argument
  // sets of its chain (SLS stores + flags, flag wait, CTR all-gather, CTR-flag wait), the
  // gathered CTRs of the whole batch, and the slot's epoch counter
  int last_slot = -1;                // staging slot of the last synth_submit (its stage events)
  bool x_external = false;
  P2PArgs sh_sls{}, sh_wait{}, sh_ctr{}, sh_ctrwait{};
  float* sh_ctr_gather = nullptr;    // [G * Bq] CTRs of every rank's block (items 0..B-1)
  uint4* sh_ll = nullptr;  // this slot's LL receive buffer (flag-in-data exchange; inside sh_arena)
  unsigned sh_epoch = 0;
  int4* gsegs_local = nullptr;       // device segments of this rank's item block (> kParamSegs)
};

// S-D pipeline lane: one captured graph over N workspaces that
// runs N batches with the SparseNet and DenseNet stages decoupled — all N SLS kernels on one
// stream as a programmatic-dependent-launch chain (each launch's gathers overlap the previous
// one's drain), every batch's dense features + bottom MLP on its workspace's branch stream,
// and its interaction + top MLP on a third stream once both halves are done.
struct PipeLane {
  std::vector<int> ws;               // workspace of batch i (ws[0]'s stream launches the graph)
  std::vector<SegBatch*> sb;         // host copies of the by-value batch descriptors
  std::vector<GenArgs> ga;
  std::vector<SlsSynthArgs> sa;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  std::vector<cudaGraphNode_t> sls_node, dense_node;
  cudaEvent_t free = nullptr;        // the lane's last graph launch completed
  int kernels = 0;                   // kernels per launch
};

struct ProfEvent {
  int kernel;
  cudaEvent_t a, b;
};

}  // namespace rec

struct rec_model_s {
  // description
  int T = 0, D = 0, F = 0, Fpad = 0, lo = 0, hi = 0;
  std::vector<int64_t> rows;
  std::vector<int> bottom_w, top_w;
  int top_shift = 0, value_mode = 0, index_dist = 0, max_batch = 0, nstreams = 0, device = 0;
  int shard = 0, rank = 0, world = 1;
  uint64_t seed = 0;
  uint32_t k0 = 0, k1 = 0;
  int emb_shift = 0;
  int64_t l2_persist_bytes = 0;
  // hot-row partition (rec_hot_remap): old row -> arena row per
  // table (concatenated, offsets remap_off), the L2 persisting window it set (bytes, 0 = none)
  int* d_remap = nullptr;
  int64_t* d_remap_off = nullptr;
  int64_t hot_window = 0;
  bool counted = false;                // counted in the per-device co-located model registry
  bool stage_events = false;           // rec_serve breakdown: graphs with stage events, read by
                                       // the server (not accumulated into the profile counters)
  // embedding arena
  float* tables = nullptr;
  size_t table_bytes = 0;
  bool interleaved = false;
  int64_t row_stride = 0;              // floats between consecutive rows of one table
  std::vector<int64_t> tab_off;        // floats, start of row 0 of table t
  int64_t* d_tab_off = nullptr;
  int64_t* d_rows = nullptr;
  // TMA row-gather map over the arena (device copy) for the synthetic-index SLS
  CUtensorMap* d_tmap_rows = nullptr;
  int sls_tma = 0, nsm = 0;
  int sls_pdl = 1;    // REC_PDL=0 disables programmatic dependent launch of the SLS
  int sls_interleave = 0;  // REC_SLS_GRID=1: bags round-robin over one wave (k_sls_synth;
                           // measured: RMC1 304k vs 326k QPS, serialized 0.56 either way)
  int fuse_dense = 0;  // REC_FUSE_DENSE=1: dense features generated inside the SLS kernel
  int chain_pdl = 1;    // top fused MLP launched with PDL after the interaction (REC_CHAIN_PDL)
  int green_sms = 0;    // SMs reserved for the dense stages (REC_GREEN_SMS; 0 = shared SMs)
  void* green[2] = {nullptr, nullptr};  // CUgreenCtx: [0] dense partition, [1] SLS partition
  void* green_cu[2] = {nullptr, nullptr};  // their CUcontext handles (graph node updates)
  int fuse_interact = 0; // dot interaction inside the top chain (REC_FUSE_INTERACT=1; measured -0.4 %)
  int tower_group = 1;  // MT-WnD: one grouped launch per tower layer (REC_TOWER_GROUP=0: per task)  // dense features generated by the SLS kernel (REC_FUSE_DENSE)
  int diag_skip = 0;  // REC_STEP_DIAG (diagnostic): stages dropped from the synthetic step
  // MLP
  std::vector<rec::Layer> bottom, top;  // top excludes the width-1 output layer
  float* w_last = nullptr;
  float b_last = 0.f;
  // MT-WnD (arch 1): towers of tasks 1..N-1 (task 0 = `top`), their output layers, and the
  // wide vectors of all tasks [N][Ktop]
  int arch = 0, tasks = 1;
  std::vector<std::vector<rec::Layer>> towers;
  std::vector<float*> w_last_t;
  std::vector<float> b_last_t;
  float* wide_v = nullptr;
  // fused FC stacks (one kernel per MLP per 128-row tile) when they fit
  bool chain_bottom = false, chain_top = false;
  rec::ChainArgs chain_bottom_args{}, chain_top_args{};
  float* bias_bottom_all = nullptr;
  float* bias_top_all = nullptr;
  int Ktop = 0, Ktop_pad = 0, hmax = 0;
  // streams + workspaces
  std::vector<rec::Workspace> ws;
  // S-D pipeline lanes (rec_set_pipeline); pipe_active: the last synthetic submission used
  // the lanes (switching modes synchronises, workspaces are shared)
  std::vector<rec::PipeLane> pipe;
  std::atomic<int> pipe_active{0};
  int pipe_next = 0;
  // profiling
  bool prof = false;
  std::vector<rec::ProfEvent> prof_events;
  std::vector<cudaEvent_t> prof_pool;
  double prof_ms[4] = {0, 0, 0, 0};
  int64_t prof_n[4] = {0, 0, 0, 0};
  std::atomic<int64_t> launches{0};    // kernels launched by this handle (all streams)
  // distributed (sharded modes)
  void* nccl_comm = nullptr;
  int t0 = 0, T_loc = 0;               // local tables [t0, t0 + T_loc)
  int64_t row_lo = 0, row_hi = 0x7fffffff;  // local rows of every table (row-wise sharding)
  float* sh_send = nullptr;            // [B_pad][T_loc][D] (table) or [B_pad][T][D] (row)
  float* sh_recv = nullptr;            // [world][Bq][T_loc][D] (table) or [Bq][T][D] (row)
  float* sh_ctr = nullptr;             // [world * Bq]
  // table-wise sharding with the all-to-all fused into the SLS (peer stores over NVLink)
  bool p2p = false;
  float** d_peer_X = nullptr;          // [world] device array of every rank's ws[0].X
  unsigned** d_peer_flags = nullptr;   // [world] device array of every rank's arrival flags
  unsigned* p2p_flags = nullptr;       // this rank's arrival flags [world]
  float** d_peer_ctr = nullptr;        // [world] device array of every rank's sh_ctr
  unsigned** d_peer_ctr_flags = nullptr;
  unsigned* p2p_ctr_flags = nullptr;   // this rank's CTR-gather flags [world]
  unsigned* p2p_counter = nullptr;     // CTA counter of the fused SLS launch
  float* p2p_stage = nullptr;          // row-wise: partial sums of every source rank [G][Bq][T][D]
  unsigned p2p_epoch = 0;
  std::vector<void*> p2p_opened;       // IPC mappings to close
  // table-wise sharding, asynchronous slot exchange (dist.cu): one IPC-exported arena of
  // `nstreams` slots [X | CTR gather | arrival flags | CTR flags | CTA counter | words]
  bool p2p_slots = false;
  uint8_t* sh_arena = nullptr;
  size_t sh_slot_bytes = 0;
  void** d_sh_ptrs = nullptr;          // per slot: peer X / flags / CTR / CTR flags [4][G]
};

namespace rec {
struct ShardPlan {
  int t0, t_local;           // global index of the first local table, local table count
  int64_t row_lo, row_hi;    // rows of every table held here (row-wise), else [0, INT32_MAX)
};
rec_status shard_plan(int T, const int64_t* rows, int world, int rank, int shard, ShardPlan* p);
// Launch the forward of `batch` items on workspace `w` whose inputs are already in
// w.indices / w.offsets / w.dense_bf (or caller device pointers).  ctr_out: device.
rec_status forward_enqueue(rec_model_s* m, Workspace& w, const int* indices, const int* offsets,
                           int batch, const int* dB, float* ctr_out, float* logit_out,
                           cudaEvent_t* gev,    // gev: 8 stage events (graph capture) or null
                           int64_t idx_limit = 0x7fffffff);  // readable indices (SLS clamp)
// Device-synthesised batch (segment list on the host) through a staging slot: inputs (a2)
// and forward (a3-a6) enqueued on w.stream, CTRs in w.ctr.
rec_status synth_submit(rec_model_s* m, Workspace& w, const int32_t* segs, int nseg, int* batch_out,
                        float* dense_f32_out);
rec_status capture_graphs(rec_model_s* m, Workspace& w);
void fill_genargs(rec_model_s* m, Workspace& w, GenArgs& ga, SlsSynthArgs& sa, float* dense_f32_out);
const cudaGraphNode_t* last_node(cudaStream_t s, size_t* n);
// Leave pipeline mode (wait for every lane) before a non-pipeline submission.
rec_status pipe_leave(rec_model_s* m);
void pipe_destroy(rec_model_s* m);
// Submit nbatches synthetic batches through the lanes (groups of N = batches per lane); a
// remainder < N goes through the per-stream slot graphs.  ctr_out (device, optional): the
// CTRs of all batches, concatenated in batch order.
rec_status pipe_submit(rec_model_s* m, const int32_t* segs, const int64_t* batch_start,
                       int64_t nbatches, float* ctr_out);
void enqueue_bottom(rec_model_s* m, Workspace& w, cudaStream_t st, int B, const int* dB,
                    cudaEvent_t* gev);
void enqueue_interact_top(rec_model_s* m, Workspace& w, cudaStream_t st, int B, const int* dB,
                          float* ctr_out, float* logit_out, cudaEvent_t* gev);
// Model-parallel forward of a global batch (inputs staged on the device, identical on every
// rank): local SLS -> all-to-all (table-wise) / reduce-scatter (row-wise) -> dense part on this
// rank's item block -> all-gather of the CTRs into ctr (host or device) on every rank.
rec_status sharded_forward(rec_model_s* m, Workspace& w, const float* d_dense, const int* d_idx,
                           const int* d_off, int B, float* ctr, float* logits);
rec_status sharded_alloc(rec_model_s* m);
// All ranks' values (variable counts) on every rank through the model's communicator (C4).
rec_status allgather_doubles(rec_model_s* m, const std::vector<double>& mine, std::vector<double>& all);
// Table-wise sharding over peer memory, asynchronous (dist.cu): the chain of one global batch
// on workspace w.  Caller mode (segs == nullptr): inputs already on the device (global dense /
// indices / offsets); synthetic mode: the slot's SegBatch descriptors (captured graph).
rec_status shard_enqueue(rec_model_s* m, Workspace& w, const float* d_dense, const int* d_idx,
                         const int* d_off, int B, int64_t idx_limit);
rec_status shard_capture(rec_model_s* m, Workspace& w);
// Host side of a synthetic sharded batch: sl.sb_local = this rank's item block of the global
// batch given as host segments; returns the block size.
int shard_fill_local(rec_model_s* m, Workspace& w, SynthSlot& sl, const int32_t* segs, int nseg,
                     int B, int4* stage);
rec_status p2p_slots_init(rec_model_s* m);
cudaEvent_t prof_begin(rec_model_s* m, cudaStream_t s);
rec_status dist_init(rec_model_s* m, const void* nccl_id);   // dist.cu
rec_status p2p_init(rec_model_s* m);                          // dist.cu (fused table-wise exchange)
void dist_destroy(rec_model_s* m);
void prof_end(rec_model_s* m, cudaStream_t s, int kernel, cudaEvent_t a);
}  // namespace rec
