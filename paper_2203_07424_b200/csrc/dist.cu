// dist.cu — multi-GPU embedding sharding.
//
// One process per GPU; the ncclUniqueId is created by rank 0 (rec_nccl_get_unique_id) and
// broadcast by the caller (torch.distributed is bootstrap plumbing only).
//
// Table-wise (REC_SHARD_TABLE, e.g. RMC2: 40 tables = 8 x 5): rank r holds tables
// [r*T/G, (r+1)*T/G) and pools them for ALL B items straight into an all-to-all send buffer
// laid out [B_pad][T/G][D] — item b's block of rows belongs to the rank that owns item b
// (contiguous item blocks of Bq = ceil(B/G), reading R22), so no repacking is needed.  One
// ncclAlltoAll (C1) delivers to every rank the pooled vectors of its items for every table;
// the rank runs the bottom MLP, interaction and top MLP for its Bq items, and an
// ncclAllGather (C3) returns every CTR to every rank.  Each bag is pooled by the same kernel
// in the same order and the GEMMs are batch-invariant, so results are bit-identical to
// replicas.
// Row-wise (REC_SHARD_ROW, 10-table configs where 10 % 8 != 0): rank r holds rows
// [r*R/G, (r+1)*R/G) of every table; every rank pools its rows of every bag (partial sums,
// [B_pad][T][D]); one ncclReduceScatter (C2, sum) leaves each rank the full pooled vectors
// of its Bq items.  The cross-rank sum changes the fp32 association: bit-exact in int8-exact
// value mode (G4), within the SLS tolerance otherwise.
#include <nccl.h>

#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <vector>

#include "model.h"

namespace rec {

#define REC_NCCL(call)                                                          \
  do {                                                                          \
    ncclResult_t _r = (call);                                                   \
    if (_r != ncclSuccess) {                                                    \
      set_error("NCCL error %s in %s", ncclGetErrorString(_r), #call);          \
      return REC_E_NCCL;                                                        \
    }                                                                           \
  } while (0)

rec_status dist_init(rec_model_s* m, const void* nccl_id) {
  if (!nccl_id) {
    set_error("nccl_id must be non-null when world > 1 and shard != REPLICA");
    return REC_E_INVALID_ARG;
  }
  ncclUniqueId id;
  memcpy(&id, nccl_id, sizeof(id));
  ncclComm_t comm = nullptr;
  REC_NCCL(ncclCommInitRank(&comm, m->world, id, m->rank));
  m->nccl_comm = comm;
  if (m->shard == REC_SHARD_REPLICA) return REC_OK;  // serving percentiles only
  rec_status st = sharded_alloc(m);
  if (st != REC_OK) return st;
  return p2p_init(m);
}

// ---------------------------------------------------------------------------------------------
// Table-wise sharding, asynchronous slot exchange.
//
// Every co-located stream slot s of every rank owns a region of one exchange arena (a single
// cudaMalloc per rank, exported once with CUDA IPC):
//   [X: cap x (T+1) x D fp32 | CTR gather: G x Bq fp32 | arrival flags [G] | CTR flags [G] |
//    CTA counter | words: epoch, B | LL lines: Bq x T x D/4 x 2 x 16 B]
// The k-th batch submitted on slot s is the same global batch on every rank (a deterministic
// global dispatch: every rank submits the same batch sequence round-robin over the slots) and
// carries epoch k + 1 on that slot.  Its chain on rank r:
//   SLS of the local tables for all B items; the pooled vector of a remote item (blocks of
//     Bq = ceil(B / G)) goes over NVLink as two flag-in-data LL lines {v, epoch, v, epoch}
//     into LL_s of its owner, an own item's straight into the local X_s; the last CTA raises
//     flags_s[r] = epoch on every rank (st.release.sys, a hint)          -- fused all-to-all C1
//     (caller-index chains, REC_P2P_LL=0: every vector into the owner's X_s behind a per-CTA
//     system-scope fence, and the flag is the guarantee)
//   || dense features + bottom MLP of the own block (branch stream)
//   wait flags_s[0..G) >= epoch -> LL unpack (each line's epoch checked) into X_s ->
//   interaction + top MLP of the own block
//   CTRs of the own block stored into CTR_s of every rank, CTR flags raised  -- all-gather C3
//   wait CTR flags_s[0..G) >= epoch
// Reuse of X_s / LL_s by batch k + m is safe: rank r issues it only after its CTR-flag wait of
// batch k, and every rank raised its CTR flag of k after its interaction had read X_s.  Slots are
// independent, so m batches are in flight per rank with no host synchronisation.
static size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

struct SlotLayout {
  size_t x, ctr, flags, ctrflags, counter, words, ll, bytes;
};
static SlotLayout slot_layout(const rec_model_s* m) {
  const int G = m->world;
  const int64_t Bq = (m->max_batch + G - 1) / G;
  SlotLayout L{};
  L.x = 0;
  L.ctr = al256(static_cast<size_t>(m->max_batch) * (m->T + 1) * m->D * sizeof(float));
  L.flags = L.ctr + al256(sizeof(float) * G * Bq);
  L.ctrflags = L.flags + al256(sizeof(unsigned) * G);
  L.counter = L.ctrflags + al256(sizeof(unsigned) * G);
  L.words = L.counter + 256;
  L.ll = L.words + 256;  // LL receive lines: [Bq][T][D / 4][2] x 16 B
  L.bytes = L.ll + al256(static_cast<size_t>(Bq) * m->T * (m->D / 4) * 2 * sizeof(uint4));
  return L;
}

static unsigned long long p2p_timeout_ns();

rec_status p2p_slots_init(rec_model_s* m) {
  const int G = m->world, M = m->nstreams;
  const SlotLayout L = slot_layout(m);
  m->sh_slot_bytes = L.bytes;
  REC_CUDA(cudaMalloc(reinterpret_cast<void**>(&m->sh_arena), L.bytes * M));
  REC_CUDA(cudaMemset(m->sh_arena, 0, L.bytes * M));
  cudaIpcMemHandle_t mine;
  REC_CUDA(cudaIpcGetMemHandle(&mine, m->sh_arena));
  uint8_t* dh = nullptr;
  REC_CUDA(cudaMalloc(reinterpret_cast<void**>(&dh), sizeof(mine) * (G + 1)));
  REC_CUDA(cudaMemcpy(dh + sizeof(mine) * G, &mine, sizeof(mine), cudaMemcpyHostToDevice));
  REC_NCCL(ncclAllGather(dh + sizeof(mine) * G, dh, sizeof(mine), ncclUint8,
                         static_cast<ncclComm_t>(m->nccl_comm), m->ws[0].stream));
  REC_CUDA(cudaStreamSynchronize(m->ws[0].stream));
  std::vector<cudaIpcMemHandle_t> all(G);
  REC_CUDA(cudaMemcpy(all.data(), dh, sizeof(mine) * G, cudaMemcpyDeviceToHost));
  cudaFree(dh);
  std::vector<uint8_t*> base(G);
  for (int q = 0; q < G; ++q) {
    if (q == m->rank) {
      base[q] = m->sh_arena;
      continue;
    }
    void* a = nullptr;
    REC_CUDA(cudaIpcOpenMemHandle(&a, all[q], cudaIpcMemLazyEnablePeerAccess));
    m->p2p_opened.push_back(a);
    base[q] = static_cast<uint8_t*>(a);
  }
  // per slot: [peer X][peer flags][peer CTR][peer CTR flags][peer LL], G pointers each
  std::vector<void*> ptrs(static_cast<size_t>(M) * 5 * G);
  for (int s = 0; s < M; ++s)
    for (int q = 0; q < G; ++q) {
      uint8_t* b = base[q] + L.bytes * s;
      ptrs[(s * 5 + 0) * G + q] = b + L.x;
      ptrs[(s * 5 + 1) * G + q] = b + L.flags;
      ptrs[(s * 5 + 2) * G + q] = b + L.ctr;
      ptrs[(s * 5 + 3) * G + q] = b + L.ctrflags;
      ptrs[(s * 5 + 4) * G + q] = b + L.ll;
    }
  REC_CUDA(cudaMalloc(reinterpret_cast<void**>(&m->d_sh_ptrs), sizeof(void*) * ptrs.size()));
  REC_CUDA(cudaMemcpy(m->d_sh_ptrs, ptrs.data(), sizeof(void*) * ptrs.size(), cudaMemcpyHostToDevice));
  for (int s = 0; s < M; ++s) {
    Workspace& w = m->ws[s];
    uint8_t* mb = m->sh_arena + L.bytes * s;
    if (!w.x_external) cudaFree(w.X);
    w.X = reinterpret_cast<float*>(mb + L.x);
    w.x_external = true;
    w.sh_ctr_gather = reinterpret_cast<float*>(mb + L.ctr);
    void** P = m->d_sh_ptrs + static_cast<size_t>(s) * 5 * G;
    w.sh_ll = reinterpret_cast<uint4*>(mb + L.ll);
    unsigned* words = reinterpret_cast<unsigned*>(mb + L.words);
    P2PArgs a{};
    a.G = G;
    a.rank = m->rank;
    a.words = words;
    a.err_flag = w.flag;
    a.timeout_ns = p2p_timeout_ns();
    {
      // fenced protocol (caller-index chains, or REC_P2P_LL=0): fence.sc.sys per CTA (default)
      // or one acq_rel.sys atomic (REC_P2P_FENCE=0): measured equal (44.8k vs 44.7k QPS, RMC2
      // on 2 GPUs), so the plainly correct fence stays
      const char* f = getenv("REC_P2P_FENCE");
      a.sc_fence = f ? atoi(f) : 1;
    }
    w.sh_sls = a;
    w.sh_sls.peer_X = reinterpret_cast<float* const*>(P);
    w.sh_sls.peer_flags = reinterpret_cast<unsigned* const*>(P + G);
    w.sh_sls.counter = reinterpret_cast<unsigned*>(mb + L.counter);
    w.sh_sls.peer_ll = reinterpret_cast<uint4* const*>(P + 4 * G);
    w.sh_sls.T_all = m->T;
    {
      // flag-in-data lines for remote items (captured synthetic chains); REC_P2P_LL=0: the
      // pooled vectors go straight into the owner's X behind a per-CTA system-scope fence
      const char* e = getenv("REC_P2P_LL");
      w.sh_sls.ll = (e ? atoi(e) : 1) != 0 && m->D % 4 == 0;
    }
    w.sh_wait = a;
    w.sh_wait.my_flags = reinterpret_cast<unsigned*>(mb + L.flags);
    w.sh_ctr = a;
    w.sh_ctr.peer_X = reinterpret_cast<float* const*>(P + 2 * G);
    w.sh_ctr.peer_flags = reinterpret_cast<unsigned* const*>(P + 3 * G);
    w.sh_ctrwait = a;
    w.sh_ctrwait.my_flags = reinterpret_cast<unsigned*>(mb + L.ctrflags);
    if (!w.gsegs_local)
      REC_CUDA(cudaMalloc(reinterpret_cast<void**>(&w.gsegs_local), sizeof(int4) * (w.cap + 1)));
  }
  // every rank's arena is zeroed before any peer may write into it
  int* f = nullptr;
  REC_CUDA(cudaMalloc(reinterpret_cast<void**>(&f), sizeof(int)));
  REC_CUDA(cudaMemsetAsync(f, 0, sizeof(int), m->ws[0].stream));
  REC_NCCL(ncclAllReduce(f, f, 1, ncclInt32, ncclSum, static_cast<ncclComm_t>(m->nccl_comm), m->ws[0].stream));
  REC_CUDA(cudaStreamSynchronize(m->ws[0].stream));
  cudaFree(f);
  m->p2p_slots = true;
  m->p2p = true;
  if (getenv("REC_VERBOSE"))
    fprintf(stderr, "[rec] rank %d: fused all-to-all over peer memory, %d async slots (%d ranks)\n",
            m->rank, M, G);
  return REC_OK;
}

// Dense part of this rank's item block + the exchange waits + the CTR all-gather, on w.stream
// after the SLS (and on w.stream_b for the bottom branch, forked by the caller).  epoch == 0:
// the kernels read epoch / B from the slot words (captured graphs); else by value.
static rec_status shard_tail(rec_model_s* m, Workspace& w, int B, const int* dB, cudaEvent_t join,
                             unsigned epoch = 0, int Bl = 0, int item0 = 0) {
  cudaStream_t s = w.stream;
  P2PArgs wa = w.sh_wait, ca = w.sh_ctr, cw = w.sh_ctrwait;
  if (epoch) {
    wa.words = ca.words = cw.words = nullptr;
    wa.epoch = ca.epoch = cw.epoch = epoch;
  }
  launch_p2p_wait(wa, s);
  if (!epoch && w.sh_sls.ll) {  // captured chains: remote tables' vectors from the LL lines
    launch_p2p_ll_unpack(wa, w.sh_ll, w.X, m->T, m->D, m->t0, m->T_loc, m->nsm, s);
    m->launches += 1;
  }
  REC_CUDA(cudaStreamWaitEvent(s, join, 0));
  enqueue_interact_top(m, w, s, B, dB, w.ctr, w.logit, nullptr);
  launch_p2p_ctr_scatter(w.ctr, Bl, item0, ca, s);
  launch_p2p_wait(cw, s);
  m->launches += 3;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "sharded chain launch");
  return REC_OK;
}

// Caller mode: global dense [B][F], indices / offsets of all T tables (table-major CSR) on the
// device.  Direct launches, epoch and batch passed by value.
rec_status shard_enqueue(rec_model_s* m, Workspace& w, const float* d_dense, const int* d_idx,
                         const int* d_off, int B, int64_t idx_limit) {
  const int G = m->world, r = m->rank, TL = m->T_loc, D = m->D, T = m->T;
  const int Bq = (B + G - 1) / G, item0 = r * Bq;
  const int Bl = std::max(0, std::min(Bq, B - item0));
  cudaStream_t s = w.stream, sb = w.stream_b;
  const unsigned epoch = ++w.sh_epoch;
  REC_CUDA(cudaEventRecord(w.ev_fork, s));
  REC_CUDA(cudaStreamWaitEvent(sb, w.ev_fork, 0));
  if (Bl > 0) {
    launch_dense_to_bf16(d_dense + static_cast<size_t>(item0) * m->F, Bl, m->F, m->Fpad, w.dense_bf, sb);
    m->launches += 1;
    enqueue_bottom(m, w, sb, Bl, nullptr, nullptr);
  }
  REC_CUDA(cudaEventRecord(w.ev_join, sb));
  P2PArgs pa = w.sh_sls;
  pa.ll = 0;  // (the caller-index kernel stores into X behind the fence protocol)
  pa.words = nullptr;
  pa.epoch = epoch;
  pa.Bq = Bq;
  pa.row_off = 0;
  launch_sls_p2p(m->tables, m->d_tab_off, m->row_stride, m->d_rows, d_idx, d_off + m->t0 * B, B, TL, D,
                 (T + 1) * D, 1 + m->t0, w.flag, pa, s, 0, 0x7fffffff,
                 static_cast<int>(std::min<int64_t>(idx_limit, 0x7fffffff)));
  m->launches += 1;
  return shard_tail(m, w, Bl, nullptr, w.ev_join, epoch, Bl, item0);
}

// Synthetic mode, captured once per staging slot: SLS over device-synthesised indices of the
// local tables (global batch sl.sb) || dense features of the own block (sl.sb_local) -> bottom;
// then shard_tail.  Both first kernels take their batch by value (graph node updates).
rec_status shard_capture(rec_model_s* m, Workspace& w) {
  cudaStream_t s = w.stream, sb = w.stream_b;
  for (auto& sl : w.slots) {
    SynthSlot::Variant& V = sl.var[0];
    sl.sa.tables = m->tables;
    sl.sa.T = m->T_loc;
    sl.sa.t0 = m->t0;
    sl.sa.dB = nullptr;
    sl.sa.pdl = 0;
    sl.sa.dense_bf = nullptr;
    sl.sa.hot_rows = 0;
    sl.sa.tma = 0;
    sl.sa.p2p = w.sh_sls;
    const int64_t before = m->launches;
    REC_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    cudaEventRecord(w.ev_fork, s);
    cudaStreamWaitEvent(sb, w.ev_fork, 0);
    launch_gen_dense_seg(*sl.sb_local, sl.ga, sb);  // writes dB = own block size
    {
      size_t n = 0;
      const cudaGraphNode_t* d = last_node(sb, &n);
      if (n == 1) V.dense_node = d[0];
    }
    enqueue_bottom(m, w, sb, w.cap, w.dB, nullptr);
    cudaEventRecord(w.ev_join, sb);
    launch_sls_synth(*sl.sb, sl.sa, s);
    {
      size_t n = 0;
      const cudaGraphNode_t* d = last_node(s, &n);
      if (n == 1) V.gen_node = d[0];
    }
    m->launches += 2;
    rec_status st = shard_tail(m, w, w.cap, w.dB, w.ev_join);
    cudaGraph_t g = nullptr;
    cudaError_t ce = cudaStreamEndCapture(s, &g);
    if (st != REC_OK) return st;
    if (ce != cudaSuccess) return cuda_fail(ce, "cudaStreamEndCapture (sharded chain)");
    if (!V.gen_node || !V.dense_node) {
      set_error("sharded graph capture: first-kernel nodes not found");
      return REC_E_CUDA;
    }
    V.graph = g;
    ce = cudaGraphInstantiate(&V.exec, g, 0);
    if (ce != cudaSuccess) return cuda_fail(ce, "cudaGraphInstantiate (sharded chain)");
    w.graph_kernels = static_cast<int>(m->launches - before);
    m->launches = before;
    sl.var[1] = SynthSlot::Variant{};  // no profiling variant in sharded mode
  }
  return REC_OK;
}

// The own item block [r * Bq, r * Bq + Bl) of a global batch given as host segments
// (qid, start, len), Bq = ceil(B / G): clipped segments into sl.sb_local (long lists through
// `stage` (pinned) -> w.gsegs_local on w.stream).  Returns the block size Bl.
int shard_fill_local(rec_model_s* m, Workspace& w, SynthSlot& sl, const int32_t* segs, int nseg,
                     int B, int4* stage) {
  const int G = m->world, Bq = (B + G - 1) / G, lo = m->rank * Bq;
  const int hi = std::min(B, lo + Bq);
  SegBatch& l = *sl.sb_local;
  int n = 0, row = 0;
  int4* dst = nseg > kParamSegs ? stage : l.seg;
  for (int i = 0; i < nseg; ++i) {
    const int len = segs[3 * i + 2];
    const int a = std::max(lo, row), b = std::min(hi, row + len);
    if (a < b) dst[n++] = make_int4(segs[3 * i], segs[3 * i + 1] + (a - row), b - a, a - lo);
    row += len;
  }
  l.B = std::max(0, hi - lo);
  l.nseg = n;
  l.gsegs = w.gsegs_local;
  if (n > kParamSegs) {
    cudaMemcpyAsync(w.gsegs_local, stage, sizeof(int4) * n, cudaMemcpyHostToDevice, w.stream);
  } else if (nseg > kParamSegs) {
    for (int i = 0; i < n; ++i) l.seg[i] = stage[i];
  }
  return l.B;
}

// Fused table-wise exchange: map every peer's X buffer and arrival flags into
// this process (CUDA IPC; handles exchanged with one ncclAllGather) so the SLS kernel stores
// pooled vectors straight into the owning rank's X over NVLink.  Off with REC_P2P=0, for the
// row-wise mode, or when some pair of GPUs has no peer access (NCCL path then).
rec_status p2p_init(rec_model_s* m) {
  const char* e = getenv("REC_P2P");
  if (m->shard == REC_SHARD_REPLICA || (e && atoi(e) == 0)) return REC_OK;
  const int G = m->world;
  // peer access: every rank must reach every other rank's memory
  int ok = 1;
  {
    int ndev = 0;
    REC_CUDA(cudaGetDeviceCount(&ndev));
    std::vector<int> devs(G, -1);
    // each rank contributes its device ordinal (same box: ordinals are comparable)
    int* d = nullptr;
    REC_CUDA(cudaMalloc(reinterpret_cast<void**>(&d), sizeof(int) * (G + 1)));
    REC_CUDA(cudaMemcpy(d + G, &m->device, sizeof(int), cudaMemcpyHostToDevice));
    ncclComm_t comm = static_cast<ncclComm_t>(m->nccl_comm);
    REC_NCCL(ncclAllGather(d + G, d, 1, ncclInt32, comm, m->ws[0].stream));
    REC_CUDA(cudaStreamSynchronize(m->ws[0].stream));
    REC_CUDA(cudaMemcpy(devs.data(), d, sizeof(int) * G, cudaMemcpyDeviceToHost));
    cudaFree(d);
    for (int q = 0; q < G; ++q) {
      if (q == m->rank) continue;
      int can = 0;
      if (devs[q] < 0 || devs[q] >= ndev || devs[q] == m->device ||
          cudaDeviceCanAccessPeer(&can, m->device, devs[q]) != cudaSuccess || !can)
        ok = 0;
    }
    // all ranks must agree: MIN over ranks
    int* f = nullptr;
    REC_CUDA(cudaMalloc(reinterpret_cast<void**>(&f), sizeof(int)));
    REC_CUDA(cudaMemcpy(f, &ok, sizeof(int), cudaMemcpyHostToDevice));
    REC_NCCL(ncclAllReduce(f, f, 1, ncclInt32, ncclMin, comm, m->ws[0].stream));
    REC_CUDA(cudaStreamSynchronize(m->ws[0].stream));
    REC_CUDA(cudaMemcpy(&ok, f, sizeof(int), cudaMemcpyDeviceToHost));
    cudaFree(f);
  }
  if (!ok) return REC_OK;
  if (m->shard == REC_SHARD_TABLE) return p2p_slots_init(m);
  REC_CUDA(cudaMalloc(reinterpret_cast<void**>(&m->p2p_flags), sizeof(unsigned) * G));
  REC_CUDA(cudaMemset(m->p2p_flags, 0, sizeof(unsigned) * G));
  REC_CUDA(cudaMalloc(reinterpret_cast<void**>(&m->p2p_counter), sizeof(unsigned)));
  float* target = m->ws[0].X;
  if (m->shard == REC_SHARD_ROW) {  // partial sums of every source rank: [G][Bq][T][D]
    const int64_t Bq = (m->max_batch + G - 1) / G;
    REC_CUDA(cudaMalloc(reinterpret_cast<void**>(&m->p2p_stage),
                        sizeof(float) * G * Bq * m->T * static_cast<int64_t>(m->D)));
    target = m->p2p_stage;
  }
  REC_CUDA(cudaMalloc(reinterpret_cast<void**>(&m->p2p_ctr_flags), sizeof(unsigned) * G));
  REC_CUDA(cudaMemset(m->p2p_ctr_flags, 0, sizeof(unsigned) * G));
  constexpr int NH = 4;  // exported buffers: X / staging, arrival flags, CTR gather, CTR flags
  cudaIpcMemHandle_t mine[NH];
  REC_CUDA(cudaIpcGetMemHandle(&mine[0], target));
  REC_CUDA(cudaIpcGetMemHandle(&mine[1], m->p2p_flags));
  REC_CUDA(cudaIpcGetMemHandle(&mine[2], m->sh_ctr));
  REC_CUDA(cudaIpcGetMemHandle(&mine[3], m->p2p_ctr_flags));
  const size_t hb = sizeof(mine);
  uint8_t* dh = nullptr;
  REC_CUDA(cudaMalloc(reinterpret_cast<void**>(&dh), hb * (G + 1)));
  REC_CUDA(cudaMemcpy(dh + hb * G, mine, hb, cudaMemcpyHostToDevice));
  REC_NCCL(ncclAllGather(dh + hb * G, dh, hb, ncclUint8, static_cast<ncclComm_t>(m->nccl_comm),
                         m->ws[0].stream));
  REC_CUDA(cudaStreamSynchronize(m->ws[0].stream));
  std::vector<cudaIpcMemHandle_t> all(NH * G);
  REC_CUDA(cudaMemcpy(all.data(), dh, hb * G, cudaMemcpyDeviceToHost));
  cudaFree(dh);
  std::vector<float*> px(G), pc(G);
  std::vector<unsigned*> pf(G), pcf(G);
  for (int q = 0; q < G; ++q) {
    if (q == m->rank) {
      px[q] = target;
      pf[q] = m->p2p_flags;
      pc[q] = m->sh_ctr;
      pcf[q] = m->p2p_ctr_flags;
      continue;
    }
    void* a[NH] = {};
    for (int k = 0; k < NH; ++k) {
      REC_CUDA(cudaIpcOpenMemHandle(&a[k], all[NH * q + k], cudaIpcMemLazyEnablePeerAccess));
      m->p2p_opened.push_back(a[k]);
    }
    px[q] = static_cast<float*>(a[0]);
    pf[q] = static_cast<unsigned*>(a[1]);
    pc[q] = static_cast<float*>(a[2]);
    pcf[q] = static_cast<unsigned*>(a[3]);
  }
  REC_CUDA(cudaMalloc(reinterpret_cast<void**>(&m->d_peer_X), sizeof(float*) * G));
  REC_CUDA(cudaMalloc(reinterpret_cast<void**>(&m->d_peer_flags), sizeof(unsigned*) * G));
  REC_CUDA(cudaMalloc(reinterpret_cast<void**>(&m->d_peer_ctr), sizeof(float*) * G));
  REC_CUDA(cudaMalloc(reinterpret_cast<void**>(&m->d_peer_ctr_flags), sizeof(unsigned*) * G));
  REC_CUDA(cudaMemcpy(m->d_peer_X, px.data(), sizeof(float*) * G, cudaMemcpyHostToDevice));
  REC_CUDA(cudaMemcpy(m->d_peer_flags, pf.data(), sizeof(unsigned*) * G, cudaMemcpyHostToDevice));
  REC_CUDA(cudaMemcpy(m->d_peer_ctr, pc.data(), sizeof(float*) * G, cudaMemcpyHostToDevice));
  REC_CUDA(cudaMemcpy(m->d_peer_ctr_flags, pcf.data(), sizeof(unsigned*) * G, cudaMemcpyHostToDevice));
  m->p2p = true;
  if (getenv("REC_VERBOSE"))
    fprintf(stderr, "[rec] rank %d: fused %s exchange over peer memory (%d ranks)\n", m->rank,
            m->shard == REC_SHARD_TABLE ? "all-to-all" : "reduce-scatter", G);
  return REC_OK;
}

// C4: every rank's values (variable counts) to every rank, through the model's communicator.
rec_status allgather_doubles(rec_model_s* m, const std::vector<double>& mine, std::vector<double>& all) {
  const int G = m->world;
  ncclComm_t comm = static_cast<ncclComm_t>(m->nccl_comm);
  cudaStream_t s = m->ws[0].stream;
  int64_t* dc = nullptr;
  REC_CUDA(cudaMalloc(reinterpret_cast<void**>(&dc), sizeof(int64_t) * (G + 1)));
  const int64_t n = static_cast<int64_t>(mine.size());
  REC_CUDA(cudaMemcpy(dc + G, &n, sizeof(int64_t), cudaMemcpyHostToDevice));
  REC_NCCL(ncclAllGather(dc + G, dc, 1, ncclInt64, comm, s));
  std::vector<int64_t> cnt(G);
  REC_CUDA(cudaStreamSynchronize(s));
  REC_CUDA(cudaMemcpy(cnt.data(), dc, sizeof(int64_t) * G, cudaMemcpyDeviceToHost));
  cudaFree(dc);
  int64_t mx = 1;
  for (int64_t c : cnt) mx = std::max(mx, c);
  double* dv = nullptr;
  REC_CUDA(cudaMalloc(reinterpret_cast<void**>(&dv), sizeof(double) * mx * (G + 1)));
  std::vector<double> pad(mx, 0.0);
  std::copy(mine.begin(), mine.end(), pad.begin());
  REC_CUDA(cudaMemcpy(dv + mx * G, pad.data(), sizeof(double) * mx, cudaMemcpyHostToDevice));
  REC_NCCL(ncclAllGather(dv + mx * G, dv, mx, ncclFloat64, comm, s));
  std::vector<double> buf(mx * G);
  REC_CUDA(cudaStreamSynchronize(s));
  REC_CUDA(cudaMemcpy(buf.data(), dv, sizeof(double) * mx * G, cudaMemcpyDeviceToHost));
  cudaFree(dv);
  all.clear();
  for (int q = 0; q < G; ++q) all.insert(all.end(), buf.begin() + q * mx, buf.begin() + q * mx + cnt[q]);
  return REC_OK;
}

rec_status sharded_alloc(rec_model_s* m) {
  const int G = m->world, cap = m->max_batch, D = m->D;
  const int64_t Bq = (cap + G - 1) / G;
  const int64_t per_item = (m->shard == REC_SHARD_TABLE ? m->T_loc : m->T) * static_cast<int64_t>(D);
  const size_t send = sizeof(float) * Bq * G * per_item;
  const size_t recv = m->shard == REC_SHARD_TABLE ? send : sizeof(float) * Bq * per_item;
  REC_CUDA(cudaMalloc(reinterpret_cast<void**>(&m->sh_send), send));
  REC_CUDA(cudaMalloc(reinterpret_cast<void**>(&m->sh_recv), recv));
  REC_CUDA(cudaMalloc(reinterpret_cast<void**>(&m->sh_ctr), sizeof(float) * Bq * G));
  REC_CUDA(cudaMemset(m->sh_send, 0, send));
  return REC_OK;
}

void dist_destroy(rec_model_s* m) {
  if (!m) return;
  for (void* p : m->p2p_opened) cudaIpcCloseMemHandle(p);
  m->p2p_opened.clear();
  cudaFree(m->d_peer_X);
  cudaFree(m->d_peer_flags);
  cudaFree(m->p2p_flags);
  cudaFree(m->p2p_counter);
  cudaFree(m->p2p_stage);
  cudaFree(m->d_peer_ctr);
  cudaFree(m->d_peer_ctr_flags);
  cudaFree(m->p2p_ctr_flags);
  m->p2p_stage = nullptr;
  m->d_peer_ctr = nullptr;
  m->d_peer_ctr_flags = nullptr;
  m->p2p_ctr_flags = nullptr;
  m->d_peer_X = nullptr;
  m->d_peer_flags = nullptr;
  m->p2p_flags = nullptr;
  m->p2p_counter = nullptr;
  m->p2p = false;
  cudaFree(m->sh_arena);
  cudaFree(m->d_sh_ptrs);
  m->sh_arena = nullptr;
  m->d_sh_ptrs = nullptr;
  m->p2p_slots = false;
  if (m->nccl_comm) {
    ncclCommDestroy(static_cast<ncclComm_t>(m->nccl_comm));
    m->nccl_comm = nullptr;
  }
  cudaFree(m->sh_send);
  cudaFree(m->sh_recv);
  cudaFree(m->sh_ctr);
  m->sh_send = m->sh_recv = m->sh_ctr = nullptr;
}

// Bound of a peer-flag wait (k_p2p_wait): REC_P2P_TIMEOUT_S seconds, default 60.
static unsigned long long p2p_timeout_ns() {
  static const unsigned long long ns = [] {
    const char* e = getenv("REC_P2P_TIMEOUT_S");
    const double sec = e ? atof(e) : 60.0;
    return static_cast<unsigned long long>((sec > 0 ? sec : 60.0) * 1e9);
  }();
  return ns;
}

rec_status sharded_forward(rec_model_s* m, Workspace& w, const float* d_dense, const int* d_idx,
                           const int* d_off, int B, float* ctr, float* logits) {
  const int G = m->world, r = m->rank, T = m->T, TL = m->T_loc, D = m->D;
  const int Bq = (B + G - 1) / G;
  const int item0 = r * Bq;
  const int Bl = B - item0 < 0 ? 0 : (B - item0 < Bq ? B - item0 : Bq);
  cudaStream_t s = w.stream;
  ncclComm_t comm = static_cast<ncclComm_t>(m->nccl_comm);
  const size_t xs = sizeof(float) * (T + 1) * D;
  // a3 on this GPU's shard, written in all-to-all / reduce-scatter order
  if (m->p2p_slots) {  // table-wise, asynchronous slot exchange on slot 0, then wait
    rec_status st = shard_enqueue(m, w, d_dense, d_idx, d_off, B, 0x7fffffff);
    if (st != REC_OK) return st;
    REC_CUDA(cudaMemcpyAsync(w.flag_host, w.flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    REC_CUDA(cudaStreamSynchronize(s));
    const int f = *w.flag_host;
    REC_CUDA(cudaMemsetAsync(w.flag, 0, sizeof(int), s));
    if (f & 1) {
      set_error("an index is outside [0, rows_t) (REC_E_INDEX_OOB)");
      return REC_E_INDEX_OOB;
    }
    if (f & 2) {
      set_error("offsets are not non-decreasing from 0 (REC_E_OFFSETS)");
      return REC_E_OFFSETS;
    }
    if (f & 4) {
      set_error("a peer rank missed the exchange deadline (REC_P2P_TIMEOUT_S); results invalid");
      return REC_E_NCCL;
    }
    REC_CUDA(cudaMemcpyAsync(ctr, w.sh_ctr_gather, sizeof(float) * B, cudaMemcpyDefault, s));
    if (logits && Bl > 0)
      REC_CUDA(cudaMemcpyAsync(logits + item0, w.logit, sizeof(float) * Bl, cudaMemcpyDefault, s));
    REC_CUDA(cudaStreamSynchronize(s));
    return REC_OK;
  }
  if (m->p2p) {
    // fused: pooled vectors land in the owners' X slots 1 + t0 .. over NVLink, then wait for
    // every rank's arrival flag of this epoch (the previous epoch's X readers all finished:
    // every rank raised its CTR flag of the previous epoch after its interaction, and this
    // rank saw all of them before the previous query returned)
    P2PArgs pa{};
    pa.peer_X = m->d_peer_X;
    pa.peer_flags = m->d_peer_flags;
    pa.counter = m->p2p_counter;
    pa.my_flags = m->p2p_flags;
    pa.Bq = Bq;
    pa.G = G;
    pa.rank = r;
    pa.epoch = ++m->p2p_epoch;
    pa.sc_fence = 1;
    pa.err_flag = w.flag;
    pa.timeout_ns = p2p_timeout_ns();
    REC_CUDA(cudaMemsetAsync(m->p2p_counter, 0, sizeof(unsigned), s));
    if (m->shard == REC_SHARD_TABLE) {
      pa.row_off = 0;
      launch_sls_p2p(m->tables, m->d_tab_off, m->row_stride, m->d_rows, d_idx, d_off + m->t0 * B, B,
                     TL, D, (T + 1) * D, 1 + m->t0, w.flag, pa, s);
      launch_p2p_wait(pa, s);
      m->launches += 2;
    } else {  // row-wise: partial sums into the owner's staging slot of this rank, then reduce
      pa.row_off = r * Bq;
      launch_sls_p2p(m->tables, m->d_tab_off, m->row_stride, m->d_rows, d_idx, d_off, B, T, D,
                     T * D, 0, w.flag, pa, s, static_cast<int>(m->row_lo), static_cast<int>(m->row_hi));
      launch_p2p_wait(pa, s);
      launch_p2p_reduce(m->p2p_stage, w.X, Bl, Bq, T, D, G, s);
      m->launches += 3;
    }
  } else if (m->shard == REC_SHARD_TABLE) {
    launch_sls(m->tables, m->d_tab_off, m->row_stride, m->d_rows, d_idx, d_off + m->t0 * B, B,
               nullptr, TL, D, m->sh_send, TL * D, 0, w.flag, s);
    REC_NCCL(ncclAlltoAll(m->sh_send, m->sh_recv, static_cast<size_t>(Bq) * TL * D, ncclFloat, comm, s));
    if (Bl > 0)
      for (int p = 0; p < G; ++p)  // peer p's tables [p*TL, (p+1)*TL) of my items -> X slots
        REC_CUDA(cudaMemcpy2DAsync(w.X + (1 + p * TL) * D, xs,
                                   m->sh_recv + static_cast<size_t>(p) * Bq * TL * D,
                                   sizeof(float) * TL * D, sizeof(float) * TL * D, Bl,
                                   cudaMemcpyDeviceToDevice, s));
  } else {
    launch_sls(m->tables, m->d_tab_off, m->row_stride, m->d_rows, d_idx, d_off, B, nullptr, T, D,
               m->sh_send, T * D, 0, w.flag, s, static_cast<int>(m->row_lo), static_cast<int>(m->row_hi));
    REC_NCCL(ncclReduceScatter(m->sh_send, m->sh_recv, static_cast<size_t>(Bq) * T * D, ncclFloat,
                               ncclSum, comm, s));
    if (Bl > 0)
      REC_CUDA(cudaMemcpy2DAsync(w.X + D, xs, m->sh_recv, sizeof(float) * T * D, sizeof(float) * T * D,
                                 Bl, cudaMemcpyDeviceToDevice, s));
  }
  m->launches += 1;
  // a4-a6 for this rank's item block
  if (Bl > 0) {
    launch_dense_to_bf16(d_dense + static_cast<size_t>(item0) * m->F, Bl, m->F, m->Fpad, w.dense_bf, s);
    m->launches += 1;
    enqueue_bottom(m, w, s, Bl, nullptr, nullptr);
    enqueue_interact_top(m, w, s, Bl, nullptr, w.ctr, w.logit, nullptr);
  }
  // C3: every rank gets every CTR (positions >= B of the padded gather are ignored)
  if (m->p2p) {  // peer stores + flags (this also orders the next query's X writes, see above)
    P2PArgs pc{};
    pc.peer_X = m->d_peer_ctr;
    pc.peer_flags = m->d_peer_ctr_flags;
    pc.my_flags = m->p2p_ctr_flags;
    pc.G = G;
    pc.rank = r;
    pc.epoch = m->p2p_epoch;
    pc.err_flag = w.flag;
    pc.timeout_ns = p2p_timeout_ns();
    launch_p2p_ctr_scatter(w.ctr, Bl, item0, pc, s);
    launch_p2p_wait(pc, s);
    m->launches += 2;
  } else {
    REC_NCCL(ncclAllGather(w.ctr, m->sh_ctr, Bq, ncclFloat, comm, s));
  }
  REC_CUDA(cudaMemcpyAsync(w.flag_host, w.flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  REC_CUDA(cudaStreamSynchronize(s));
  const int f = *w.flag_host;
  if (f & 1) {
    set_error("an index is outside [0, rows_t) (REC_E_INDEX_OOB)");
    return REC_E_INDEX_OOB;
  }
  if (f & 2) {
    set_error("offsets are not non-decreasing from 0 (REC_E_OFFSETS)");
    return REC_E_OFFSETS;
  }
  if (f & 4) {
    set_error("a peer rank missed the exchange deadline (REC_P2P_TIMEOUT_S); results invalid");
    return REC_E_NCCL;
  }
  REC_CUDA(cudaMemcpyAsync(ctr, m->sh_ctr, sizeof(float) * B, cudaMemcpyDefault, s));
  if (logits) {  // logits of this rank's own items only (diagnostic)
    if (Bl > 0)
      REC_CUDA(cudaMemcpyAsync(logits + item0, w.logit, sizeof(float) * Bl, cudaMemcpyDefault, s));
  }
  REC_CUDA(cudaStreamSynchronize(s));
  return REC_OK;
}

}  // namespace rec

extern "C" {

int32_t rec_nccl_unique_id_size(void) { return static_cast<int32_t>(sizeof(ncclUniqueId)); }

rec_status rec_nccl_get_unique_id(void* out) {
  if (!out) {
    rec::set_error("out must be non-null");
    return REC_E_INVALID_ARG;
  }
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) {
    rec::set_error("ncclGetUniqueId failed: %s", ncclGetErrorString(r));
    return REC_E_NCCL;
  }
  memcpy(out, &id, sizeof(id));
  return REC_OK;
}

rec_status rec_shard_plan(int32_t num_tables, const int64_t* rows, int32_t world, int32_t rank,
                          int32_t shard, int32_t batch, int64_t* out) {
  if (!rows || !out || num_tables < 1 || world < 1 || rank < 0 || rank >= world || batch < 0) {
    rec::set_error("bad argument");
    return REC_E_INVALID_ARG;
  }
  rec::ShardPlan p{};
  rec_status st = rec::shard_plan(num_tables, rows, world, rank, shard, &p);
  if (st != REC_OK) return st;
  const int64_t Bq = world > 1 && shard != REC_SHARD_REPLICA ? (batch + world - 1) / world : batch;
  const int64_t item0 = world > 1 && shard != REC_SHARD_REPLICA ? rank * Bq : 0;
  int64_t cnt = batch - item0;
  cnt = cnt < 0 ? 0 : (cnt < Bq ? cnt : Bq);
  out[0] = p.t0;
  out[1] = p.t_local;
  out[2] = p.row_lo;
  out[3] = p.row_hi;
  out[4] = item0;
  out[5] = cnt;
  return REC_OK;
}

}  // extern "C"
