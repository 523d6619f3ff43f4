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
  rec_status st = sharded_alloc(m);
  if (st != REC_OK) return st;
  return p2p_init(m);
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
