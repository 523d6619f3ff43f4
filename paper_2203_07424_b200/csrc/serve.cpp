// serve.cpp — query splitter / fuser (S1, S2) and the serving runtime rec_serve (a1, a7).
//
// "each large inference query is split into multiple sub-queries ...
// On accelerators, the inference queries are fused into one large batch ... query fusion";
// model co-location = m concurrent inference threads on one accelerator, here
// m CUDA streams (one workspace each) with one dispatcher thread each; the objective
// is throughput under a tail-latency SLA.
//
// Real clock: queries are released open-loop at their trace arrival times (busy-waiting on
// CLOCK_MONOTONIC); whenever a stream is idle its dispatcher fuses FIFO sub-queries into a
// batch (Σ <= d) and submits input materialisation + the forward chain (one captured graph)
// on that stream; completion is observed by polling a host-mapped word the stream writes
// after the batch; a query's latency ends when the host observes the completion of its last
// sub-query (reading R16).
// Virtual clock (S4): identical dispatch rules on a simulated clock with service time
// alpha + beta * items, so the batch list is unique and bit-exact with oracle/serving.py;
// the kernels still run for every batch (CTRs are real).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <mutex>
#include <thread>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <queue>
#include <vector>

#include <nccl.h>

#include "model.h"

static inline void cpu_relax() {
#if defined(__x86_64__) || defined(__i386__)
  __builtin_ia32_pause();
#endif
}

namespace rec {

struct Chunk {
  int32_t qid, start, len;
  int64_t pos;  // trace row
};

// S1: chunks of d, remainder last (reading R14).
static void split_query(const rec_trace_row& r, int64_t pos, int32_t d, std::vector<Chunk>& out) {
  const int32_t k = (r.size + d - 1) / d;
  for (int32_t c = 0; c < k; ++c)
    out.push_back(Chunk{r.qid, c * d, c < k - 1 ? d : r.size - (k - 1) * d, pos});
}

// S2: number of FIFO-head chunks whose cumulative length stays <= d (at least one).
static int64_t fuse_head(const std::vector<Chunk>& fifo, int64_t head, int32_t d, int64_t* items) {
  int64_t k = 0, tot = 0;
  for (int64_t i = head; i < static_cast<int64_t>(fifo.size()); ++i) {
    if (k > 0 && tot + fifo[i].len > d) break;
    tot += fifo[i].len;
    ++k;
  }
  *items = tot;
  return k;
}

static inline double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static int64_t pct_rank(int pct, int64_t n) { return std::max<int64_t>((pct * n + 99) / 100, 1); }

struct Batch {
  int stream = -1;
  int64_t first_chunk = 0, nchunks = 0, items = 0;
  double t_dispatch = 0, t_done = 0;
  int slot = -1;            // staging slot whose graph (with stage events) ran the batch
  double host_in_ms = 0;    // host-input mode: packing into pinned staging (host clock)
};

// Per-stream state of the serving loop.
struct Lane {
  bool busy = false;
  int64_t batch = -1;
  cudaEvent_t done = nullptr;
  float* ctr_host = nullptr;       // pinned [cap]
  uint32_t* flag_host = nullptr;   // pinned + mapped: batch sequence number written by the GPU
  CUdeviceptr flag_dev = 0;
  cudaEvent_t hev[8] = {};         // host-input mode: stage events of the lane's batch
};

// Stage times of a finished batch (P:418 latency components), ms: [0] input (H2D / pack),
// [1] sparse (SLS incl. fused index generation), [2] dense (chain device time not in the SLS:
// the bottom branch beyond the SLS, interaction, top MLP).  ev: the stage events of forward_
// enqueue / synth_chain (0 start, 1 inputs done, 2 SLS done, 5 top done).
static void stage_times(const cudaEvent_t* ev, bool host_mode, double host_in_ms, double out[3]) {
  auto el = [&](int a, int b) {
    float x = 0.f;
    if (!ev[a] || !ev[b] || cudaEventElapsedTime(&x, ev[a], ev[b]) != cudaSuccess) {
      cudaGetLastError();
      return 0.0;
    }
    return static_cast<double>(x);
  };
  if (host_mode) {  // 0 -> 1: host packing + the batch's H2D copies (ev 0 is recorded before
                   // the packing); then SLS; the rest is dense
    (void)host_in_ms;
    const double in = el(0, 1), sp = el(1, 2), all = el(0, 5);
    out[0] = in;
    out[1] = sp;
    out[2] = std::max(0.0, all - in - sp);
  } else {         // device-synthesised inputs are generated inside the SLS / dense kernels
    const double sp = el(0, 2), all = el(0, 5);
    out[0] = 0.0;
    out[1] = sp;   // chain start -> SLS done (incl. waiting for SMs held by co-located batches)
    out[2] = std::max(0.0, all - sp);
  }
}

// cuStreamWriteValue32 through the runtime's driver entry point (no libcuda link).
static rec_status stream_write_u32(cudaStream_t s, CUdeviceptr addr, uint32_t v) {
  using Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
  static Fn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q);
    return reinterpret_cast<Fn>(p);
  }();
  if (!fn) return REC_E_UNSUPPORTED;
  return fn(reinterpret_cast<CUstream>(s), addr, v, 0) == CUDA_SUCCESS ? REC_OK : REC_E_CUDA;
}

// Host-input mode: per-query materialised inputs (table-major within the query).
struct HostInputs {
  std::vector<int64_t> q_item_base;  // first global item of query p
  std::vector<int64_t> idx_base;     // [p*T + t] -> start in idx
  std::vector<int32_t> idx;          // all indices
  std::vector<int32_t> len;          // [item*T + t] bag lengths
  std::vector<float> dense;          // [item][F]
};

static rec_status build_host_inputs(rec_model_s* m, const rec_trace_row* tr, int64_t n,
                                    HostInputs& H) {
  const int T = m->T, F = m->F;
  Workspace& w = m->ws[0];
  H.q_item_base.resize(n + 1);
  int64_t items = 0;
  for (int64_t p = 0; p < n; ++p) {
    H.q_item_base[p] = items;
    items += tr[p].size;
  }
  H.q_item_base[n] = items;
  H.len.assign(items * T, 0);
  H.dense.assign(items * F, 0.f);
  H.idx_base.assign(n * T + 1, 0);
  // generate per query in chunks of <= cap items through the device generator (G2-G4)
  std::vector<int32_t> off_h(static_cast<size_t>(T) * w.cap + 1);
  std::vector<int32_t> idx_h(w.idx_cap);
  std::vector<std::vector<int32_t>> per_q_t;  // scratch for one query
  for (int64_t p = 0; p < n; ++p) {
    per_q_t.assign(T, {});
    for (int32_t s0 = 0; s0 < tr[p].size; s0 += w.cap) {
      const int32_t ln = std::min<int32_t>(w.cap, tr[p].size - s0);
      int32_t seg[3] = {tr[p].qid, s0, ln};
      rec_status st = rec_gen_batch(m, seg, 1, idx_h.data(), off_h.data(),
                                    H.dense.data() + (H.q_item_base[p] + s0) * F);
      if (st != REC_OK) return st;
      for (int t = 0; t < T; ++t) {
        for (int b = 0; b < ln; ++b) {
          const int g = t * ln + b;
          H.len[(H.q_item_base[p] + s0 + b) * T + t] = off_h[g + 1] - off_h[g];
          per_q_t[t].insert(per_q_t[t].end(), idx_h.begin() + off_h[g], idx_h.begin() + off_h[g + 1]);
        }
      }
    }
    for (int t = 0; t < T; ++t) {
      H.idx_base[p * T + t] = static_cast<int64_t>(H.idx.size());
      H.idx.insert(H.idx.end(), per_q_t[t].begin(), per_q_t[t].end());
    }
  }
  H.idx_base[n * T] = static_cast<int64_t>(H.idx.size());
  return REC_OK;
}

// Pack a batch's host inputs into the workspace's pinned staging and copy them over
// PCIe (the paper's data-loading stage).  Returns the number of items.
static rec_status host_input_enqueue(rec_model_s* m, Workspace& w, const HostInputs& H,
                                     const std::vector<Chunk>& fifo, int64_t c0, int64_t nc,
                                     int* B_out) {
  const int T = m->T, F = m->F;
  REC_CUDA(cudaEventSynchronize(w.pin_free));
  int B = 0;
  for (int64_t c = c0; c < c0 + nc; ++c) B += fifo[c].len;
  int32_t* off = reinterpret_cast<int32_t*>(w.pin);
  size_t off_bytes = ((sizeof(int32_t) * (static_cast<size_t>(T) * B + 1)) + 255) & ~size_t(255);
  int32_t* idx = reinterpret_cast<int32_t*>(w.pin + off_bytes);
  // offsets + indices, table-major over the batch
  int64_t nnz = 0;
  int g = 0;
  off[0] = 0;
  for (int t = 0; t < T; ++t) {
    for (int64_t c = c0; c < c0 + nc; ++c) {
      const Chunk& ch = fifo[c];
      const int64_t item0 = H.q_item_base[ch.pos] + ch.start;
      // indices of this chunk for table t are contiguous in the query's table-t list
      int64_t skip = 0;
      for (int64_t it = H.q_item_base[ch.pos]; it < item0; ++it) skip += H.len[it * T + t];
      int64_t cnt = 0;
      for (int b = 0; b < ch.len; ++b) {
        cnt += H.len[(item0 + b) * T + t];
        off[++g] = static_cast<int32_t>(nnz + cnt);
      }
      memcpy(idx + nnz, H.idx.data() + H.idx_base[ch.pos * T + t] + skip, sizeof(int32_t) * cnt);
      nnz += cnt;
    }
  }
  size_t idx_bytes = ((sizeof(int32_t) * nnz) + 255) & ~size_t(255);
  float* dn = reinterpret_cast<float*>(w.pin + off_bytes + idx_bytes);
  int row = 0;
  for (int64_t c = c0; c < c0 + nc; ++c) {
    const Chunk& ch = fifo[c];
    memcpy(dn + static_cast<size_t>(row) * F,
           H.dense.data() + (H.q_item_base[ch.pos] + ch.start) * F, sizeof(float) * ch.len * F);
    row += ch.len;
  }
  cudaStream_t s = w.stream;
  REC_CUDA(cudaMemcpyAsync(w.offsets, off, sizeof(int32_t) * (static_cast<size_t>(T) * B + 1),
                           cudaMemcpyHostToDevice, s));
  REC_CUDA(cudaMemcpyAsync(w.indices, idx, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, s));
  if (F > 0)
    REC_CUDA(cudaMemcpyAsync(w.dense_f32, dn, sizeof(float) * B * F, cudaMemcpyHostToDevice, s));
  REC_CUDA(cudaEventRecord(w.pin_free, s));
  launch_dense_to_bf16(w.dense_f32, B, F, m->Fpad, w.dense_bf, s);
  m->launches += 1;
  *B_out = B;
  return REC_OK;
}

// S5 report: per-query latency = completion of the last sub-query - arrival (R16), nearest-
// rank percentiles over queries arriving after the warm-up window, offered / achieved rate.
static void fill_report(const rec_trace_row* trace, int64_t n, double sla_ms, double warmup_frac,
                        const std::vector<double>& release, const std::vector<double>& disp_t,
                        const std::vector<double>& done_t, int64_t completed, int64_t nbatches,
                        double items_tot, double* latency_ms, rec_serve_report* out,
                        const std::vector<double>* comp = nullptr, rec_model_s* gm = nullptr) {
  const double t_first = trace[0].arrival_s, t_last = trace[n - 1].arrival_s;
  const double w_end = t_first + warmup_frac * (t_last - t_first);
  std::vector<double> lat;
  double sum_lat = 0, sum_q = 0, sum_svc = 0, t_max = t_first, sum_c[3] = {0, 0, 0};
  for (int64_t p = 0; p < n; ++p) {
    const double l = done_t[p] - release[p];
    if (latency_ms) latency_ms[p] = l * 1e3;
    t_max = std::max(t_max, done_t[p]);
    if (release[p] >= w_end) {
      lat.push_back(l * 1e3);
      sum_lat += l * 1e3;
      sum_q += (disp_t[p] - release[p]) * 1e3;
      sum_svc += (done_t[p] - disp_t[p]) * 1e3;
      if (comp)
        for (int k = 0; k < 3; ++k) sum_c[k] += comp[k][p];
    }
  }
  double offered = t_last > t_first ? n / (t_last - t_first) : INFINITY;
  double achieved = t_max > t_first ? n / (t_max - t_first) : 0;
  bool stable = (completed == n) && achieved >= 0.98 * offered;
  int ranks = 1;
  int64_t n_all = n;
  if (gm) {  // replicas with a communicator: percentiles over every rank's queries (C4)
    std::vector<double> mine = {static_cast<double>(completed), static_cast<double>(n), stable ? 1.0 : 0.0,
                                offered, achieved, sum_lat, sum_q, sum_svc, sum_c[0], sum_c[1], sum_c[2],
                                static_cast<double>(nbatches), items_tot};
    std::vector<double> sc, all_lat;
    if (allgather_doubles(gm, mine, sc) == REC_OK && allgather_doubles(gm, lat, all_lat) == REC_OK) {
      ranks = gm->world;
      completed = 0;
      n_all = 0;
      offered = achieved = sum_lat = sum_q = sum_svc = items_tot = 0;
      sum_c[0] = sum_c[1] = sum_c[2] = 0;
      nbatches = 0;
      for (int q = 0; q < ranks; ++q) {
        const double* v = sc.data() + 13 * q;
        completed += static_cast<int64_t>(v[0]);
        n_all += static_cast<int64_t>(v[1]);
        stable = stable && v[2] > 0.5;
        offered += v[3];
        achieved += v[4];
        sum_lat += v[5];
        sum_q += v[6];
        sum_svc += v[7];
        for (int k = 0; k < 3; ++k) sum_c[k] += v[8 + k];
        nbatches += static_cast<int64_t>(v[11]);
        items_tot += v[12];
      }
      lat.swap(all_lat);
    }
  }
  std::sort(lat.begin(), lat.end());
  const int64_t nm = static_cast<int64_t>(lat.size());
  memset(out, 0, sizeof(*out));
  out->ranks = ranks;
  out->completed = completed;
  out->dropped = n_all - completed;
  out->batches = nbatches;
  out->mean_batch = nbatches ? items_tot / nbatches : 0;
  if (nm > 0) {
    out->p50_ms = lat[pct_rank(50, nm) - 1];
    out->p95_ms = lat[pct_rank(95, nm) - 1];
    out->p99_ms = lat[pct_rank(99, nm) - 1];
    out->mean_ms = sum_lat / nm;
    out->breakdown_ms[0] = sum_q / nm;   // queueing (arrival -> dispatch of last sub-query)
    if (comp) {                          // stages of the batch that completed the query
      out->breakdown_ms[1] = sum_c[0] / nm;  // input (H2D + host packing; 0 device-synth)
      out->breakdown_ms[2] = sum_c[1] / nm;  // sparse (SLS)
      out->breakdown_ms[3] = sum_c[2] / nm;  // dense (bottom beyond the SLS, interaction, top)
    } else {
      out->breakdown_ms[2] = sum_svc / nm;   // dispatch -> observed completion, undivided
    }
  }
  out->offered_qps = offered;
  out->achieved_qps = achieved;
  out->stable = stable;
  out->sla_met = out->stable && out->p95_ms <= sla_ms;
}

// ------------------------------------------------------------------------------------------
// Table-wise sharded serving: every rank runs the
// SAME global batch sequence, because each rank's chain exchanges pooled vectors and CTRs with
// every other rank's chain of that batch.  Batch composition therefore cannot depend on when
// a rank's streams become idle (S2's work-conserving trigger): a deterministic global
// dispatcher cuts batches from the trace alone (reading R31) -
//   the FIFO of sub-queries (S1) is cut into batches of whole sub-queries with cumulative
//   size <= d; a batch closes when it is full (the next sub-query would not fit, or it holds
//   exactly d items) or tau after its first sub-query arrived, whichever comes first;
//   batch k goes to stream slot k mod m.
// Every rank releases batch k at max(its close time, completion of batch k - m on that slot)
// on its own clock (clocks aligned by an NCCL barrier before the trace starts); the device
// flags order the exchange, so no host message is needed per batch.
struct ShardBatch {
  int64_t c0, nc, items;
  double close;  // trace time
};

static void cut_batches(const rec_trace_row* trace, const std::vector<Chunk>& ch, int32_t d, double tau,
                        std::vector<ShardBatch>& out) {
  double prev = -INFINITY;
  const int64_t nch = static_cast<int64_t>(ch.size());
  for (int64_t i = 0; i < nch;) {
    const double first = trace[ch[i].pos].arrival_s, deadline = first + tau;
    int64_t j = i, items = 0;
    while (j < nch && items + ch[j].len <= d && trace[ch[j].pos].arrival_s <= deadline) items += ch[j++].len;
    if (j == i) items += ch[j++].len;  // (a sub-query is never larger than d)
    double close = deadline;
    if (items == d) close = trace[ch[j - 1].pos].arrival_s;                      // exactly full
    else if (j < nch && trace[ch[j].pos].arrival_s <= deadline) close = trace[ch[j].pos].arrival_s;  // next overflows
    close = std::max(close, prev);
    out.push_back(ShardBatch{i, j - i, items, close});
    prev = close;
    i = j;
  }
}

static rec_status serve_sharded(rec_model_s* m, const rec_trace_row* trace, int64_t n, double sla_ms,
                                const rec_serve_policy* pol, rec_serve_report* out, double* latency_ms,
                                int32_t* batch_log, int64_t log_cap, int64_t* log_rows, float* ctr_out) {
  if (pol->input_mode != REC_INPUT_DEVICE_SYNTH || pol->clock != REC_CLOCK_REAL) {
    set_error("sharded serving: device-synthesised inputs and the real clock only");
    return REC_E_UNSUPPORTED;
  }
  if (!(m->p2p_slots && m->ws[0].slots[0].var[0].exec)) {
    set_error("sharded serving needs table-wise sharding over peer memory and fixed pooling");
    return REC_E_UNSUPPORTED;
  }
  const int M = pol->streams;
  const int32_t d = pol->max_batch;
  // tau (R31): the policy's fusion timeout, else SLA / 50 (1 ms at RMC2's 50 ms SLA)
  const double tau = (pol->fusion_timeout_ms > 0 ? pol->fusion_timeout_ms : sla_ms / 50.0) * 1e-3;
  std::vector<Chunk> ch;
  ch.reserve(static_cast<size_t>(n) * 2);
  for (int64_t p = 0; p < n; ++p) split_query(trace[p], p, d, ch);
  std::vector<ShardBatch> bt;
  cut_batches(trace, ch, d, tau, bt);
  const int64_t nb = static_cast<int64_t>(bt.size());
  std::vector<int64_t> item_base;
  if (ctr_out) {
    item_base.resize(n);
    int64_t acc = 0;
    for (int64_t p = 0; p < n; ++p) {
      item_base[p] = acc;
      acc += trace[p].size;
    }
  }
  std::vector<Lane> lanes(M);
  auto cleanup = [&]() {
    for (auto& L : lanes) {
      if (L.ctr_host) cudaFreeHost(L.ctr_host);
      if (L.flag_host) cudaFreeHost(L.flag_host);
    }
  };
  for (int s = 0; s < M; ++s) {
    void* hp = nullptr;
    void* dp = nullptr;
    if (cudaHostAlloc(&hp, 64, cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer(&dp, hp, 0) != cudaSuccess) {
      cleanup();
      set_error("mapped completion words unavailable");
      return REC_E_CUDA;
    }
    lanes[s].flag_host = static_cast<uint32_t*>(hp);
    lanes[s].flag_dev = reinterpret_cast<CUdeviceptr>(dp);
    *lanes[s].flag_host = 0;
    if (ctr_out && cudaMallocHost(reinterpret_cast<void**>(&lanes[s].ctr_host), sizeof(float) * d) != cudaSuccess) {
      cleanup();
      return REC_E_OOM;
    }
  }
  for (int s = 0; s < M; ++s) {
    rec_status st = rec_sync(m, s);
    if (st != REC_OK) { cleanup(); return st; }
  }
  // clock alignment: every rank leaves this barrier within a few microseconds
  {
    int* f = nullptr;
    REC_CUDA(cudaMalloc(reinterpret_cast<void**>(&f), sizeof(int)));
    REC_CUDA(cudaMemsetAsync(f, 0, sizeof(int), m->ws[0].stream));
    ncclResult_t r = ncclAllReduce(f, f, 1, ncclInt32, ncclSum, static_cast<ncclComm_t>(m->nccl_comm),
                                   m->ws[0].stream);
    cudaStreamSynchronize(m->ws[0].stream);
    cudaFree(f);
    if (r != ncclSuccess) {
      cleanup();
      set_error("NCCL barrier failed: %s", ncclGetErrorString(r));
      return REC_E_NCCL;
    }
  }
  std::vector<int32_t> remaining(n);
  for (int64_t p = 0; p < n; ++p) remaining[p] = (trace[p].size + d - 1) / d;
  std::vector<double> done_t(n, NAN), release(n), disp_t(n, NAN);
  for (int64_t p = 0; p < n; ++p) release[p] = trace[p].arrival_s;
  // depth 2: a slot's next batch waits in its stream behind the running one, so a slot never
  // idles between a completion and the host's next submit (REC_SERVE_DEPTH overrides; the
  // CTR read-back staging is per slot, so depth 1 when CTRs are returned)
  int depth = 2;
  if (const char* e = getenv("REC_SERVE_DEPTH")) depth = std::max(1, std::min(4, atoi(e)));
  if (ctr_out) depth = 1;
  std::vector<std::deque<std::pair<int64_t, uint32_t>>> pend(M);
  std::vector<uint32_t> seq(M, 0);
  std::vector<int32_t> segs;
  int64_t completed = 0, logged = 0;
  const double t_first = trace[0].arrival_s;
  const double t0 = now_s() - t_first;
  auto finish = [&](int s) {
    const int64_t k = pend[s].front().first;
    const double tc = now_s() - t0;
    for (int64_t c = bt[k].c0; c < bt[k].c0 + bt[k].nc; ++c)
      if (--remaining[ch[c].pos] == 0) {
        done_t[ch[c].pos] = tc;
        ++completed;
      }
    if (ctr_out) {
      int row = 0;
      for (int64_t c = bt[k].c0; c < bt[k].c0 + bt[k].nc; ++c) {
        memcpy(ctr_out + item_base[ch[c].pos] + ch[c].start, lanes[s].ctr_host + row, sizeof(float) * ch[c].len);
        row += ch[c].len;
      }
    }
    pend[s].pop_front();
  };
  auto poll = [&]() {
    for (int s = 0; s < M; ++s)
      while (!pend[s].empty() &&
             static_cast<int32_t>(*reinterpret_cast<volatile uint32_t*>(lanes[s].flag_host) -
                                  pend[s].front().second) >= 0)
        finish(s);
  };
  for (int64_t k = 0; k < nb; ++k) {
    const int s = static_cast<int>(k % M);
    while (static_cast<int>(pend[s].size()) >= depth || now_s() - t0 < bt[k].close) {
      poll();
      cpu_relax();
    }
    Workspace& w = m->ws[s];
    segs.resize(3 * bt[k].nc);
    for (int64_t c = 0; c < bt[k].nc; ++c) {
      const Chunk& x = ch[bt[k].c0 + c];
      segs[3 * c] = x.qid;
      segs[3 * c + 1] = x.start;
      segs[3 * c + 2] = x.len;
      if (batch_log && logged < log_cap) {
        int32_t* r = batch_log + 5 * logged++;
        r[0] = static_cast<int32_t>(k);
        r[1] = s;
        r[2] = x.qid;
        r[3] = x.start;
        r[4] = x.len;
      }
    }
    const double td = now_s() - t0;
    int B = 0;
    rec_status st = synth_submit(m, w, segs.data(), static_cast<int>(bt[k].nc), &B, nullptr);
    if (st == REC_OK && ctr_out &&
        cudaMemcpyAsync(lanes[s].ctr_host, w.sh_ctr_gather, sizeof(float) * B, cudaMemcpyDeviceToHost,
                        w.stream) != cudaSuccess)
      st = REC_E_CUDA;
    if (st == REC_OK) st = stream_write_u32(w.stream, lanes[s].flag_dev, ++seq[s]);
    if (st != REC_OK) { cleanup(); return st; }
    for (int64_t c = bt[k].c0; c < bt[k].c0 + bt[k].nc; ++c) disp_t[ch[c].pos] = td;
    pend[s].emplace_back(k, seq[s]);
  }
  bool any = true;
  while (any) {
    poll();
    any = false;
    for (int s = 0; s < M; ++s) any = any || !pend[s].empty();
    if (any) cpu_relax();
  }
  for (int s = 0; s < M; ++s) {
    rec_status st = rec_sync(m, s);
    if (st != REC_OK) { cleanup(); return st; }
  }
  cleanup();
  double items_tot = 0;
  for (auto& b : bt) items_tot += b.items;
  fill_report(trace, n, sla_ms, pol->warmup_frac, release, disp_t, done_t, completed, nb, items_tot,
              latency_ms, out);
  if (log_rows) *log_rows = logged;
  return REC_OK;
}

}  // namespace rec

using namespace rec;

extern "C" {

rec_status rec_split_fuse(const rec_trace_row* trace, int64_t n, int32_t max_batch,
                          int32_t* segs_out, int64_t seg_cap, int64_t* batch_start, int64_t bcap,
                          int64_t* nbatches, int64_t* nsegs) {
  if (!trace || !segs_out || !batch_start || !nbatches || !nsegs || n < 0) {
    set_error("null argument");
    return REC_E_INVALID_ARG;
  }
  if (max_batch < 1) {
    set_error("max_batch = %d must be >= 1", max_batch);
    return REC_E_INVALID_ARG;
  }
  std::vector<Chunk> fifo;
  for (int64_t p = 0; p < n; ++p) {
    if (trace[p].size < 1) {
      set_error("trace[%lld].size = %d must be >= 1", (long long)p, trace[p].size);
      return REC_E_INVALID_ARG;
    }
    split_query(trace[p], p, max_batch, fifo);
  }
  if (static_cast<int64_t>(fifo.size()) > seg_cap) {
    set_error("seg_cap = %lld < %zu sub-queries", (long long)seg_cap, fifo.size());
    return REC_E_INVALID_ARG;
  }
  int64_t head = 0, b = 0;
  batch_start[0] = 0;
  while (head < static_cast<int64_t>(fifo.size())) {
    int64_t items = 0;
    const int64_t k = fuse_head(fifo, head, max_batch, &items);
    if (b + 1 > bcap) {
      set_error("bcap = %lld too small", (long long)bcap);
      return REC_E_INVALID_ARG;
    }
    for (int64_t i = head; i < head + k; ++i) {
      segs_out[3 * i] = fifo[i].qid;
      segs_out[3 * i + 1] = fifo[i].start;
      segs_out[3 * i + 2] = fifo[i].len;
    }
    head += k;
    batch_start[++b] = head;
  }
  *nbatches = b;
  *nsegs = head;
  return REC_OK;
}

rec_status rec_global_batches(const rec_trace_row* trace, int64_t n, int32_t max_batch, double tau_ms,
                              int32_t* segs_out, int64_t seg_cap, int64_t* batch_start, double* close_s,
                              int64_t bcap, int64_t* nbatches, int64_t* nsegs) {
  if (!trace || !segs_out || !batch_start || !close_s || !nbatches || !nsegs || n < 0) {
    set_error("null argument");
    return REC_E_INVALID_ARG;
  }
  if (max_batch < 1 || !(tau_ms > 0)) {
    set_error("max_batch >= 1 and tau_ms > 0 are required");
    return REC_E_INVALID_ARG;
  }
  std::vector<Chunk> ch;
  for (int64_t p = 0; p < n; ++p) {
    if (trace[p].size < 1 || (p > 0 && trace[p].arrival_s < trace[p - 1].arrival_s)) {
      set_error("trace[%lld]: size >= 1 and non-decreasing arrival_s required", (long long)p);
      return REC_E_INVALID_ARG;
    }
    split_query(trace[p], p, max_batch, ch);
  }
  std::vector<ShardBatch> bt;
  cut_batches(trace, ch, max_batch, tau_ms * 1e-3, bt);
  if (static_cast<int64_t>(ch.size()) > seg_cap || static_cast<int64_t>(bt.size()) > bcap) {
    set_error("capacity too small (%zu sub-queries, %zu batches)", ch.size(), bt.size());
    return REC_E_INVALID_ARG;
  }
  for (size_t i = 0; i < ch.size(); ++i) {
    segs_out[3 * i] = ch[i].qid;
    segs_out[3 * i + 1] = ch[i].start;
    segs_out[3 * i + 2] = ch[i].len;
  }
  batch_start[0] = 0;
  for (size_t k = 0; k < bt.size(); ++k) {
    batch_start[k + 1] = bt[k].c0 + bt[k].nc;
    close_s[k] = bt[k].close;
  }
  *nbatches = static_cast<int64_t>(bt.size());
  *nsegs = static_cast<int64_t>(ch.size());
  return REC_OK;
}

rec_status rec_serve(rec_model_t m, const rec_trace_row* trace, int64_t n, double sla_ms,
                     const rec_serve_policy* pol, rec_serve_report* out, double* latency_ms,
                     int32_t* batch_log, int64_t log_cap, int64_t* log_rows, float* ctr_out) {
  // ------------------------------------------------ validation (before any work)
  if (!m || !trace || !pol || !out || n < 1) {
    set_error("model, trace (n >= 1), policy and report are required");
    return REC_E_INVALID_ARG;
  }
  if (pol->streams < 1 || pol->streams > m->nstreams) {
    set_error("policy.streams = %d must be in [1, model streams = %d]", pol->streams, m->nstreams);
    return REC_E_INVALID_ARG;
  }
  if (pol->max_batch < 1 || pol->max_batch > m->max_batch) {
    set_error("policy.max_batch = %d must be in [1, model max_batch = %d]", pol->max_batch,
              m->max_batch);
    return REC_E_INVALID_ARG;
  }
  if (!(pol->fusion_timeout_ms >= 0) || !(pol->warmup_frac >= 0 && pol->warmup_frac < 1) ||
      (pol->clock != REC_CLOCK_REAL && pol->clock != REC_CLOCK_VIRTUAL) ||
      (pol->input_mode != REC_INPUT_DEVICE_SYNTH && pol->input_mode != REC_INPUT_HOST) ||
      !(sla_ms > 0)) {
    set_error("policy: fusion_timeout_ms >= 0, warmup_frac in [0,1), known clock/input_mode "
              "and sla_ms > 0 are required");
    return REC_E_INVALID_ARG;
  }
  if (pol->clock == REC_CLOCK_VIRTUAL && !(pol->alpha_ns >= 0 && pol->beta_ns >= 0 &&
                                           pol->alpha_ns + pol->beta_ns > 0)) {
    set_error("virtual clock needs alpha_ns, beta_ns >= 0 with alpha_ns + beta_ns > 0");
    return REC_E_INVALID_ARG;
  }
  for (int64_t p = 0; p < n; ++p) {
    if (trace[p].size < 1 || trace[p].qid < 0 || (p > 0 && trace[p].arrival_s < trace[p - 1].arrival_s)) {
      set_error("trace[%lld]: size >= 1, qid >= 0 and non-decreasing arrival_s required", (long long)p);
      return REC_E_INVALID_ARG;
    }
  }
  REC_CUDA(cudaSetDevice(m->device));
  if (m->world > 1 && m->shard != REC_SHARD_REPLICA)
    return serve_sharded(m, trace, n, sla_ms, pol, out, latency_ms, batch_log, log_cap, log_rows, ctr_out);
  const int M = pol->streams;
  const int32_t d = pol->max_batch;
  const bool virt = pol->clock == REC_CLOCK_VIRTUAL;
  const double tau = pol->fusion_timeout_ms * 1e-3;

  HostInputs H;
  if (pol->input_mode == REC_INPUT_HOST) {
    rec_status st = build_host_inputs(m, trace, n, H);
    if (st != REC_OK) return st;
  }
  std::vector<int64_t> item_base;
  if (ctr_out) {
    item_base.resize(n);
    int64_t acc = 0;
    for (int64_t p = 0; p < n; ++p) {
      item_base[p] = acc;
      acc += trace[p].size;
    }
  }
  std::vector<Lane> lanes(M);
  for (int s = 0; s < M; ++s) {
    REC_CUDA(cudaEventCreateWithFlags(&lanes[s].done, cudaEventDisableTiming));
    if (pol->input_mode == REC_INPUT_HOST)
      for (auto& e : lanes[s].hev) REC_CUDA(cudaEventCreate(&e));
    if (ctr_out)
      REC_CUDA(cudaMallocHost(reinterpret_cast<void**>(&lanes[s].ctr_host), sizeof(float) * d * m->tasks));
    if (!virt) {  // host-mapped completion word (falls back to event polling if unavailable)
      void* hp = nullptr;
      void* dp = nullptr;
      if (cudaHostAlloc(&hp, 64, cudaHostAllocMapped) == cudaSuccess &&
          cudaHostGetDevicePointer(&dp, hp, 0) == cudaSuccess &&
          stream_write_u32(m->ws[s].stream, reinterpret_cast<CUdeviceptr>(dp), 0) == REC_OK &&
          cudaStreamSynchronize(m->ws[s].stream) == cudaSuccess) {
        lanes[s].flag_host = static_cast<uint32_t*>(hp);
        lanes[s].flag_dev = reinterpret_cast<CUdeviceptr>(dp);
      } else {
        cudaGetLastError();
        if (hp) cudaFreeHost(hp);
      }
    }
  }
  // latency breakdown while profiling is on (rec_profile): the synthetic graphs with
  // stage events / host-mode lane events.  Off by default: per-batch event nodes and their
  // read-back cost serving throughput (measured: RMC1 lambda* 317k -> 206k QPS)
  const bool breakdown = m->prof;
  const bool synth_events = breakdown && m->ws[0].slots[0].var[1].exec != nullptr;
  // during serving the stage events are read per batch here; the profile counters (which
  // would read them again when a staging slot is reused) stay off
  struct ProfGuard {  // restores the profiling state on every return path
    rec_model_s* m;
    bool prof;
    ~ProfGuard() {
      m->prof = prof;
      m->stage_events = false;
    }
  } prof_guard{m, m->prof};
  if (breakdown) {
    for (auto& w : m->ws) REC_CUDA(cudaStreamSynchronize(w.stream));
    m->prof = false;
    m->stage_events = synth_events;
  }
  auto cleanup = [&]() {
    for (auto& L : lanes) {
      if (L.done) cudaEventDestroy(L.done);
      if (L.ctr_host) cudaFreeHost(L.ctr_host);
      if (L.flag_host) cudaFreeHost(L.flag_host);
      for (auto e : L.hev)
        if (e) cudaEventDestroy(e);
    }
  };
  std::vector<double> comp[3];
  for (auto& c : comp) c.assign(n, 0.0);

  std::vector<Chunk> fifo;
  fifo.reserve(static_cast<size_t>(n) * 2);
  std::vector<int32_t> remaining(n);
  for (int64_t p = 0; p < n; ++p) remaining[p] = (trace[p].size + d - 1) / d;
  std::vector<double> done_t(n, NAN), release(n), disp_t(n, NAN);
  std::vector<Batch> batches;
  std::vector<int32_t> segbuf;
  int64_t head = 0, a = 0, completed = 0, logged = 0;
  const double t_first = trace[0].arrival_s;

  // virtual clock: heap of (completion time, stream, batch)
  using VEv = std::tuple<double, int, int64_t>;
  std::priority_queue<VEv, std::vector<VEv>, std::greater<VEv>> vbusy;
  std::vector<int> idle;
  for (int s = 0; s < M; ++s) idle.push_back(s);

  auto finish_batch = [&](int64_t bi, double t_c) {
    Batch& bt = batches[bi];
    bt.t_done = t_c;
    double st[3] = {0, 0, 0};
    if (breakdown && pol->input_mode == REC_INPUT_HOST) stage_times(lanes[bt.stream].hev, true, bt.host_in_ms, st);
    else if (synth_events && bt.slot >= 0) stage_times(m->ws[bt.stream].slots[bt.slot].ev, false, 0.0, st);
    for (int64_t c = bt.first_chunk; c < bt.first_chunk + bt.nchunks; ++c) {
      const Chunk& ch = fifo[c];
      if (--remaining[ch.pos] == 0) {
        done_t[ch.pos] = t_c;
        for (int k = 0; k < 3; ++k) comp[k][ch.pos] = st[k];
        ++completed;
      }
    }
    if (ctr_out) {
      const float* src = lanes[bt.stream].ctr_host;
      int row = 0;
      for (int64_t c = bt.first_chunk; c < bt.first_chunk + bt.nchunks; ++c) {
        const Chunk& ch = fifo[c];
        memcpy(ctr_out + (item_base[ch.pos] + ch.start) * m->tasks, src + int64_t(row) * m->tasks,
               sizeof(float) * ch.len * m->tasks);
        row += ch.len;
      }
    }
  };

  auto dispatch = [&](int s, double t_now, int64_t k, int64_t items) -> rec_status {
    Workspace& w = m->ws[s];
    const int64_t bi = static_cast<int64_t>(batches.size());
    batches.push_back(Batch{s, head, k, items, t_now, 0});
    int B = 0;
    rec_status st;
    if (pol->input_mode == REC_INPUT_DEVICE_SYNTH) {
      segbuf.resize(3 * k);
      for (int64_t c = 0; c < k; ++c) {
        segbuf[3 * c] = fifo[head + c].qid;
        segbuf[3 * c + 1] = fifo[head + c].start;
        segbuf[3 * c + 2] = fifo[head + c].len;
      }
      st = synth_submit(m, w, segbuf.data(), static_cast<int>(k), &B, nullptr);  // a2-a6
      if (st != REC_OK) return st;
      batches[bi].slot = w.last_slot;
    } else {
      const double h0 = now_s();
      if (breakdown) REC_CUDA(cudaEventRecord(lanes[s].hev[0], w.stream));
      st = host_input_enqueue(m, w, H, fifo, head, k, &B);
      if (st != REC_OK) return st;
      batches[bi].host_in_ms = (now_s() - h0) * 1e3;
      if (breakdown) REC_CUDA(cudaEventRecord(lanes[s].hev[1], w.stream));
      st = forward_enqueue(m, w, w.indices, w.offsets, B, nullptr, w.ctr, w.logit,
                           breakdown ? lanes[s].hev : nullptr, w.idx_cap);
      if (st != REC_OK) return st;
    }
    if (ctr_out)
      REC_CUDA(cudaMemcpyAsync(lanes[s].ctr_host, w.ctr, sizeof(float) * B * m->tasks,
                               cudaMemcpyDeviceToHost, w.stream));
    REC_CUDA(cudaEventRecord(lanes[s].done, w.stream));
    lanes[s].busy = true;
    lanes[s].batch = bi;
    for (int64_t c = head; c < head + k; ++c) disp_t[fifo[c].pos] = t_now;
    if (batch_log && logged < log_cap) {
      for (int64_t c = head; c < head + k && logged < log_cap; ++c, ++logged) {
        int32_t* r = batch_log + 5 * logged;
        r[0] = static_cast<int32_t>(bi);
        r[1] = s;
        r[2] = fifo[c].qid;
        r[3] = fifo[c].start;
        r[4] = fifo[c].len;
      }
    }
    head += k;
    return REC_OK;
  };

  // fire condition (S2 with timeout, R15); times are in trace coordinates (arrival_s)
  auto should_fire = [&](double t_now, int64_t k, int64_t items) {
    if (tau <= 0) return true;
    const bool full = items == d || head + k < static_cast<int64_t>(fifo.size());
    return full || t_now >= trace[fifo[head].pos].arrival_s + tau;
  };

  rec_status st = REC_OK;
  if (virt) {
    double now = t_first;  // virtual clock in trace coordinates (same arithmetic as S4)
    while (true) {
      while (a < n && trace[a].arrival_s <= now) {
        split_query(trace[a], a, d, fifo);
        release[a] = trace[a].arrival_s;
        ++a;
      }
      while (!vbusy.empty() && std::get<0>(vbusy.top()) <= now) {
        auto [t_c, s, bi] = vbusy.top();
        vbusy.pop();
        st = rec_sync(m, s);
        if (st != REC_OK) { cleanup(); return st; }
        finish_batch(bi, t_c);
        lanes[s].busy = false;
        idle.push_back(s);
        std::sort(idle.begin(), idle.end());
      }
      while (!idle.empty() && head < static_cast<int64_t>(fifo.size())) {
        int64_t items = 0;
        const int64_t k = fuse_head(fifo, head, d, &items);
        if (!should_fire(now, k, items)) break;
        const int s = idle.front();
        idle.erase(idle.begin());
        const int64_t bi = static_cast<int64_t>(batches.size());
        st = dispatch(s, now, k, items);
        if (st != REC_OK) { cleanup(); return st; }
        vbusy.push(VEv{now + (pol->alpha_ns + pol->beta_ns * static_cast<double>(items)) * 1e-9, s, bi});
      }
      double nxt = INFINITY;
      if (a < n) nxt = std::min(nxt, trace[a].arrival_s);
      if (!vbusy.empty()) nxt = std::min(nxt, std::get<0>(vbusy.top()));
      if (tau > 0 && head < static_cast<int64_t>(fifo.size()) && !idle.empty())
        nxt = std::min(nxt, trace[fifo[head].pos].arrival_s + tau);
      if (!std::isfinite(nxt)) break;
      if (!(nxt > now)) {
        set_error("virtual clock made no progress");
        cleanup();
        return REC_E_INVALID_ARG;
      }
      now = nxt;
    }
  } else {
    // Real clock: trace time t maps to wall time t0 + (t - t_first).  This thread releases
    // arrivals open-loop into the FIFO; one dispatcher thread per co-located stream takes a
    // fused batch whenever its stream is idle (work-conserving, S2/S3), submits it, and
    // detects completion by polling a host-mapped sequence word the stream writes after
    // the batch (no CUDA API call on the polling path).  The FIFO, the batch list and the
    // per-query counters are shared under one mutex.
    std::mutex mu;
    std::atomic<int64_t> avail{0}, head_a{0};  // lock-free "is there work" hint
    std::atomic<int64_t> done_q{0};
    std::atomic<bool> failed{false};
    std::atomic<int> fail_status{REC_OK};
    const double t0 = now_s() - t_first;
    // Dispatcher threads: ONE thread polls every stream's mapped completion word and submits
    // (streams s = t, t + nthreads, ...).  Measured (scripts/serve_probe.py, RMC1, m = 8):
    // 1 thread sustains 305k QPS, 2 threads 288k, 8 threads 277k — concurrent graph launches
    // from several host threads contend inside the CUDA driver.  REC_SERVE_THREADS overrides.
    // Host-input mode: each batch's inputs are packed into pinned staging on the
    // host (megabytes per batch), so packing, not graph launching, bounds a single thread —
    // one dispatcher thread per stream (at most 8) packs in parallel.
    int nthreads = pol->input_mode == REC_INPUT_HOST ? std::min(M, 8) : 1;
    if (const char* e = getenv("REC_SERVE_THREADS")) nthreads = std::max(1, std::min(M, atoi(e)));
    struct Own {
      uint32_t seq = 0;
      int64_t my_batch = -1;
      std::deque<std::pair<int64_t, uint32_t>> pend;  // (batch, sequence word) in flight
    };
    std::vector<Own> own(M);
    // batches in flight per stream: 1 = the paper's co-located instance (one batch at a time);
    // 2 lets the next fused batch wait in the stream queue so the GPU never idles between a
    // completion and the host's next submit (REC_SERVE_DEPTH; needs the mapped completion word
    // and no CTR read-back, whose staging buffer is per stream)
    int depth = 1;
    if (const char* e = getenv("REC_SERVE_DEPTH")) depth = std::max(1, std::min(4, atoi(e)));
    if (ctr_out || !lanes[0].flag_host || pol->input_mode == REC_INPUT_HOST) depth = 1;  // per-lane staging
    auto worker = [&](int tid) {
      cudaSetDevice(m->device);
      std::vector<int32_t> segs_local;
      int idle_polls = 0;
      while (done_q.load(std::memory_order_relaxed) < n && !failed.load(std::memory_order_relaxed)) {
        bool progressed = false;
        for (int s = tid; s < M; s += nthreads) {
          Workspace& w = m->ws[s];
          Lane& L = lanes[s];
          Own& O = own[s];
          if (!O.pend.empty()) {
            if (L.flag_host) {
              const uint32_t done_seq = *reinterpret_cast<volatile uint32_t*>(L.flag_host);
              while (!O.pend.empty() && static_cast<int32_t>(done_seq - O.pend.front().second) >= 0) {
                const double t_c = now_s() - t0;
                std::lock_guard<std::mutex> g(mu);
                finish_batch(O.pend.front().first, t_c);
                done_q.store(completed, std::memory_order_relaxed);
                O.pend.pop_front();
                progressed = true;
              }
            } else if (cudaEventQuery(L.done) == cudaSuccess) {
              const double t_c = now_s() - t0;
              std::lock_guard<std::mutex> g(mu);
              finish_batch(O.pend.front().first, t_c);
              done_q.store(completed, std::memory_order_relaxed);
              O.pend.pop_front();
              progressed = true;
            }
            L.busy = !O.pend.empty();
            if (static_cast<int>(O.pend.size()) >= depth) continue;
          }
          int64_t k = 0, items = 0, c0 = 0;
          if (avail.load(std::memory_order_acquire) <= head_a.load(std::memory_order_acquire)) continue;
          {
            std::lock_guard<std::mutex> g(mu);
            if (head >= static_cast<int64_t>(fifo.size())) continue;
            k = fuse_head(fifo, head, d, &items);
            const double tn = now_s() - t0;
            if (!should_fire(tn, k, items)) continue;
            c0 = head;
            O.my_batch = static_cast<int64_t>(batches.size());
            batches.push_back(Batch{s, head, k, items, tn, 0});
            segs_local.resize(3 * k);
            for (int64_t c = 0; c < k; ++c) {
              const Chunk& ch = fifo[head + c];
              segs_local[3 * c] = ch.qid;
              segs_local[3 * c + 1] = ch.start;
              segs_local[3 * c + 2] = ch.len;
              disp_t[ch.pos] = tn;
              if (batch_log && logged < log_cap) {
                int32_t* r = batch_log + 5 * logged++;
                r[0] = static_cast<int32_t>(O.my_batch);
                r[1] = s;
                r[2] = ch.qid;
                r[3] = ch.start;
                r[4] = ch.len;
              }
            }
            head += k;
            head_a.store(head, std::memory_order_release);
          }
          int B = 0;
          rec_status rs;
          if (pol->input_mode == REC_INPUT_DEVICE_SYNTH) {
            rs = synth_submit(m, w, segs_local.data(), static_cast<int>(k), &B, nullptr);
            std::lock_guard<std::mutex> g(mu);
            batches[O.my_batch].slot = w.last_slot;
          } else {
            std::vector<Chunk> local(k);
            {
              std::lock_guard<std::mutex> g(mu);
              for (int64_t c = 0; c < k; ++c) local[c] = fifo[c0 + c];
            }
            const double h0 = now_s();
            if (breakdown) cudaEventRecord(L.hev[0], w.stream);
            rs = host_input_enqueue(m, w, H, local, 0, k, &B);
            const double hin = (now_s() - h0) * 1e3;
            if (breakdown) cudaEventRecord(L.hev[1], w.stream);
            if (rs == REC_OK)
              rs = forward_enqueue(m, w, w.indices, w.offsets, B, nullptr, w.ctr, w.logit,
                                   breakdown ? L.hev : nullptr, w.idx_cap);
            std::lock_guard<std::mutex> g(mu);
            batches[O.my_batch].host_in_ms = hin;
          }
          if (rs == REC_OK && ctr_out)
            if (cudaMemcpyAsync(L.ctr_host, w.ctr, sizeof(float) * B * m->tasks, cudaMemcpyDeviceToHost,
                                w.stream) != cudaSuccess)
              rs = REC_E_CUDA;
          if (rs == REC_OK) {
            ++O.seq;
            if (L.flag_host) {
              if (stream_write_u32(w.stream, L.flag_dev, O.seq) != REC_OK) rs = REC_E_CUDA;
            } else if (cudaEventRecord(L.done, w.stream) != cudaSuccess) {
              rs = REC_E_CUDA;
            }
          }
          if (rs != REC_OK) {
            fail_status.store(rs);
            failed.store(true);
            return;
          }
          O.pend.emplace_back(O.my_batch, O.seq);
          L.busy = true;
          progressed = true;
        }
        if (progressed) {
          idle_polls = 0;
        } else if (++idle_polls > 64) {
          std::this_thread::yield();  // batches in flight, nothing queued: let others run
        } else {
          cpu_relax();
        }
      }
    };
    std::vector<std::thread> th;
    for (int t = 0; t < nthreads; ++t) th.emplace_back(worker, t);
    while (a < n && !failed.load()) {
      const double now = now_s() - t0;
      if (trace[a].arrival_s > now) {  // open-loop release: spin until the next arrival
        cpu_relax();
        continue;
      }
      std::lock_guard<std::mutex> g(mu);
      while (a < n && trace[a].arrival_s <= now) {
        split_query(trace[a], a, d, fifo);
        release[a] = trace[a].arrival_s;
        ++a;
      }
      avail.store(static_cast<int64_t>(fifo.size()), std::memory_order_release);
    }
    for (auto& t : th) t.join();
    if (failed.load()) {
      cleanup();
      return static_cast<rec_status>(fail_status.load());
    }
  }
  for (int s = 0; s < M; ++s) {
    st = rec_sync(m, s);
    if (st != REC_OK) { cleanup(); return st; }
  }
  cleanup();

  // ------------------------------------------------ report (S5)
  double items_tot = 0;
  for (auto& b : batches) items_tot += b.items;
  rec_model_s* gm = m->world > 1 && m->shard == REC_SHARD_REPLICA && m->nccl_comm ? m : nullptr;
  fill_report(trace, n, sla_ms, pol->warmup_frac, release, disp_t, done_t, completed,
              static_cast<int64_t>(batches.size()), items_tot, latency_ms, out,
              breakdown ? comp : nullptr, gm);
  if (log_rows) *log_rows = logged;
  return REC_OK;
}

}  // extern "C"
