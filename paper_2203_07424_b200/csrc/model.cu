// model.cu — rec_model_create/destroy, rec_query*, rec_gen_batch, profiling (include/rec.h).
//
// Host side of the hot path: validates the model description (Table I shapes),
// allocates the fp32 embedding arena and bf16 MLP weights on the device, generates every
// parameter there from the seed (G4/G5), encodes the TMA tensor maps of every GEMM operand
// once, and enqueues the per-batch kernel chain  [input] -> SLS -> bottom GEMMs ->
// interaction -> top GEMMs (+ width-1 layer + sigmoid)  on one CUDA stream per co-located
// "inference thread" (model co-location).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>

#include <cuda.h>

#include "common.cuh"
#include "model.h"

// ------------------------------------------------------------------ SM partitions
// REC_GREEN_SMS=n (experiment): the dense stages (dense features, bottom, interaction, top)
// run on streams of a green context holding n SMs, the SLS on the remaining SMs, so no SM
// hosts both (DESIGN.md §6 co-location).  Driver entry points are resolved at run time.
template <typename F>
static F drv_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<F>(p);
}
static bool green_setup(int device, int n_dense, void** out) {  // out[4]: 2 CUgreenCtx + 2 CUcontext
  auto getdev = drv_fn<decltype(&cuDeviceGet)>("cuDeviceGet");
  auto getres = drv_fn<decltype(&cuDeviceGetDevResource)>("cuDeviceGetDevResource");
  auto split = drv_fn<decltype(&cuDevSmResourceSplitByCount)>("cuDevSmResourceSplitByCount");
  auto gen = drv_fn<decltype(&cuDevResourceGenerateDesc)>("cuDevResourceGenerateDesc");
  auto create = drv_fn<decltype(&cuGreenCtxCreate)>("cuGreenCtxCreate");
  if (!getdev || !getres || !split || !gen || !create) return false;
  CUdevice dev;
  if (getdev(&dev, device) != CUDA_SUCCESS) return false;
  CUdevResource all{}, part[1]{}, rest{};
  unsigned nb = 1;
  if (getres(dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS) return false;
  if (split(part, &nb, &all, &rest, 0, static_cast<unsigned>(n_dense)) != CUDA_SUCCESS || nb != 1) return false;
  CUdevResourceDesc dd, ds;
  if (gen(&dd, part, 1) != CUDA_SUCCESS || gen(&ds, &rest, 1) != CUDA_SUCCESS) return false;
  CUgreenCtx g0, g1;
  if (create(&g0, dd, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS) return false;
  if (create(&g1, ds, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS) return false;
  out[0] = g0;
  out[1] = g1;
  auto toctx = drv_fn<decltype(&cuCtxFromGreenCtx)>("cuCtxFromGreenCtx");
  CUcontext c0, c1;
  if (!toctx || toctx(&c0, g0) != CUDA_SUCCESS || toctx(&c1, g1) != CUDA_SUCCESS) return false;
  out[2] = c0;
  out[3] = c1;
  if (getenv("REC_VERBOSE"))
    fprintf(stderr, "[rec] SM partition: dense %u SMs, SLS %u SMs\n", part[0].sm.smCount, rest.sm.smCount);
  return true;
}
// Kernel-node update of a graph node captured on a green-context stream: the runtime update
// would name the primary context, so the driver call carries the kernel handle and the
// partition's context.
static cudaError_t green_node_update(cudaGraphExec_t exec, cudaGraphNode_t node, void* ctx,
                                     const cudaKernelNodeParams& kp) {
  static auto upd = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuGraphExecKernelNodeSetParams", &p, 12000, cudaEnableDefault, &q) !=
            cudaSuccess || q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<CUresult (*)(CUgraphExec, CUgraphNode, const CUDA_KERNEL_NODE_PARAMS_v2*)>(p);
  }();
  if (!upd) return cudaErrorNotSupported;
  CUDA_KERNEL_NODE_PARAMS_v2 p{};
  cudaKernel_t k;
  cudaError_t e = cudaGetKernel(&k, kp.func);
  if (e != cudaSuccess) return e;
  p.func = nullptr;
  p.kern = reinterpret_cast<CUkernel>(k);
  p.ctx = static_cast<CUcontext>(ctx);
  p.gridDimX = kp.gridDim.x;
  p.gridDimY = kp.gridDim.y;
  p.gridDimZ = kp.gridDim.z;
  p.blockDimX = kp.blockDim.x;
  p.blockDimY = kp.blockDim.y;
  p.blockDimZ = kp.blockDim.z;
  p.sharedMemBytes = kp.sharedMemBytes;
  p.kernelParams = kp.kernelParams;
  return upd(reinterpret_cast<CUgraphExec>(exec), reinterpret_cast<CUgraphNode>(node), &p) == CUDA_SUCCESS
             ? cudaSuccess
             : cudaErrorInvalidValue;
}
static bool green_stream(void* g, cudaStream_t* s) {
  auto mk = drv_fn<decltype(&cuGreenCtxStreamCreate)>("cuGreenCtxStreamCreate");
  CUstream cs;
  if (!mk || mk(&cs, static_cast<CUgreenCtx>(g), CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS) return false;
  *s = reinterpret_cast<cudaStream_t>(cs);
  return true;
}

namespace rec {

static thread_local std::string g_err;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
}

rec_status cuda_fail(cudaError_t e, const char* what) {
  set_error("CUDA error %s (%s) in %s", cudaGetErrorName(e), cudaGetErrorString(e), what);
  return REC_E_CUDA;
}

static int pad8(int x) { return (x + 7) & ~7; }

static bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

cudaEvent_t prof_begin(rec_model_s* m, cudaStream_t s) {
  if (!m->prof) return nullptr;
  cudaEvent_t a;
  if (!m->prof_pool.empty()) {
    a = m->prof_pool.back();
    m->prof_pool.pop_back();
  } else {
    cudaEventCreate(&a);
  }
  cudaEventRecord(a, s);
  return a;
}

void prof_end(rec_model_s* m, cudaStream_t s, int kernel, cudaEvent_t a) {
  if (!a) return;
  cudaEvent_t b;
  if (!m->prof_pool.empty()) {
    b = m->prof_pool.back();
    m->prof_pool.pop_back();
  } else {
    cudaEventCreate(&b);
  }
  cudaEventRecord(b, s);
  m->prof_events.push_back(ProfEvent{kernel, a, b});
}

static void collect_slot(rec_model_s* m, SynthSlot& sl);

static void prof_collect(rec_model_s* m) {
  for (auto& w : m->ws)
    for (auto& sl : w.slots) collect_slot(m, sl);
  for (auto& e : m->prof_events) {
    cudaEventSynchronize(e.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e.a, e.b);
    m->prof_ms[e.kernel] += ms;
    m->prof_n[e.kernel] += 1;
    m->prof_pool.push_back(e.a);
    m->prof_pool.push_back(e.b);
  }
  m->prof_events.clear();
}

// ------------------------------------------------------------------ forward chain
// Stage helpers.  B = batch, or the workspace capacity when dB != nullptr (then every kernel
// reads the batch from *dB: the form captured in CUDA graphs).  gev != nullptr: graph capture
// with stage events recorded as external event nodes; else per-kernel profiling events.
//   gev: 0 chain start, 1 inputs done, 2 SLS done, 3 join, 4 interaction done, 5 top done,
//        6/7 bottom-branch start/end (the branch stream)
static inline void mark(cudaEvent_t* gev, int i, cudaStream_t st) {
  if (!gev) return;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  // inside a capture: an external event node of the graph; outside (host-input serving with
  // stage events): a plain record
  if (cs == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(gev[i], st, cudaEventRecordExternal);
  else cudaEventRecord(gev[i], st);
}

void enqueue_bottom(rec_model_s* m, Workspace& w, cudaStream_t st, int B, const int* dB,
                    cudaEvent_t* gev) {
  const int T = m->T, D = m->D;
  const int nb = static_cast<int>(m->bottom.size());
  if (nb == 0) return;    // MT-WnD: no Bottom-FC
  if (m->chain_bottom) {  // whole bottom MLP in one kernel (k_mlp.cu)
    ChainArgs a = m->chain_bottom_args;
    a.M = B;
    a.dM = dB;
    a.out_f32 = w.X;
    a.ldo = (T + 1) * D;
    cudaEvent_t e = gev ? nullptr : prof_begin(m, st);
    launch_mlp_chain(w.chain_bottom, a, st);
    prof_end(m, st, 1, e);
    m->launches += 1;
    return;
  }
  for (int l = 0; l < nb; ++l) {
    const Layer& L = m->bottom[l];
    GemmArgs a{};
    a.M = B;
    a.dM = dB;
    a.N = L.N;
    a.K = L.K;
    a.bias = L.bias;
    a.relu = 1;
    if (l == nb - 1) {
      a.mode = GEMM_OUT_X_F32;
      a.out_f32 = w.X;
      a.ldo = (T + 1) * D;
    } else {
      a.mode = GEMM_OUT_BF16;
      a.out_bf16 = static_cast<__nv_bfloat16*>(w.out_bottom[l]);
      a.ldo = L.Npad;
    }
    cudaEvent_t e = gev ? nullptr : prof_begin(m, st);
    launch_gemm_tc(&w.tmap_a_bottom[l], &L.tmap_w, a, st, &L.tmap_w128, &L.tmap_w64);
    prof_end(m, st, 1, e);
  }
  m->launches += nb;
}

void enqueue_interact_top(rec_model_s* m, Workspace& w, cudaStream_t st, int B, const int* dB,
                          float* ctr_out, float* logit_out, cudaEvent_t* gev) {
  const int T = m->T, D = m->D;
  if (m->arch == REC_ARCH_MTWND) {  // concat + wide part, then one tower per task
    cudaEvent_t e1 = gev ? nullptr : prof_begin(m, st);
    launch_concat(w.X, B, dB, T, D, w.A_top, m->Ktop_pad, m->wide_v, m->tasks, w.wide, st);
    prof_end(m, st, 2, e1);
    mark(gev, 4, st);
    const int nt = static_cast<int>(m->top.size());
    // the same layer of up to kMaxGroup towers in ONE grouped launch (grid.z = task)
    const int gmax = m->tower_group ? kMaxGroup : 1;
    for (int k0 = 0; k0 < m->tasks; k0 += gmax) {
    const int kn = std::min(gmax, m->tasks - k0);
    for (int j = 0; j < nt; ++j) {
      GemmGroup grp;
      grp.n = kn;
      for (int k = k0; k < k0 + kn; ++k) {
        const std::vector<Layer>& Ls = k == 0 ? m->top : m->towers[k - 1];
        const Layer& L = Ls[j];
        GemmArgs a{};
        a.M = B;
        a.dM = dB;
        a.N = L.N;
        a.K = L.K;
        a.bias = L.bias;
        a.relu = 1;
        if (j == nt - 1) {
          a.mode = GEMM_OUT_CTR;
          a.w_last = k == 0 ? m->w_last : m->w_last_t[k - 1];
          a.b_last = k == 0 ? m->b_last : m->b_last_t[k - 1];
          a.ctr = ctr_out + k;
          a.logit = logit_out ? logit_out + k : nullptr;
          a.ctr_stride = m->tasks;
          a.logit_add = w.wide + k;
          a.add_stride = m->tasks;
        } else {
          a.mode = GEMM_OUT_BF16;
          a.out_bf16 = static_cast<__nv_bfloat16*>(k == 0 ? w.out_top[j] : w.out_task[k][j]);
          a.ldo = L.Npad;
        }
        grp.ta[k - k0] = k == 0 ? w.tmap_a_top[j] : w.tmap_a_task[k][j];
        grp.tw[k - k0] = L.tmap_w;
        grp.tw_half[k - k0] = L.tmap_w128;
        grp.a[k - k0] = a;
      }
      cudaEvent_t e = gev ? nullptr : prof_begin(m, st);
      launch_gemm_group(grp, st);
      prof_end(m, st, 1, e);
    }
    }
    mark(gev, 5, st);
    m->launches += 1 + ((m->tasks + gmax - 1) / gmax) * nt;
    return;
  }
  // a5: interaction -> A_top
  cudaEvent_t e1 = gev ? nullptr : prof_begin(m, st);
  const bool fused = m->chain_top && m->fuse_interact;
  if (!(m->diag_skip & 4) && !fused) launch_interact(w.X, B, dB, T, D, w.A_top, m->Ktop_pad, st);
  prof_end(m, st, 2, e1);
  mark(gev, 4, st);
  // a6: top MLP; the last hidden layer's epilogue applies the width-1 layer + sigmoid
  const int nt = static_cast<int>(m->top.size());
  if (m->chain_top) {  // whole top MLP in one kernel (k_mlp.cu)
    ChainArgs a = m->chain_top_args;
    // PDL only behind k_interact (it never writes *dB, which the chain reads before its
    // grid-dependency wait; see k_mlp_chain); the fused-interaction chain has no such
    // predecessor and launches plainly
    a.pdl = m->chain_pdl && !fused;
    a.M = B;
    a.dM = dB;
    a.ctr = ctr_out;
    a.logit = logit_out;
    if (fused) {
      a.ix = w.X;
      a.ir = T + 1;
    }
    cudaEvent_t e = gev ? nullptr : prof_begin(m, st);
    launch_mlp_chain(w.chain_top, a, st);
    prof_end(m, st, 1, e);
    mark(gev, 5, st);
    m->launches += fused ? 1 : 2;
    return;
  }
  for (int j = 0; j < nt; ++j) {
    const Layer& L = m->top[j];
    GemmArgs a{};
    a.M = B;
    a.dM = dB;
    a.N = L.N;
    a.K = L.K;
    a.bias = L.bias;
    a.relu = 1;
    if (j == nt - 1) {
      a.mode = GEMM_OUT_CTR;
      a.w_last = m->w_last;
      a.b_last = m->b_last;
      a.ctr = ctr_out;
      a.logit = logit_out;
    } else {
      a.mode = GEMM_OUT_BF16;
      a.out_bf16 = static_cast<__nv_bfloat16*>(w.out_top[j]);
      a.ldo = L.Npad;
    }
    cudaEvent_t e = gev ? nullptr : prof_begin(m, st);
    launch_gemm_tc(&w.tmap_a_top[j], &L.tmap_w, a, st, &L.tmap_w128, &L.tmap_w64);
    prof_end(m, st, 1, e);
  }
  mark(gev, 5, st);
  m->launches += 1 + nt;
}

// Forward over materialised inputs (w.indices / caller arrays).  The bottom MLP (a4)
// depends only on the dense features and the SLS (a3) only on the sparse ones: they run on
// two streams (a fork in a captured graph) and join before the interaction (a5).
rec_status forward_enqueue(rec_model_s* m, Workspace& w, const int* indices, const int* offsets,
                           int B, const int* dB, float* ctr_out, float* logit_out, cudaEvent_t* gev,
                           int64_t idx_limit) {
  cudaStream_t s = w.stream, sb = w.stream_b;
  REC_CUDA(cudaEventRecord(w.ev_fork, s));
  REC_CUDA(cudaStreamWaitEvent(sb, w.ev_fork, 0));
  mark(gev, 6, sb);
  enqueue_bottom(m, w, sb, B, dB, gev);
  mark(gev, 7, sb);
  REC_CUDA(cudaEventRecord(w.ev_join, sb));
  if (m->d_remap) {  // hot-row partition: caller / materialised ids -> arena rows
    launch_remap(indices, offsets, B, dB, m->T, m->d_rows, m->d_remap, m->d_remap_off, w.indices,
                 w.idx_cap, w.flag, s);
    m->launches += 1;
    indices = w.indices;
    idx_limit = std::min<int64_t>(idx_limit, w.idx_cap);
  }
  cudaEvent_t e0 = gev ? nullptr : prof_begin(m, s);
  launch_sls(m->tables, m->d_tab_off, m->row_stride, m->d_rows, indices, offsets, B, dB, m->T, m->D,
             w.X, (m->T + 1) * m->D, 1, w.flag, s, 0, 0x7fffffff,
             static_cast<int>(std::min<int64_t>(idx_limit, 0x7fffffff)));
  prof_end(m, s, 0, e0);
  m->launches += 1;
  mark(gev, 2, s);
  REC_CUDA(cudaStreamWaitEvent(s, w.ev_join, 0));  // join
  mark(gev, 3, s);
  enqueue_interact_top(m, w, s, B, dB, ctr_out, logit_out, gev);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return cuda_fail(err, "forward kernel launch");
  return REC_OK;
}

static rec_status wait_pin(Workspace& w) {
  REC_CUDA(cudaEventSynchronize(w.pin_free));
  return REC_OK;
}

void fill_genargs(rec_model_s* m, Workspace& w, GenArgs& ga, SlsSynthArgs& sa,
                  float* dense_f32_out) {
  ga = GenArgs{};
  ga.cap = w.cap;
  ga.T = m->T;
  ga.lo = m->lo;
  ga.hi = m->hi;
  ga.index_dist = m->index_dist;
  ga.F = m->F;
  ga.Fpad = m->Fpad;
  ga.nbag_blocks = (m->T * w.cap + 7) / 8;
  ga.k0 = m->k0;
  ga.k1 = m->k1;
  ga.rows = m->d_rows;
  ga.offsets = w.offsets;
  ga.indices = w.indices;
  ga.dense_bf = w.dense_bf;
  ga.dense_f32 = dense_f32_out;
  ga.rowq = w.rowq;
  ga.rowi = w.rowi;
  ga.dB = w.dB;
  sa = SlsSynthArgs{};
  sa.tables = m->tables;
  sa.tab_off = m->d_tab_off;
  sa.row_stride = m->row_stride;
  sa.rows = m->d_rows;
  sa.cap = w.cap;
  sa.T = m->T;
  sa.D = m->D;
  sa.L = m->lo;
  sa.index_dist = m->index_dist;
  sa.k0 = m->k0;
  sa.k1 = m->k1;
  sa.X = w.X;
  sa.x_stride = (m->T + 1) * m->D;
  sa.dB = w.dB;
  sa.hot_rows = 0;
  if (m->l2_persist_bytes > 0 && m->interleaved && !(m->shard == REC_SHARD_ROW && m->world > 1))
    sa.hot_rows = static_cast<int>(std::min<int64_t>(
        m->l2_persist_bytes / (static_cast<int64_t>(m->T_loc) * m->D * 4), m->rows[m->t0]));
  {  // per-load hints are opt-in: measured slower than the window alone
    const char* e = getenv("REC_HOT_POLICY");
    if (!e || !atoi(e)) sa.hot_rows = 0;
  }
  // dense features from the SLS kernel only where it implements them (not the TMA variant)
  sa.dense_bf = m->fuse_dense && !m->sls_tma ? w.dense_bf : nullptr;
  sa.F = m->F;
  sa.Fpad = m->Fpad;
  sa.remap = m->d_remap;
  sa.remap_off = m->d_remap_off;
  sa.tma = m->d_remap ? 0 : m->sls_tma;  // (the TMA variant does not read the remap)
  sa.pdl = m->sls_pdl && !sa.tma;
  sa.tmap_rows = m->d_tmap_rows;
  sa.nsm = m->nsm;
  sa.interleave = m->sls_interleave;
  if (sa.tma) sls_tma_configure(sa);
}

const cudaGraphNode_t* last_node(cudaStream_t s, size_t* n) {
  cudaStreamCaptureStatus cs;
  const cudaGraphNode_t* deps = nullptr;
  if (cudaStreamGetCaptureInfo(s, &cs, nullptr, nullptr, &deps, n) != cudaSuccess) *n = 0;
  return deps;
}

// A device-synthesised batch described by the slot's SegBatch (a2-a6, CTRs into w.ctr).
//  * fused (fixed pooling, serving/bench path): branch stream = dense features -> bottom MLP;
//    main stream = SLS over Philox indices generated in-kernel; join -> interaction -> top.
//    Both first kernels take the batch by value, so a captured graph is re-targeted per batch
//    by two kernel-node parameter updates (no host->device copy).
//  * materialised (variable pooling, rec_gen_batch): input kernels write indices / offsets /
//    dense, then the generic forward.
static rec_status synth_chain(rec_model_s* m, Workspace& w, SynthSlot& sl, bool capture,
                              bool materialize, bool with_events = false) {
  cudaStream_t s = w.stream, sb = w.stream_b;
  cudaEvent_t* gev = capture && with_events ? sl.ev : nullptr;
  mark(gev, 0, s);
  if (!materialize && m->lo == m->hi && ((m->fuse_dense && !m->sls_tma) || m->F == 0)) {
    // dense features generated inside the SLS kernel: one stream, SLS -> bottom -> top
    mark(gev, 1, s);
    cudaEvent_t e0 = gev ? nullptr : prof_begin(m, s);
    launch_sls_synth(*sl.sb, sl.sa, s);
    prof_end(m, s, 0, e0);
    if (capture) {
      size_t n = 0;
      const cudaGraphNode_t* d = last_node(s, &n);
      if (n != 1) {
        set_error("graph capture: SLS node not found");
        return REC_E_CUDA;
      }
      *sl.cap_gen = d[0];
    }
    m->launches += 1;
    mark(gev, 2, s);
    mark(gev, 6, s);
    enqueue_bottom(m, w, s, w.cap, w.dB, gev);
    mark(gev, 7, s);
    mark(gev, 3, s);
    enqueue_interact_top(m, w, s, w.cap, w.dB, w.ctr, w.logit, gev);
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return cuda_fail(err, "synthetic chain launch");
    return REC_OK;
  }
  if (!materialize && m->lo == m->hi) {
    REC_CUDA(cudaEventRecord(w.ev_fork, s));
    REC_CUDA(cudaStreamWaitEvent(sb, w.ev_fork, 0));
    mark(gev, 6, sb);
    cudaEvent_t ed = gev ? nullptr : prof_begin(m, sb);
    launch_gen_dense_seg(*sl.sb, sl.ga, sb);
    prof_end(m, sb, 3, ed);
    if (capture) {
      size_t n = 0;
      const cudaGraphNode_t* d = last_node(sb, &n);
      if (n != 1) {
        set_error("graph capture: dense node not found");
        return REC_E_CUDA;
      }
      *sl.cap_dense = d[0];
    }
    if (!(m->diag_skip & 1)) enqueue_bottom(m, w, sb, w.cap, w.dB, gev);
    mark(gev, 7, sb);
    REC_CUDA(cudaEventRecord(w.ev_join, sb));
    mark(gev, 1, s);
    cudaEvent_t e0 = gev ? nullptr : prof_begin(m, s);
    launch_sls_synth(*sl.sb, sl.sa, s);
    prof_end(m, s, 0, e0);
    if (capture) {
      size_t n = 0;
      const cudaGraphNode_t* d = last_node(s, &n);
      if (n != 1) {
        set_error("graph capture: SLS node not found");
        return REC_E_CUDA;
      }
      *sl.cap_gen = d[0];
    }
    m->launches += 2;
    mark(gev, 2, s);
    if (m->green_sms > 0 && !(m->diag_skip & 2)) {
      // SM partitions: the join and the dense tail run on the dense partition's stream
      REC_CUDA(cudaEventRecord(w.ev_g1, s));
      REC_CUDA(cudaStreamWaitEvent(sb, w.ev_g1, 0));
      mark(gev, 3, sb);
      enqueue_interact_top(m, w, sb, w.cap, w.dB, w.ctr, w.logit, gev);
      REC_CUDA(cudaEventRecord(w.ev_g2, sb));
      REC_CUDA(cudaStreamWaitEvent(s, w.ev_g2, 0));
      cudaError_t err = cudaGetLastError();
      if (err != cudaSuccess) return cuda_fail(err, "synthetic chain launch");
      return REC_OK;
    }
    REC_CUDA(cudaStreamWaitEvent(s, w.ev_join, 0));
    mark(gev, 3, s);
    if (!(m->diag_skip & 2)) {
      enqueue_interact_top(m, w, s, w.cap, w.dB, w.ctr, w.logit, gev);
    } else {
      mark(gev, 4, s);
      mark(gev, 5, s);
    }
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return cuda_fail(err, "synthetic chain launch");
    return REC_OK;
  }
  cudaEvent_t e = gev ? nullptr : prof_begin(m, s);
  launch_gen_first(*sl.sb, sl.ga, s);
  if (capture) {
    size_t n = 0;
    const cudaGraphNode_t* d = last_node(s, &n);
    if (n != 1) {
      set_error("graph capture: input node not found");
      return REC_E_CUDA;
    }
    *sl.cap_gen = d[0];
  }
  if (m->lo != m->hi) {
    launch_gen_variable_rest(sl.ga, s);
    m->launches += 4;
  } else {
    m->launches += 1;
  }
  prof_end(m, s, 3, e);
  mark(gev, 1, s);
  if (m->world > 1 && m->shard != REC_SHARD_REPLICA) return REC_OK;  // inputs only (gen_batch)
  return forward_enqueue(m, w, w.indices, w.offsets, w.cap, w.dB, w.ctr, w.logit, gev, w.idx_cap);
}

rec_status capture_graphs(rec_model_s* m, Workspace& w) {
  for (auto& sl : w.slots) {
    for (int v = 0; v < 2; ++v) {  // 0: kernels only (production), 1: with stage events
      SynthSlot::Variant& V = sl.var[v];
      sl.cap_gen = &V.gen_node;
      sl.cap_dense = &V.dense_node;
      const int64_t before = m->launches;
      REC_CUDA(cudaStreamBeginCapture(w.stream, cudaStreamCaptureModeThreadLocal));
      rec_status st = synth_chain(m, w, sl, true, false, v == 1);
      cudaGraph_t g = nullptr;
      cudaError_t ce = cudaStreamEndCapture(w.stream, &g);
      if (st != REC_OK) return st;
      if (ce != cudaSuccess) return cuda_fail(ce, "cudaStreamEndCapture");
      V.graph = g;
      ce = cudaGraphInstantiate(&V.exec, g, cudaGraphInstantiateFlagUseNodePriority);
      if (ce != cudaSuccess) return cuda_fail(ce, "cudaGraphInstantiate");
      w.graph_kernels = static_cast<int>(m->launches - before);
      m->launches = before;
    }
  }
  return REC_OK;
}

static void collect_slot(rec_model_s* m, SynthSlot& sl) {
  if (!sl.prof_pending) return;
  float t[8] = {};
  auto el = [&](int a, int b) {
    float x = 0.f;
    cudaEventElapsedTime(&x, sl.ev[a], sl.ev[b]);
    return x;
  };
  // 0 inputs 1 | SLS 2 | branch 6 [dense gen] bottom 7 | join 3 | interact 4 | top 5
  t[0] = el(0, 1);
  t[1] = el(1, 2);
  t[2] = el(6, 7) + el(4, 5);
  t[3] = el(3, 4);
  m->prof_ms[3] += t[0];
  m->prof_ms[0] += t[1];
  m->prof_ms[1] += t[2];
  m->prof_ms[2] += t[3];
  m->prof_n[3] += 1;
  m->prof_n[0] += 1;
  m->prof_n[1] += static_cast<int64_t>(m->bottom.size() + m->top.size());
  m->prof_n[2] += 1;
  sl.prof_pending = false;
}

static inline double host_now_ns() {
  return std::chrono::duration<double, std::nano>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

// segs (host) -> a slot's batch descriptor -> graph launch (inputs + forward) on w.stream.
// dense_f32_out forces the direct (non-graph) path (rec_gen_batch needs the fp32 dense).
rec_status synth_submit(rec_model_s* m, Workspace& w, const int32_t* segs, int nseg, int* batch_out,
                        float* dense_f32_out) {
  if (nseg <= 0 || !segs) {
    set_error("segs: empty segment list");
    return REC_E_INVALID_ARG;
  }
  int64_t B = 0;
  for (int i = 0; i < nseg; ++i) {
    if (segs[3 * i + 2] <= 0 || segs[3 * i] < 0 || segs[3 * i + 1] < 0) {
      set_error("segs[%d]: qid/start must be >= 0 and len > 0", i);
      return REC_E_INVALID_ARG;
    }
    B += segs[3 * i + 2];
  }
  if (B > w.cap || nseg > w.cap) {
    set_error("segs: batch of %lld items exceeds max_batch %d", (long long)B, w.cap);
    return REC_E_INVALID_ARG;
  }
  if (m->pipe_active.load(std::memory_order_acquire)) {
    rec_status st = pipe_leave(m);
    if (st != REC_OK) return st;
  }
  const double t0 = host_now_ns();
  SynthSlot& sl = w.slots[w.next_slot];
  w.last_slot = w.next_slot;
  w.next_slot = (w.next_slot + 1) % static_cast<int>(w.slots.size());
  REC_CUDA(cudaEventSynchronize(sl.free));
  collect_slot(m, sl);
  const double t1 = host_now_ns();
  SegBatch& sb = *sl.sb;
  sb.B = static_cast<int>(B);
  sb.nseg = nseg;
  sb.gsegs = w.gsegs;
  int4* dst = sb.seg;
  if (nseg > kParamSegs) {  // long segment lists go through pinned staging + H2D
    rec_status st = wait_pin(w);
    if (st != REC_OK) return st;
    dst = reinterpret_cast<int4*>(w.pin);
  }
  int row = 0;
  for (int i = 0; i < nseg; ++i) {
    dst[i] = make_int4(segs[3 * i], segs[3 * i + 1], segs[3 * i + 2], row);
    row += segs[3 * i + 2];
  }
  if (nseg > kParamSegs)
    REC_CUDA(cudaMemcpyAsync(w.gsegs, w.pin, sizeof(int4) * nseg, cudaMemcpyHostToDevice, w.stream));
  if (m->p2p_slots) {  // table-wise sharded: this rank's item block + the slot's epoch
    shard_fill_local(m, w, sl, segs, nseg, static_cast<int>(B),
                     reinterpret_cast<int4*>(w.pin) + (w.cap + 1));
    sl.sa.p2p.epoch = ++w.sh_epoch;
    if (nseg > kParamSegs) REC_CUDA(cudaEventRecord(w.pin_free, w.stream));
  } else if (nseg > kParamSegs) {
    REC_CUDA(cudaEventRecord(w.pin_free, w.stream));
  }
  SynthSlot::Variant& V = sl.var[(m->prof || m->stage_events) && sl.var[1].exec ? 1 : 0];
  const bool direct = dense_f32_out != nullptr || !V.exec;
  if (!direct) {
    const bool fused = m->lo == m->hi;
    dim3 grid, block;
    cudaKernelNodeParams kp{};
    void* args_a[2] = {sl.sb, fused ? static_cast<void*>(&sl.sa) : static_cast<void*>(&sl.ga)};
    size_t smem = 0;
    kp.func = fused ? sls_synth_kernel(sl.sa, &grid, &block, &smem)
                    : gen_first_kernel(sl.ga, &grid, &block);
    kp.sharedMemBytes = static_cast<unsigned>(smem);
    kp.gridDim = grid;
    kp.blockDim = block;
    kp.kernelParams = args_a;
    if (m->green_sms > 0) REC_CUDA(green_node_update(V.exec, V.gen_node, m->green_cu[1], kp));
    else REC_CUDA(cudaGraphExecKernelNodeSetParams(V.exec, V.gen_node, &kp));
    if (fused && V.dense_node) {
      cudaKernelNodeParams kd{};
      void* args_d[2] = {m->p2p_slots ? sl.sb_local : sl.sb, &sl.ga};
      kd.func = gen_dense_seg_kernel(sl.ga, &grid, &block);
      kd.gridDim = grid;
      kd.blockDim = block;
      kd.kernelParams = args_d;
      if (m->green_sms > 0) REC_CUDA(green_node_update(V.exec, V.dense_node, m->green_cu[0], kd));
      else REC_CUDA(cudaGraphExecKernelNodeSetParams(V.exec, V.dense_node, &kd));
    }
    const double t2 = host_now_ns();
    REC_CUDA(cudaGraphLaunch(V.exec, w.stream));
    const double t3 = host_now_ns();
    w.host_ns[0] += t2 - t1;
    w.host_ns[1] += t3 - t2;
    w.host_ns[2] += t1 - t0;
    m->launches += w.graph_kernels;
    sl.prof_pending = m->prof;
  } else {
    GenArgs saved = sl.ga;
    sl.ga.dense_f32 = dense_f32_out;
    rec_status st = synth_chain(m, w, sl, false, dense_f32_out != nullptr);
    sl.ga = saved;
    if (st != REC_OK) return st;
  }
  REC_CUDA(cudaEventRecord(sl.free, w.stream));
  w.host_ns[3] += host_now_ns() - t0;
  *batch_out = static_cast<int>(B);
  return REC_OK;
}

static rec_status read_flag(Workspace& w) {
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
    set_error("a peer rank missed the sharded exchange deadline (REC_P2P_TIMEOUT_S)");
    return REC_E_NCCL;
  }
  return REC_OK;
}

static rec_status sync_ws(Workspace& w) {
  REC_CUDA(cudaMemcpyAsync(w.flag_host, w.flag, sizeof(int), cudaMemcpyDeviceToHost, w.stream));
  REC_CUDA(cudaMemsetAsync(w.flag, 0, sizeof(int), w.stream));
  REC_CUDA(cudaStreamSynchronize(w.stream));
  return read_flag(w);
}

// ------------------------------------------------------------------ query (sync)
static rec_status query_impl(rec_model_s* m, const float* dense, const int32_t* indices,
                             const int32_t* offsets, int32_t B, float* ctr, float* pooled,
                             float* logits, float* x_out = nullptr, uint16_t* a_top_out = nullptr) {
  if (!m || !indices || !offsets || !ctr || (!dense && m->F > 0)) {
    set_error("null argument (model, dense, indices, offsets and ctr are required)");
    return REC_E_INVALID_ARG;
  }
  if (B <= 0 || B > m->max_batch) {
    set_error("batch = %d must be in [1, max_batch = %d]", B, m->max_batch);
    return REC_E_INVALID_ARG;
  }
  if ((x_out || a_top_out) && m->world > 1 && m->shard != REC_SHARD_REPLICA) {
    set_error("rec_query_inspect: sharded models keep X / A_top distributed");
    return REC_E_UNSUPPORTED;
  }
  if (a_top_out && m->chain_top && m->fuse_interact) {
    set_error("rec_query_inspect: the fused interaction (REC_FUSE_INTERACT=1) builds A_top in "
              "shared memory only");
    return REC_E_UNSUPPORTED;
  }
  REC_CUDA(cudaSetDevice(m->device));
  if (m->pipe_active.load()) {
    rec_status st = pipe_leave(m);
    if (st != REC_OK) return st;
  }
  Workspace& w = m->ws[0];
  cudaStream_t s = w.stream;
  const int T = m->T, nb = T * B;
  rec_status st = wait_pin(w);
  if (st != REC_OK) return st;
  uint8_t* pin = w.pin;
  const bool off_dev = is_device_ptr(offsets), idx_dev = is_device_ptr(indices),
             den_dev = is_device_ptr(dense);
  const int* d_off = offsets;
  const int* d_idx = indices;
  REC_CUDA(cudaMemsetAsync(w.flag, 0, sizeof(int), s));
  size_t pos = 0;
  if (!off_dev) {
    if (offsets[0] != 0) {
      set_error("offsets[0] = %d, must be 0", offsets[0]);
      return REC_E_OFFSETS;
    }
    for (int g = 0; g < nb; ++g)
      if (offsets[g + 1] < offsets[g]) {
        set_error("offsets[%d] = %d < offsets[%d] = %d", g + 1, offsets[g + 1], g, offsets[g]);
        return REC_E_OFFSETS;
      }
    const int64_t nnz = offsets[nb];
    if (nnz > w.idx_cap) {
      set_error("offsets[T*B] = %lld exceeds the index capacity %lld (T*max_batch*pooling_hi)",
                (long long)nnz, (long long)w.idx_cap);
      return REC_E_INVALID_ARG;
    }
    memcpy(pin + pos, offsets, sizeof(int) * (nb + 1));
    REC_CUDA(cudaMemcpyAsync(w.offsets, pin + pos, sizeof(int) * (nb + 1), cudaMemcpyHostToDevice, s));
    pos += sizeof(int) * (nb + 1);
    pos = (pos + 255) & ~size_t(255);
    d_off = w.offsets;
    if (!idx_dev) {
      memcpy(pin + pos, indices, sizeof(int) * nnz);
      REC_CUDA(cudaMemcpyAsync(w.indices, pin + pos, sizeof(int) * nnz, cudaMemcpyHostToDevice, s));
      pos += sizeof(int) * nnz;
      pos = (pos + 255) & ~size_t(255);
      d_idx = w.indices;
    }
  } else {
    launch_check_offsets(offsets, nb, w.flag, s);
    if (!idx_dev) {
      set_error("indices on the host with offsets on the device is not supported");
      return REC_E_INVALID_ARG;
    }
  }
  const float* d_dense = dense;
  if (!den_dev && m->F > 0) {
    memcpy(pin + pos, dense, sizeof(float) * B * m->F);
    REC_CUDA(cudaMemcpyAsync(w.dense_f32, pin + pos, sizeof(float) * B * m->F,
                             cudaMemcpyHostToDevice, s));
    d_dense = w.dense_f32;
  }
  REC_CUDA(cudaEventRecord(w.pin_free, s));
  if (m->world > 1 && m->shard != REC_SHARD_REPLICA)  // model-parallel embeddings (dist.cu)
    return sharded_forward(m, w, d_dense, d_idx, d_off, B, ctr, logits);
  launch_dense_to_bf16(d_dense, B, m->F, m->Fpad, w.dense_bf, s);
  m->launches += 1 + (off_dev ? 1 : 0);
  st = forward_enqueue(m, w, d_idx, d_off, B, nullptr, w.ctr, w.logit, nullptr,
                       off_dev ? int64_t(0x7fffffff) : int64_t(offsets[nb]));
  if (st != REC_OK) return st;
  REC_CUDA(cudaMemcpyAsync(w.flag_host, w.flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  REC_CUDA(cudaStreamSynchronize(s));
  st = read_flag(w);
  if (st != REC_OK) return st;
  REC_CUDA(cudaMemcpyAsync(ctr, w.ctr, sizeof(float) * B * m->tasks, cudaMemcpyDefault, s));
  if (logits)
    REC_CUDA(cudaMemcpyAsync(logits, w.logit, sizeof(float) * B * m->tasks, cudaMemcpyDefault, s));
  if (pooled) {
    const int D = m->D;
    REC_CUDA(cudaMemcpy2DAsync(pooled, sizeof(float) * T * D, w.X + D, sizeof(float) * (T + 1) * D,
                               sizeof(float) * T * D, B, cudaMemcpyDefault, s));
  }
  if (x_out)
    REC_CUDA(cudaMemcpyAsync(x_out, w.X, sizeof(float) * B * (T + 1) * m->D, cudaMemcpyDefault, s));
  if (a_top_out)
    REC_CUDA(cudaMemcpyAsync(a_top_out, w.A_top, sizeof(uint16_t) * B * m->Ktop_pad, cudaMemcpyDefault, s));
  REC_CUDA(cudaStreamSynchronize(s));
  return REC_OK;
}

rec_status shard_plan(int T, const int64_t* rows, int world, int rank, int shard, ShardPlan* p) {
  p->t0 = 0;
  p->t_local = T;
  p->row_lo = 0;
  p->row_hi = 0x7fffffff;
  if (world <= 1 || shard == REC_SHARD_REPLICA) return REC_OK;
  if (shard == REC_SHARD_TABLE) {
    if (T % world != 0) {
      set_error("table-wise sharding needs num_tables (%d) divisible by world (%d)", T, world);
      return REC_E_UNSUPPORTED;
    }
    p->t_local = T / world;
    p->t0 = rank * p->t_local;
    return REC_OK;
  }
  for (int t = 1; t < T; ++t)
    if (rows[t] != rows[0]) {
      set_error("row-wise sharding needs equal rows per table");
      return REC_E_UNSUPPORTED;
    }
  p->row_lo = rows[0] * rank / world;
  p->row_hi = rows[0] * (rank + 1) / world;
  return REC_OK;
}

}  // namespace rec

using namespace rec;

// ====================================================================== C ABI
extern "C" {

const char* rec_last_error(void) { return g_err.c_str(); }
int32_t rec_version(void) { return 1; }

// Models co-located on each device: the hot-row window of rec_hot_remap is the
// persisting L2 capacity divided among them ("memory capacity / model co-location").
static std::mutex g_reg_mu;
static int g_models_on[64] = {};

static void free_model(rec_model_s* m) {
  if (!m) return;
  if (m->counted) {
    std::lock_guard<std::mutex> g(g_reg_mu);
    --g_models_on[m->device & 63];
  }
  cudaFree(m->d_remap);
  cudaFree(m->d_remap_off);
  cudaSetDevice(m->device);
  pipe_destroy(m);
  for (auto& w : m->ws) {
    if (w.stream) cudaStreamSynchronize(w.stream);
    for (auto* p : w.th) cudaFree(p);
    cudaFree(w.wide);
    cudaFree(w.indices);
    cudaFree(w.offsets);
    cudaFree(w.segs);
    cudaFree(w.rowq);
    cudaFree(w.rowi);
    cudaFree(w.dense_f32);
    cudaFree(w.dense_bf);
    if (!w.x_external) cudaFree(w.X);  // (sharded: inside the exchange arena, dist_destroy)
    cudaFree(w.gsegs_local);
    cudaFree(w.A_top);
    cudaFree(w.h[0]);
    cudaFree(w.h[1]);
    cudaFree(w.ctr);
    cudaFree(w.logit);
    cudaFree(w.flag);
    if (w.flag_host) cudaFreeHost(w.flag_host);
    if (w.pin) cudaFreeHost(w.pin);
    if (w.pin_free) cudaEventDestroy(w.pin_free);
    for (auto& sl : w.slots) {
      for (auto& V : sl.var) {
        if (V.exec) cudaGraphExecDestroy(V.exec);
        if (V.graph) cudaGraphDestroy(V.graph);
      }
      delete sl.sb;
      delete sl.sb_local;
      if (sl.free) cudaEventDestroy(sl.free);
      for (auto e : sl.ev)
        if (e) cudaEventDestroy(e);
    }
    cudaFree(w.dB);
    cudaFree(w.gsegs);
    if (w.ev_fork) cudaEventDestroy(w.ev_fork);
    if (w.ev_join) cudaEventDestroy(w.ev_join);
    if (w.ev_sls) cudaEventDestroy(w.ev_sls);
    if (w.ev_done) cudaEventDestroy(w.ev_done);
    if (w.ev_g1) cudaEventDestroy(w.ev_g1);
    if (w.ev_g2) cudaEventDestroy(w.ev_g2);
    if (w.stream_c) {
      cudaStreamSynchronize(w.stream_c);
      cudaStreamDestroy(w.stream_c);
    }
    if (w.stream_b) {
      cudaStreamSynchronize(w.stream_b);
      cudaStreamDestroy(w.stream_b);
    }
    if (w.stream) cudaStreamDestroy(w.stream);
  }
  for (auto& L : m->bottom) {
    cudaFree(L.W);
    cudaFree(L.bias);
  }
  for (auto& L : m->top) {
    cudaFree(L.W);
    cudaFree(L.bias);
  }
  cudaFree(m->w_last);
  for (auto& tw : m->towers)
    for (auto& L : tw) {
      cudaFree(L.W);
      cudaFree(L.bias);
    }
  for (float* p : m->w_last_t) cudaFree(p);
  cudaFree(m->wide_v);
  cudaFree(m->bias_bottom_all);
  cudaFree(m->bias_top_all);
  cudaFree(m->tables);
  cudaFree(m->d_tab_off);
  cudaFree(m->d_rows);
  cudaFree(m->d_tmap_rows);
  for (auto& e : m->prof_events) {
    cudaEventDestroy(e.a);
    cudaEventDestroy(e.b);
  }
  for (auto e : m->prof_pool) cudaEventDestroy(e);
  dist_destroy(m);
  if (m->green[0] || m->green[1]) {  // after the workspaces' streams are gone
    auto destroy = drv_fn<decltype(&cuGreenCtxDestroy)>("cuGreenCtxDestroy");
    for (void* g : m->green)
      if (g && destroy) destroy(static_cast<CUgreenCtx>(g));
  }
  delete m;
}

void rec_model_destroy(rec_model_t m) { free_model(m); }

#define ALLOC(ptr, bytes)                                                            \
  do {                                                                               \
    cudaError_t _e = cudaMalloc(reinterpret_cast<void**>(&(ptr)), (bytes));          \
    if (_e != cudaSuccess) {                                                         \
      set_error("cudaMalloc of %zu bytes for %s failed: %s", (size_t)(bytes), #ptr,  \
                cudaGetErrorString(_e));                                             \
      free_model(m);                                                                 \
      return REC_E_OOM;                                                              \
    }                                                                                \
  } while (0)

#define CHECK_CUDA_CREATE(call)                 \
  do {                                          \
    cudaError_t _e = (call);                    \
    if (_e != cudaSuccess) {                    \
      rec_status _s = cuda_fail(_e, #call);     \
      free_model(m);                            \
      return _s;                                \
    }                                           \
  } while (0)

rec_status rec_model_create(const rec_model_desc* d, rec_model_t* out) {
  if (!d || !out) {
    set_error("desc and out must be non-null");
    return REC_E_INVALID_ARG;
  }
  *out = nullptr;
  // ---------------------------------------------------------------- validation
  if (d->num_tables < 1 || d->num_tables > 4096) {
    set_error("num_tables = %d must be in [1, 4096]", d->num_tables);
    return REC_E_INVALID_ARG;
  }
  if (!d->rows) {
    set_error("rows must be non-null");
    return REC_E_INVALID_ARG;
  }
  for (int t = 0; t < d->num_tables; ++t) {
    if (d->rows[t] < 1) {
      set_error("rows[%d] = %lld must be >= 1", t, (long long)d->rows[t]);
      return REC_E_INVALID_ARG;
    }
    if (d->rows[t] >= (int64_t(1) << 31)) {
      set_error("rows[%d] = %lld must be < 2^31 (int32 indices, R18)", t, (long long)d->rows[t]);
      return REC_E_UNSUPPORTED;
    }
  }
  if (d->dim <= 0 || d->dim % 4 != 0 || d->dim > 128) {
    set_error("dim = %d must be a positive multiple of 4 and <= 128", d->dim);
    return d->dim <= 0 ? REC_E_INVALID_ARG : REC_E_UNSUPPORTED;
  }
  const bool mtwnd = d->arch == REC_ARCH_MTWND;
  if (d->arch != REC_ARCH_DLRM && !mtwnd) {
    set_error("arch = %d unknown", d->arch);
    return REC_E_INVALID_ARG;
  }
  if (mtwnd ? (d->n_tasks < 1 || d->n_tasks > 8) : (d->n_tasks > 1 || d->n_tasks < 0)) {
    set_error("n_tasks = %d: MT-WnD needs 1..8 task towers, DLRM 0 or 1", d->n_tasks);
    return REC_E_INVALID_ARG;
  }
  if (mtwnd && d->n_bottom != 0) {
    set_error("MT-WnD has no bottom MLP: n_bottom must be 0 (Table I, P:191)");
    return REC_E_INVALID_ARG;
  }
  if (mtwnd && d->shard != REC_SHARD_REPLICA) {
    set_error("MT-WnD serves as replicas (no sharded mode)");
    return REC_E_UNSUPPORTED;
  }
  if (!mtwnd && (!d->bottom_widths || d->n_bottom < 2)) {
    set_error("bottom_widths must list >= 2 widths (input first, R3)");
    return REC_E_INVALID_ARG;
  }
  if (!d->top_widths || d->n_top < 2) {
    set_error("top_widths must list >= 2 widths ending in 1 (R3)");
    return REC_E_INVALID_ARG;
  }
  for (int i = 0; i < d->n_bottom; ++i)
    if (d->bottom_widths[i] < 1 || d->bottom_widths[i] > 16384) {
      set_error("bottom_widths[%d] = %d out of [1, 16384]", i, d->bottom_widths[i]);
      return REC_E_INVALID_ARG;
    }
  for (int i = 0; i < d->n_top; ++i)
    if (d->top_widths[i] < 1 || d->top_widths[i] > 16384) {
      set_error("top_widths[%d] = %d out of [1, 16384]", i, d->top_widths[i]);
      return REC_E_INVALID_ARG;
    }
  if (!mtwnd && d->bottom_widths[d->n_bottom - 1] != d->dim) {
    set_error("dim = %d must equal bottom_widths[n_bottom-1] = %d (dot interaction, R4)", d->dim,
              d->bottom_widths[d->n_bottom - 1]);
    return REC_E_INVALID_ARG;
  }
  if (d->top_widths[d->n_top - 1] != 1) {
    set_error("top_widths[n_top-1] = %d must be 1 (CTR output)", d->top_widths[d->n_top - 1]);
    return REC_E_INVALID_ARG;
  }
  if (d->top_widths[d->n_top - 2] > 256) {
    set_error("top_widths[n_top-2] = %d must be <= 256 (width-1 layer fused in one N tile)",
              d->top_widths[d->n_top - 2]);
    return REC_E_UNSUPPORTED;
  }
  if (d->pooling_lo < 0 || d->pooling_hi < d->pooling_lo || d->pooling_hi > 65536) {
    set_error("pooling_lo = %d, pooling_hi = %d must satisfy 0 <= lo <= hi <= 65536",
              d->pooling_lo, d->pooling_hi);
    return REC_E_INVALID_ARG;
  }
  if (d->max_batch < 1 || d->streams < 1 || d->streams > 64) {
    set_error("max_batch = %d must be >= 1 and streams = %d in [1, 64]", d->max_batch, d->streams);
    return REC_E_INVALID_ARG;
  }
  if (d->value_mode != REC_VALUES_INT8_EXACT && d->value_mode != REC_VALUES_FP32) {
    set_error("value_mode = %d unknown", d->value_mode);
    return REC_E_INVALID_ARG;
  }
  if (d->index_dist != REC_INDEX_UNIFORM && d->index_dist != REC_INDEX_SKEW2 &&
      d->index_dist != REC_INDEX_ZIPF) {
    set_error("index_dist = %d unknown", d->index_dist);
    return REC_E_INVALID_ARG;
  }
  if (d->world < 1 || d->rank < 0 || d->rank >= d->world) {
    set_error("rank = %d / world = %d invalid", d->rank, d->world);
    return REC_E_INVALID_ARG;
  }
  if (d->shard < REC_SHARD_REPLICA || d->shard > REC_SHARD_ROW) {
    set_error("shard = %d unknown", d->shard);
    return REC_E_INVALID_ARG;
  }
  const int64_t idx_cap = int64_t(d->num_tables) * d->max_batch * (d->pooling_hi > 0 ? d->pooling_hi : 1);
  if (idx_cap >= (int64_t(1) << 31)) {
    set_error("num_tables * max_batch * pooling_hi = %lld must be < 2^31", (long long)idx_cap);
    return REC_E_UNSUPPORTED;
  }
  // ---------------------------------------------------------------- device
  int ndev = 0;
  cudaError_t ce = cudaGetDeviceCount(&ndev);
  if (ce != cudaSuccess || ndev == 0) {
    set_error("no CUDA device available (%s); this library has no CPU fallback",
              ce == cudaSuccess ? "0 devices" : cudaGetErrorString(ce));
    cudaGetLastError();
    return REC_E_CUDA;
  }
  if (d->device < 0 || d->device >= ndev) {
    set_error("device = %d out of [0, %d)", d->device, ndev);
    return REC_E_INVALID_ARG;
  }
  REC_CUDA(cudaSetDevice(d->device));
  cudaDeviceProp prop;
  REC_CUDA(cudaGetDeviceProperties(&prop, d->device));
  if (prop.major != 10) {
    set_error("device %d is sm_%d%d; this library is built for sm_100a only", d->device,
              prop.major, prop.minor);
    return REC_E_CUDA;
  }
  gemm_prepare();
  chain_prepare();
  {
    const char* e = getenv("REC_CARVEOUT");
    if (e) set_max_smem_carveout(e[0] == 'm' ? 100 : atoi(e));  // experiment: SLS carveout %
  }

  rec_model_s* m = new rec_model_s();
  m->T = d->num_tables;
  m->D = d->dim;
  m->rows.assign(d->rows, d->rows + d->num_tables);
  if (d->n_bottom > 0) m->bottom_w.assign(d->bottom_widths, d->bottom_widths + d->n_bottom);
  m->top_w.assign(d->top_widths, d->top_widths + d->n_top);
  m->arch = d->arch;
  m->tasks = mtwnd ? d->n_tasks : 1;
  m->F = mtwnd ? 0 : m->bottom_w[0];
  m->Fpad = pad8(m->F);
  m->lo = d->pooling_lo;
  m->hi = d->pooling_hi;
  m->top_shift = d->top_shift;
  m->value_mode = d->value_mode;
  m->index_dist = d->index_dist;
  m->max_batch = d->max_batch;
  m->nstreams = d->streams;
  m->device = d->device;
  m->shard = d->shard;
  m->rank = d->rank;
  m->world = d->world;
  m->seed = d->seed;
  m->k0 = static_cast<uint32_t>(d->seed & 0xFFFFFFFFull);
  m->k1 = static_cast<uint32_t>(d->seed >> 32);
  m->l2_persist_bytes = d->l2_persist_bytes;
  // s = round(log2(0.577 sqrt(mean L)))  (G4, R24)
  {
    const double L = 0.5 * (d->pooling_lo + d->pooling_hi);
    m->emb_shift = L > 0 ? static_cast<int>(std::lround(std::log2(0.577 * std::sqrt(L)))) : 0;
  }
  const int T = m->T, D = m->D;

  // ---------------------------------------------------------------- tables
  // shard plan: which tables / rows of them live on this GPU
  {
    ShardPlan sp{};
    rec_status st = shard_plan(T, m->rows.data(), m->world, m->rank, m->shard, &sp);
    if (st != REC_OK) {
      delete m;
      return st;
    }
    m->t0 = sp.t0;
    m->T_loc = sp.t_local;
    m->row_lo = sp.row_lo;
    m->row_hi = sp.row_hi;
  }
  const int TL = m->T_loc;
  auto local_rows = [&](int tl) -> int64_t {
    const int64_t R = m->rows[m->t0 + tl];
    return m->shard == REC_SHARD_ROW && m->world > 1 ? m->row_hi - m->row_lo : R;
  };
  bool equal = true;
  for (int tl = 1; tl < TL; ++tl) equal = equal && (local_rows(tl) == local_rows(0));
  m->interleaved = equal;
  m->tab_off.resize(TL);
  std::vector<int64_t> grows(TL);
  int64_t total_rows = 0;
  for (int tl = 0; tl < TL; ++tl) {
    total_rows += local_rows(tl);
    grows[tl] = m->rows[m->t0 + tl];
  }
  if (equal) {
    // row r of table t at (r*T + t)*D: hot low rows of ALL tables form one contiguous
    // prefix, which an L2 persisting window can cover (P:556-557 hot-embedding residue)
    m->row_stride = int64_t(TL) * D;
    for (int tl = 0; tl < TL; ++tl) m->tab_off[tl] = int64_t(tl) * D;
  } else {
    m->row_stride = D;
    int64_t acc = 0;
    for (int tl = 0; tl < TL; ++tl) {
      m->tab_off[tl] = acc * D;
      acc += local_rows(tl);
    }
  }
  m->table_bytes = static_cast<size_t>(total_rows) * D * sizeof(float);
  ALLOC(m->tables, m->table_bytes);
  ALLOC(m->d_tab_off, sizeof(int64_t) * TL);
  ALLOC(m->d_rows, sizeof(int64_t) * TL);
  CHECK_CUDA_CREATE(cudaMemcpy(m->d_tab_off, m->tab_off.data(), sizeof(int64_t) * TL, cudaMemcpyHostToDevice));
  CHECK_CUDA_CREATE(cudaMemcpy(m->d_rows, grows.data(), sizeof(int64_t) * TL, cudaMemcpyHostToDevice));
  for (int tl = 0; tl < TL; ++tl)
    launch_init_table(m->tables + m->tab_off[tl], local_rows(tl), D, m->row_stride, m->t0 + tl, m->k0,
                      m->k1, m->emb_shift, m->value_mode, 0,
                      m->shard == REC_SHARD_ROW && m->world > 1 ? m->row_lo : 0);
  CHECK_CUDA_CREATE(cudaGetLastError());
  // SLS over TMA row gathers (k_sls_synth_tma, REC_SLS=tma, experimental: measured ~4x slower
  // than the register kernel for 128-B rows): its bag summation order is a fixed tree, exact
  // (order-free) only for int8 x 2^e tables, so fp32 value mode never uses it.
  {
    const char* e = getenv("REC_SLS");
    const bool want = e && strcmp(e, "tma") == 0;  // measured slower: opt-in
#ifdef REC_DEBUG_KNOBS
    // diagnostic build only (-DREC_DEBUG_KNOBS; REC_STEP_DIAG): bit 0 drops the bottom MLP,
    // bit 1 the interaction + top MLP, bit 2 the interaction alone from the synthetic step
    // graphs (CTRs invalid).  The shipped library cannot drop stages.
    if (const char* d = getenv("REC_STEP_DIAG")) m->diag_skip = atoi(d);
#endif
    if (const char* fd = getenv("REC_FUSE_DENSE")) m->fuse_dense = atoi(fd) != 0;
    if (const char* tg = getenv("REC_TOWER_GROUP")) m->tower_group = atoi(tg) != 0;
    if (const char* cp = getenv("REC_CHAIN_PDL")) m->chain_pdl = atoi(cp) != 0;
    if (const char* fi = getenv("REC_FUSE_INTERACT")) m->fuse_interact = atoi(fi) != 0;
    if (const char* gs = getenv("REC_GREEN_SMS")) {
      const int n = atoi(gs);
      void* g[4] = {nullptr, nullptr, nullptr, nullptr};
      if (n > 0 && green_setup(m->device, n, g)) {
        m->green_sms = n;
        for (int k = 0; k < 2; ++k) {
          m->green[k] = g[k];
          m->green_cu[k] = g[2 + k];
        }
      }
    }
    // kernel-variant selectors (process-wide, like the kernels they pick): every model
    // create sets them from the environment, unset = the measured default, so a variant
    // never leaks from one handle's environment into a later handle
    auto env_int = [](const char* n, int dflt) {
      const char* e = getenv(n);
      return e ? atoi(e) : dflt;
    };
    g_gemm_stages = env_int("REC_GEMM_STAGES", 0);
    g_gemm_2sm = env_int("REC_GEMM_2SM", 0);
    g_gemm_2sm_serve = env_int("REC_GEMM_2SM_SERVE", 0);
    g_gemm_narrow = env_int("REC_GEMM_NARROW", 0);
    g_gemm_mt1 = env_int("REC_GEMM_MT1", 0);
    g_gemm_bn64 = env_int("REC_GEMM_BN64", 0);
    g_gemm_mt2 = env_int("REC_GEMM_MT2", 0);
    g_chain_persistent = env_int("REC_CHAIN_PERSISTENT", 1);
    g_interact_wpc = std::max(1, std::min(8, env_int("REC_INTERACT_WPC", 8)));
    g_interact_pf = env_int("REC_INTERACT_PF", 0);
    kBlockedRows = env_int("REC_INTERACT_BLOCKED", 24) > 0 ? env_int("REC_INTERACT_BLOCKED", 24) : 1 << 30;
    {
      int lo = 0, hi = 0;
      cudaDeviceGetStreamPriorityRange(&lo, &hi);
      const int pr = env_int("REC_PRIO", 0);
      g_dense_prio = pr > 0 ? hi : 0;
      g_sls_prio = pr < 0 ? hi : 0;
    }
    const char* p = getenv("REC_PDL");
    m->sls_pdl = !(p && strcmp(p, "0") == 0);
    m->sls_interleave = env_int("REC_SLS_GRID", 0);
    CHECK_CUDA_CREATE(cudaDeviceGetAttribute(&m->nsm, cudaDevAttrMultiProcessorCount, m->device));
    if (want && m->value_mode == REC_VALUES_INT8_EXACT && sls_tma_supported(D) &&
        total_rows < (int64_t(1) << 31)) {
      CUtensorMap hm;
      if (encode_tmap_rows_f32(&hm, m->tables, static_cast<uint64_t>(total_rows), D)) {
        ALLOC(m->d_tmap_rows, sizeof(CUtensorMap));
        CHECK_CUDA_CREATE(cudaMemcpy(m->d_tmap_rows, &hm, sizeof(hm), cudaMemcpyHostToDevice));
        m->sls_tma = 1;
      }
    }
  }

  // ---------------------------------------------------------------- MLP weights (G5)
  auto wexp = [](int fan_in) {
    return static_cast<int>(std::lround(std::log2(std::sqrt(3.0 / fan_in))));
  };
  auto make_layer = [&](int K, int N, int layer_id, int extra_shift, rec::Layer& L) -> rec_status {
    L.K = K;
    L.Kpad = pad8(K);
    L.N = N;
    L.Npad = pad8(N);
    L.bn = gemm_bn(N);
    L.layer_id = layer_id;
    L.exp = -7 + wexp(K) - extra_shift;
    if (cudaMalloc(reinterpret_cast<void**>(&L.W), sizeof(__nv_bfloat16) * N * L.Kpad) != cudaSuccess ||
        cudaMalloc(reinterpret_cast<void**>(&L.bias), sizeof(float) * N) != cudaSuccess) {
      set_error("cudaMalloc of layer %d weights failed", layer_id);
      return REC_E_OOM;
    }
    launch_init_layer(L.W, L.bias, N, K, L.Kpad, layer_id, L.exp, m->k0, m->k1, 0);
    if (!encode_tmap_bf16(&L.tmap_w64, L.W, N, K, L.Kpad, std::min(L.bn, 64))) {
      set_error("cuTensorMapEncodeTiled failed for layer %d weights", layer_id);
      return REC_E_CUDA;
    }
    if (!encode_tmap_bf16(&L.tmap_w128, L.W, N, K, L.Kpad, std::min(L.bn, 128))) {
      set_error("cuTensorMapEncodeTiled failed for layer %d weights", layer_id);
      return REC_E_CUDA;
    }
    if (!encode_tmap_bf16(&L.tmap_w, L.W, N, K, L.Kpad, L.bn)) {
      set_error("cuTensorMapEncodeTiled failed for layer %d weights", layer_id);
      return REC_E_CUDA;
    }
    return REC_OK;
  };
  const int nbl = std::max(0, d->n_bottom - 1);
  m->bottom.resize(nbl);
  for (int l = 0; l < nbl; ++l) {
    rec_status st = make_layer(m->bottom_w[l], m->bottom_w[l + 1], l, 0, m->bottom[l]);
    if (st != REC_OK) {
      free_model(m);
      return st;
    }
  }
  m->Ktop = m->arch == REC_ARCH_MTWND ? T * D : D + T * (T + 1) / 2;
  m->Ktop_pad = pad8(m->Ktop);
  std::vector<int> tw;
  tw.push_back(m->Ktop);
  for (int v : m->top_w) tw.push_back(v);
  const int ntl = d->n_top - 1;  // GEMM layers (the width-1 output layer is an epilogue)
  m->top.resize(ntl);
  for (int j = 0; j < ntl; ++j) {
    rec_status st = make_layer(tw[j], tw[j + 1], TOP_LAYER_BASE + j, j == 0 ? m->top_shift : 0, m->top[j]);
    if (st != REC_OK) {
      free_model(m);
      return st;
    }
  }
  {
    const int Kf = tw[ntl];
    ALLOC(m->w_last, sizeof(float) * (Kf + 1));
    const int ef = -7 + wexp(Kf) - (ntl == 0 ? m->top_shift : 0);
    launch_init_final(m->w_last, m->w_last + Kf, Kf, TOP_LAYER_BASE + ntl, ef, m->k0, m->k1, 0);
    CHECK_CUDA_CREATE(cudaMemcpy(&m->b_last, m->w_last + Kf, sizeof(float), cudaMemcpyDeviceToHost));
  }
  if (m->arch == REC_ARCH_MTWND) {
    // towers of tasks 1..N-1 (layer ids TOP_LAYER_BASE + 16 k + l, oracle/gen.py) and the wide
    // vectors of every task (id TOP_LAYER_BASE + 16 k + 15: the weight row of a fan-out-1 layer)
    constexpr int kTaskStride = 16, kWide = 15;
    m->towers.resize(m->tasks - 1);
    m->w_last_t.assign(m->tasks - 1, nullptr);
    m->b_last_t.assign(m->tasks - 1, 0.f);
    const int Kf = tw[ntl];
    for (int k = 1; k < m->tasks; ++k) {
      auto& L = m->towers[k - 1];
      L.resize(ntl);
      for (int j = 0; j < ntl; ++j) {
        rec_status st = make_layer(tw[j], tw[j + 1], TOP_LAYER_BASE + kTaskStride * k + j,
                                   j == 0 ? m->top_shift : 0, L[j]);
        if (st != REC_OK) {
          free_model(m);
          return st;
        }
      }
      ALLOC(m->w_last_t[k - 1], sizeof(float) * (Kf + 1));
      const int ef = -7 + wexp(Kf) - (ntl == 0 ? m->top_shift : 0);
      launch_init_final(m->w_last_t[k - 1], m->w_last_t[k - 1] + Kf, Kf,
                        TOP_LAYER_BASE + kTaskStride * k + ntl, ef, m->k0, m->k1, 0);
      CHECK_CUDA_CREATE(cudaMemcpy(&m->b_last_t[k - 1], m->w_last_t[k - 1] + Kf, sizeof(float),
                                   cudaMemcpyDeviceToHost));
    }
    ALLOC(m->wide_v, sizeof(float) * (int64_t(m->tasks) * m->Ktop + 1));
    const int ew = -7 + wexp(m->Ktop) - m->top_shift;
    for (int k = 0; k < m->tasks; ++k)  // row k of [N][Ktop]; the "bias" lands on row k+1's
      launch_init_final(m->wide_v + int64_t(k) * m->Ktop, m->wide_v + int64_t(k + 1) * m->Ktop,
                        m->Ktop, TOP_LAYER_BASE + kTaskStride * k + kWide, ew, m->k0, m->k1, 0);
    CHECK_CUDA_CREATE(cudaDeviceSynchronize());  // (row k's bias slot is rewritten by row k+1)
  }
  m->hmax = 8;
  for (int l = 1; l < d->n_bottom - 1; ++l) m->hmax = std::max(m->hmax, pad8(m->bottom_w[l]));
  for (int j = 0; j < d->n_top - 2; ++j) m->hmax = std::max(m->hmax, pad8(m->top_w[j]));

  // ---------------------------------------------------------------- fused FC stacks
  {
    const char* e = getenv("REC_MLP");
    const bool allow = !(e && e[0] == 'l');  // REC_MLP=layers: per-layer GEMMs (A/B profiling)
    auto build = [&](std::vector<rec::Layer>& Ls, ChainArgs& ca, float** bias_all, int mode) -> bool {
      const int nl = static_cast<int>(Ls.size());
      if (!allow || nl < 1 || nl > 4) return false;
      ca = ChainArgs{};
      ca.nlayers = nl;
      int total = 0, maxn = 0, act = 0;
      for (int l = 0; l < nl; ++l) {
        ca.K[l] = Ls[l].K;
        ca.N[l] = Ls[l].N;
        ca.wbox[l] = Ls[l].bn;
        total += Ls[l].N;
        maxn = std::max(maxn, Ls[l].N);
        if (l < nl - 1) act = std::max(act, (Ls[l].N + 63) / 64);
      }
      ca.bias_total = total;
      ca.act_kblocks = act;
      int tc = 32;
      while (tc < maxn) tc *= 2;
      // layers wider than 256 (RMC2/RMC3's 512-wide hidden layers) run as per-layer GEMMs: such
      // chains never meet the co-location shared-memory budget, and they are not validated
      if (tc > 256) return false;
      ca.tmem_cols = tc;
      ca.mode_last = mode;
      ca.wl_n = mode == GEMM_OUT_CTR ? Ls[nl - 1].N : 0;
      if (!chain_configure(ca)) return false;
      for (int l = 0; l < nl; ++l) ca.wbox[l] = std::min(Ls[l].bn, ca.nchunk);
      if (cudaMalloc(reinterpret_cast<void**>(bias_all), sizeof(float) * total) != cudaSuccess) return false;
      int off = 0;
      for (int l = 0; l < nl; ++l) {
        cudaMemcpy(*bias_all + off, Ls[l].bias, sizeof(float) * Ls[l].N, cudaMemcpyDeviceToDevice);
        off += Ls[l].N;
      }
      ca.bias_all = *bias_all;
      if (mode == GEMM_OUT_CTR) {
        ca.w_last = m->w_last;
        ca.b_last = m->b_last;
      }
      return true;
    };
    CHECK_CUDA_CREATE(cudaDeviceSynchronize());  // biases initialised
    m->chain_bottom = build(m->bottom, m->chain_bottom_args, &m->bias_bottom_all, GEMM_OUT_X_F32);
    if (m->arch == REC_ARCH_DLRM)  // MT-WnD towers run as per-layer GEMMs (1024-wide)
      m->chain_top = build(m->top, m->chain_top_args, &m->bias_top_all, GEMM_OUT_CTR);
    // the fused interaction builds layer 0's A (Ktop_pad columns) in the activation buffer
    if (!(m->chain_top && m->arch == REC_ARCH_DLRM && chain_interact_supported(m->T, m->D) &&
          m->chain_top_args.act_kblocks * 64 >= m->chain_top_args.K[0]))
      m->fuse_interact = 0;
  }

  // ---------------------------------------------------------------- workspaces
  const int cap = m->max_batch;
  m->ws.resize(m->nstreams);
  for (int s = 0; s < m->nstreams; ++s) {
    rec::Workspace& w = m->ws[s];
    w.cap = cap;
    w.idx_cap = idx_cap;
    if (m->green_sms > 0) {
      if (!green_stream(m->green[1], &w.stream) || !green_stream(m->green[0], &w.stream_b)) {
        set_error("green-context stream creation failed");
        free_model(m);
        return REC_E_CUDA;
      }
      CHECK_CUDA_CREATE(cudaEventCreateWithFlags(&w.ev_g1, cudaEventDisableTiming));
      CHECK_CUDA_CREATE(cudaEventCreateWithFlags(&w.ev_g2, cudaEventDisableTiming));
    } else {
      CHECK_CUDA_CREATE(cudaStreamCreateWithFlags(&w.stream, cudaStreamNonBlocking));
      CHECK_CUDA_CREATE(cudaStreamCreateWithFlags(&w.stream_b, cudaStreamNonBlocking));
    }
    CHECK_CUDA_CREATE(cudaEventCreateWithFlags(&w.ev_fork, cudaEventDisableTiming));
    CHECK_CUDA_CREATE(cudaEventCreateWithFlags(&w.ev_join, cudaEventDisableTiming));
    CHECK_CUDA_CREATE(cudaStreamCreateWithFlags(&w.stream_c, cudaStreamNonBlocking));
    CHECK_CUDA_CREATE(cudaEventCreateWithFlags(&w.ev_sls, cudaEventDisableTiming));
    CHECK_CUDA_CREATE(cudaEventCreateWithFlags(&w.ev_done, cudaEventDisableTiming));
    ALLOC(w.dB, sizeof(int) * 4);
    ALLOC(w.gsegs, sizeof(int4) * (cap + 1));
    CHECK_CUDA_CREATE(cudaEventCreateWithFlags(&w.pin_free, cudaEventDisableTiming));
    ALLOC(w.indices, sizeof(int) * (idx_cap > 0 ? idx_cap : 1));
    ALLOC(w.offsets, sizeof(int) * (int64_t(T) * cap + 1));
    ALLOC(w.segs, sizeof(int4) * cap);
    ALLOC(w.rowq, sizeof(int) * cap);
    ALLOC(w.rowi, sizeof(int) * cap);
    ALLOC(w.dense_f32, sizeof(float) * int64_t(cap) * std::max(m->F, 1));
    ALLOC(w.dense_bf, sizeof(__nv_bfloat16) * int64_t(cap) * std::max(m->Fpad, 8));
    ALLOC(w.X, sizeof(float) * int64_t(cap) * (T + 1) * D);
    ALLOC(w.A_top, sizeof(__nv_bfloat16) * int64_t(cap) * m->Ktop_pad);
    ALLOC(w.h[0], sizeof(__nv_bfloat16) * int64_t(cap) * m->hmax);
    ALLOC(w.h[1], sizeof(__nv_bfloat16) * int64_t(cap) * m->hmax);
    ALLOC(w.ctr, sizeof(float) * cap * m->tasks);
    ALLOC(w.logit, sizeof(float) * cap * m->tasks);
    if (m->arch == REC_ARCH_MTWND) ALLOC(w.wide, sizeof(float) * cap * m->tasks);
    ALLOC(w.flag, sizeof(int));
    CHECK_CUDA_CREATE(cudaMemset(w.flag, 0, sizeof(int)));
    CHECK_CUDA_CREATE(cudaMemset(w.dense_bf, 0, sizeof(__nv_bfloat16) * int64_t(cap) * m->Fpad));
    CHECK_CUDA_CREATE(cudaMemset(w.A_top, 0, sizeof(__nv_bfloat16) * int64_t(cap) * m->Ktop_pad));
    CHECK_CUDA_CREATE(cudaMemset(w.h[0], 0, sizeof(__nv_bfloat16) * int64_t(cap) * m->hmax));
    CHECK_CUDA_CREATE(cudaMemset(w.h[1], 0, sizeof(__nv_bfloat16) * int64_t(cap) * m->hmax));
    CHECK_CUDA_CREATE(cudaMallocHost(reinterpret_cast<void**>(&w.flag_host), sizeof(int)));
    w.pin_bytes = sizeof(int) * (int64_t(T) * cap + 1) + sizeof(int) * idx_cap +
                  sizeof(float) * int64_t(cap) * m->F + 2 * sizeof(int4) * (cap + 1) + 4096;
    if (cudaMallocHost(reinterpret_cast<void**>(&w.pin), w.pin_bytes) != cudaSuccess) {
      set_error("cudaMallocHost of %zu pinned staging bytes failed", w.pin_bytes);
      free_model(m);
      return REC_E_OOM;
    }
    CHECK_CUDA_CREATE(cudaEventRecord(w.pin_free, w.stream));
    // A operand tensor maps + outputs of every GEMM layer on this workspace
    w.tmap_a_bottom.resize(nbl);
    w.out_bottom.resize(nbl);
    for (int l = 0; l < nbl; ++l) {
      const void* a_base = l == 0 ? static_cast<void*>(w.dense_bf) : static_cast<void*>(w.h[(l - 1) & 1]);
      const int K = m->bottom[l].K;
      const int ld = l == 0 ? m->Fpad : m->bottom[l - 1].Npad;
      if (!encode_tmap_bf16(&w.tmap_a_bottom[l], a_base, cap, K, ld, 128)) {
        set_error("cuTensorMapEncodeTiled failed (bottom layer %d activations)", l);
        free_model(m);
        return REC_E_CUDA;
      }
      w.out_bottom[l] = (l == nbl - 1) ? static_cast<void*>(w.X) : static_cast<void*>(w.h[l & 1]);
    }
    w.tmap_a_top.resize(ntl);
    w.out_top.resize(ntl);
    for (int j = 0; j < ntl; ++j) {
      const void* a_base = j == 0 ? static_cast<void*>(w.A_top) : static_cast<void*>(w.h[(j - 1) & 1]);
      const int K = m->top[j].K;
      const int ld = j == 0 ? m->Ktop_pad : m->top[j - 1].Npad;
      if (!encode_tmap_bf16(&w.tmap_a_top[j], a_base, cap, K, ld, 128)) {
        set_error("cuTensorMapEncodeTiled failed (top layer %d activations)", j);
        free_model(m);
        return REC_E_CUDA;
      }
      w.out_top[j] = (j == ntl - 1) ? nullptr : static_cast<void*>(w.h[j & 1]);
    }
    if (m->arch == REC_ARCH_MTWND && m->tasks > 1) {  // towers 1..N-1 run in the same launches
      w.th.assign(2 * m->tasks, nullptr);
      w.tmap_a_task.assign(m->tasks, std::vector<CUtensorMap>(ntl));
      w.out_task.assign(m->tasks, std::vector<void*>(ntl, nullptr));
      for (int k = 1; k < m->tasks; ++k) {
        ALLOC(w.th[2 * k], sizeof(__nv_bfloat16) * int64_t(cap) * m->hmax);
        ALLOC(w.th[2 * k + 1], sizeof(__nv_bfloat16) * int64_t(cap) * m->hmax);
        for (int j = 0; j < ntl; ++j) {
          const void* a_base = j == 0 ? static_cast<void*>(w.A_top) : static_cast<void*>(w.th[2 * k + ((j - 1) & 1)]);
          const int K = m->top[j].K;
          const int ld = j == 0 ? m->Ktop_pad : m->top[j - 1].Npad;
          if (!encode_tmap_bf16(&w.tmap_a_task[k][j], a_base, cap, K, ld, 128)) {
            set_error("cuTensorMapEncodeTiled failed (tower %d layer %d activations)", k, j);
            free_model(m);
            return REC_E_CUDA;
          }
          w.out_task[k][j] = (j == ntl - 1) ? nullptr : static_cast<void*>(w.th[2 * k + (j & 1)]);
        }
      }
    }
    auto fill_maps = [&](ChainMaps& mp, const CUtensorMap& a0, std::vector<rec::Layer>& Ls, int nch) {
      mp.a0 = a0;
      CUtensorMap* ws_[4] = {&mp.w0, &mp.w1, &mp.w2, &mp.w3};
      for (int l = 0; l < 4; ++l) {
        const rec::Layer& L = Ls[std::min<int>(l, static_cast<int>(Ls.size()) - 1)];
        *ws_[l] = nch == 128 ? L.tmap_w128 : L.tmap_w;
      }
    };
    if (!m->bottom.empty())
      fill_maps(w.chain_bottom, w.tmap_a_bottom[0], m->bottom, m->chain_bottom_args.nchunk);
    fill_maps(w.chain_top, w.tmap_a_top[0], m->top, m->chain_top_args.nchunk);
  }
  // synthetic-batch staging ring + one captured CUDA graph per slot (a2-a6 chain)
  constexpr int kSlots = 4;
  for (auto& w : m->ws) {
    w.slots.resize(kSlots);
    for (auto& sl : w.slots) {
      sl.sb = new SegBatch();
      memset(sl.sb, 0, sizeof(SegBatch));
      sl.sb_local = new SegBatch();
      memset(sl.sb_local, 0, sizeof(SegBatch));
      sl.sb->B = 1;
      sl.sb->nseg = 1;
      sl.sb->seg[0] = make_int4(0, 0, 1, 0);
      fill_genargs(m, w, sl.ga, sl.sa, nullptr);
      CHECK_CUDA_CREATE(cudaEventCreateWithFlags(&sl.free, cudaEventDisableTiming));
      CHECK_CUDA_CREATE(cudaEventRecord(sl.free, w.stream));
      for (auto& e : sl.ev) CHECK_CUDA_CREATE(cudaEventCreate(&e));
    }
  }
  CHECK_CUDA_CREATE(cudaDeviceSynchronize());

  // L2 persisting window over the hot row prefix (interleaved layout only)
  if (m->l2_persist_bytes > 0) {
    if (!m->interleaved) {
      set_error("l2_persist_bytes needs equal rows per table (interleaved arena)");
      free_model(m);
      return REC_E_UNSUPPORTED;
    }
    size_t win = std::min<size_t>(static_cast<size_t>(m->l2_persist_bytes), m->table_bytes);
    win = std::min<size_t>(win, static_cast<size_t>(prop.accessPolicyMaxWindowSize));
    const size_t carve = std::min<size_t>(win, prop.persistingL2CacheMaxSize);
    CHECK_CUDA_CREATE(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, carve));
    for (auto& w : m->ws) {
      cudaStreamAttrValue v{};
      v.accessPolicyWindow.base_ptr = m->tables;
      v.accessPolicyWindow.num_bytes = win;
      // a window larger than the persisting carve-out would thrash it: persist a random
      // carve/win fraction of the window's lines (the rest stream)
      v.accessPolicyWindow.hitRatio = static_cast<float>(std::min(1.0, double(carve) / double(win)));
      v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      CHECK_CUDA_CREATE(cudaStreamSetAttribute(w.stream, cudaStreamAttributeAccessPolicyWindow, &v));
    }
  }

  // capture after the stream attributes (L2 window) are final: graph kernel nodes keep them
  for (auto& w : m->ws) {
    if (m->world > 1 && m->shard != REC_SHARD_REPLICA) break;  // no synthetic chain when sharded
    rec_status st = capture_graphs(m, w);
    if (st != REC_OK) {
      free_model(m);
      return st;
    }
  }

  if (m->world > 1 && m->shard == REC_SHARD_REPLICA && d->nccl_id) {
    // replicas: a communicator only for rec_serve's all-rank percentiles (no data path use)
    rec_status st = dist_init(m, d->nccl_id);
    if (st != REC_OK) {
      free_model(m);
      return st;
    }
  }
  if (m->world > 1 && m->shard != REC_SHARD_REPLICA) {
    rec_status st = dist_init(m, d->nccl_id);
    if (st != REC_OK) {
      free_model(m);
      return st;
    }
    // table-wise over peer memory: one captured graph per staging slot of the asynchronous
    // sharded chain (device-synthesised inputs need fixed pooling, as for replicas)
    if (m->p2p_slots && m->lo == m->hi && m->arch == REC_ARCH_DLRM)
      for (auto& w : m->ws) {
        st = shard_capture(m, w);
        if (st != REC_OK) {
          free_model(m);
          return st;
        }
      }
  }
  {
    std::lock_guard<std::mutex> g(g_reg_mu);
    ++g_models_on[m->device & 63];
    m->counted = true;
  }
  *out = m;
  return REC_OK;
}

rec_status rec_query(rec_model_t m, const float* dense, const int32_t* indices,
                     const int32_t* offsets, int32_t batch, float* ctr) {
  return query_impl(m, dense, indices, offsets, batch, ctr, nullptr, nullptr);
}

rec_status rec_query_debug(rec_model_t m, const float* dense, const int32_t* indices,
                           const int32_t* offsets, int32_t batch, float* ctr, float* pooled,
                           float* logits) {
  return query_impl(m, dense, indices, offsets, batch, ctr, pooled, logits);
}

// ---------------------------------------------------------------- hot-row partition (f3)
// L2 persisting window over the first `bytes` of the arena (the hot-row prefix: with the
// interleaved layout row r of every table precedes row r + 1 of any table).
static rec_status set_l2_window(rec_model_s* m, size_t bytes) {
  cudaDeviceProp prop;
  REC_CUDA(cudaGetDeviceProperties(&prop, m->device));
  size_t win = std::min<size_t>(bytes, m->table_bytes);
  win = std::min<size_t>(win, static_cast<size_t>(prop.accessPolicyMaxWindowSize));
  const size_t carve = std::min<size_t>(win, prop.persistingL2CacheMaxSize);
  if (win > 0) REC_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, carve));
  for (auto& w : m->ws) {
    cudaStreamAttrValue v{};
    v.accessPolicyWindow.base_ptr = win > 0 ? m->tables : nullptr;
    v.accessPolicyWindow.num_bytes = win;
    v.accessPolicyWindow.hitRatio = win > 0 ? static_cast<float>(std::min(1.0, double(carve) / double(win))) : 0.f;
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    REC_CUDA(cudaStreamSetAttribute(w.stream, cudaStreamAttributeAccessPolicyWindow, &v));
  }
  m->hot_window = static_cast<int64_t>(win);
  return REC_OK;
}

// Re-derive every staging slot's kernel arguments and re-capture its graphs (graph kernel
// nodes keep the stream attributes of their capture, e.g. the L2 window).
static rec_status recapture(rec_model_s* m) {
  for (auto& w : m->ws) {
    REC_CUDA(cudaStreamSynchronize(w.stream));
    for (auto& sl : w.slots) {
      fill_genargs(m, w, sl.ga, sl.sa, nullptr);
      for (auto& V : sl.var) {
        if (V.exec) cudaGraphExecDestroy(V.exec);
        if (V.graph) cudaGraphDestroy(V.graph);
        V = SynthSlot::Variant{};
      }
    }
    rec_status st = capture_graphs(m, w);
    if (st != REC_OK) return st;
  }
  return REC_OK;
}

rec_status rec_hot_remap(rec_model_t m, const int32_t* indices, const int32_t* offsets, int32_t batch,
                         int64_t window_bytes, int64_t* hot_rows) {
  if (!m || !indices || !offsets || batch < 1) {
    set_error("model, indices, offsets and batch >= 1 are required");
    return REC_E_INVALID_ARG;
  }
  if (m->world > 1 && m->shard != REC_SHARD_REPLICA) {
    set_error("rec_hot_remap: replicated models only");
    return REC_E_UNSUPPORTED;
  }
  if (!m->interleaved) {
    set_error("rec_hot_remap needs equal rows per table (interleaved arena: the hot rows of all "
              "tables form one prefix)");
    return REC_E_UNSUPPORTED;
  }
  if (!m->pipe.empty()) {
    set_error("rec_hot_remap: remove the pipeline lanes first (rec_set_pipeline(m, 0))");
    return REC_E_INVALID_ARG;
  }
  REC_CUDA(cudaSetDevice(m->device));
  REC_CUDA(cudaDeviceSynchronize());
  const int T = m->T, D = m->D;
  // 1. access-frequency profile of the sample (host copy of the caller's arrays)
  const int nb = T * batch;
  std::vector<int32_t> off(nb + 1);
  REC_CUDA(cudaMemcpy(off.data(), offsets, sizeof(int32_t) * (nb + 1), cudaMemcpyDefault));
  for (int g = 0; g < nb; ++g)
    if (off[0] != 0 || off[g + 1] < off[g]) {
      set_error("offsets are not non-decreasing from 0");
      return REC_E_OFFSETS;
    }
  std::vector<int32_t> idx(off[nb]);
  REC_CUDA(cudaMemcpy(idx.data(), indices, sizeof(int32_t) * idx.size(), cudaMemcpyDefault));
  std::vector<int64_t> roff(T + 1, 0);
  for (int t = 0; t < T; ++t) roff[t + 1] = roff[t] + m->rows[t];
  std::vector<uint32_t> cnt(roff[T], 0);
  for (int t = 0; t < T; ++t)
    for (int64_t j = off[t * batch]; j < off[(t + 1) * batch]; ++j) {
      const int32_t r = idx[j];
      if (r < 0 || r >= m->rows[t]) {
        set_error("profile index %d of table %d outside [0, %lld)", r, t, (long long)m->rows[t]);
        return REC_E_INDEX_OOB;
      }
      ++cnt[roff[t] + r];
    }
  // 2. per table: rows by descending count (ties by row id) -> arena position
  std::vector<int32_t> inv(roff[T]), remap(roff[T]);
  for (int t = 0; t < T; ++t) {
    int32_t* iv = inv.data() + roff[t];
    for (int64_t r = 0; r < m->rows[t]; ++r) iv[r] = static_cast<int32_t>(r);
    const uint32_t* c = cnt.data() + roff[t];
    std::stable_sort(iv, iv + m->rows[t], [c](int32_t a, int32_t b) { return c[a] > c[b]; });
    for (int64_t p = 0; p < m->rows[t]; ++p) remap[roff[t] + iv[p]] = static_cast<int32_t>(p);
  }
  // 3. regenerate the tables in id order and permute them into the arena
  int* d_inv = nullptr;
  float* tmp = nullptr;
  if (!m->d_remap) {
    REC_CUDA(cudaMalloc(reinterpret_cast<void**>(&m->d_remap), sizeof(int32_t) * roff[T]));
    REC_CUDA(cudaMalloc(reinterpret_cast<void**>(&m->d_remap_off), sizeof(int64_t) * T));
  }
  REC_CUDA(cudaMemcpy(m->d_remap, remap.data(), sizeof(int32_t) * roff[T], cudaMemcpyHostToDevice));
  REC_CUDA(cudaMemcpy(m->d_remap_off, roff.data(), sizeof(int64_t) * T, cudaMemcpyHostToDevice));
  if (cudaMalloc(reinterpret_cast<void**>(&d_inv), sizeof(int32_t) * roff[T]) != cudaSuccess ||
      cudaMalloc(reinterpret_cast<void**>(&tmp), m->table_bytes) != cudaSuccess) {
    cudaFree(d_inv);
    set_error("rec_hot_remap: no device memory for the permutation");
    return REC_E_OOM;
  }
  REC_CUDA(cudaMemcpy(d_inv, inv.data(), sizeof(int32_t) * roff[T], cudaMemcpyHostToDevice));
  int64_t maxr = 0;
  for (int t = 0; t < T; ++t) {
    maxr = std::max(maxr, m->rows[t]);
    launch_init_table(tmp + m->tab_off[t], m->rows[t], D, m->row_stride, m->t0 + t, m->k0, m->k1,
                      m->emb_shift, m->value_mode, 0, 0);
  }
  launch_permute_rows(tmp, m->tables, m->d_tab_off, m->row_stride, m->d_rows, T, D, d_inv,
                      m->d_remap_off, maxr, 0);
  cudaError_t e = cudaDeviceSynchronize();
  cudaFree(tmp);
  cudaFree(d_inv);
  if (e != cudaSuccess) return cuda_fail(e, "rec_hot_remap permute");
  // 4. persisting L2 window over the hot prefix: capacity / co-located models
  size_t win = 0;
  if (window_bytes > 0) {
    win = static_cast<size_t>(window_bytes);
  } else if (window_bytes == 0) {
    cudaDeviceProp prop;
    REC_CUDA(cudaGetDeviceProperties(&prop, m->device));
    int models = 1;
    {
      std::lock_guard<std::mutex> g(g_reg_mu);
      models = std::max(1, g_models_on[m->device & 63]);
    }
    win = static_cast<size_t>(prop.persistingL2CacheMaxSize) / models;
  }
  rec_status st = set_l2_window(m, win);
  if (st != REC_OK) return st;
  st = recapture(m);
  if (st != REC_OK) return st;
  if (hot_rows) *hot_rows = m->hot_window / (static_cast<int64_t>(T) * D * 4);
  return REC_OK;
}

rec_status rec_query_inspect(rec_model_t m, const float* dense, const int32_t* indices,
                             const int32_t* offsets, int32_t batch, float* ctr, float* x,
                             uint16_t* a_top, int32_t* a_top_ld) {
  if (!m) {
    set_error("null model");
    return REC_E_INVALID_ARG;
  }
  if (a_top_ld) *a_top_ld = m->Ktop_pad;
  return query_impl(m, dense, indices, offsets, batch, ctr, nullptr, nullptr, x, a_top);
}

rec_status rec_query_async(rec_model_t m, int32_t slot, const float* dense, const int32_t* indices,
                           const int32_t* offsets, int64_t nnz, int32_t batch, float* ctr) {
  if (!m || !indices || !offsets || !ctr || (!dense && m->F > 0)) {
    set_error("null argument");
    return REC_E_INVALID_ARG;
  }
  const bool sharded = m->world > 1 && m->shard != REC_SHARD_REPLICA;
  if (sharded && !m->p2p_slots) {
    set_error("row-wise / NCCL-exchange sharded models are synchronous collectives: use rec_query");
    return REC_E_UNSUPPORTED;
  }
  if (slot < 0 || slot >= m->nstreams) {
    set_error("slot = %d out of [0, %d)", slot, m->nstreams);
    return REC_E_INVALID_ARG;
  }
  if (batch <= 0 || batch > m->max_batch) {
    set_error("batch = %d must be in [1, max_batch = %d]", batch, m->max_batch);
    return REC_E_INVALID_ARG;
  }
  if (nnz < 0) {
    set_error("nnz = %lld must be >= 0", (long long)nnz);
    return REC_E_INVALID_ARG;
  }
  REC_CUDA(cudaSetDevice(m->device));
  if (m->pipe_active.load()) {
    rec_status st = pipe_leave(m);
    if (st != REC_OK) return st;
  }
  Workspace& w = m->ws[slot];
  cudaStream_t s = w.stream;
  // host buffers (pinned: fully asynchronous) are copied straight into this slot's device
  // buffers on its stream; the CTRs come back the same way (e2e serving path)
  const int nb = m->T * batch;
  const int* d_off = offsets;
  const int* d_idx = indices;
  const float* d_dense = dense;
  const bool off_dev = is_device_ptr(offsets), idx_dev = is_device_ptr(indices);
  if (!idx_dev && nnz > w.idx_cap) {
    set_error("nnz = %lld exceeds the index capacity %lld", (long long)nnz, (long long)w.idx_cap);
    return REC_E_INVALID_ARG;
  }
  if (nnz > 0x7fffffff) {
    set_error("nnz = %lld must be < 2^31", (long long)nnz);
    return REC_E_UNSUPPORTED;
  }
  if (!off_dev) {  // host offsets: validated here, before anything is enqueued
    if (offsets[0] != 0) {
      set_error("offsets[0] = %d, must be 0", offsets[0]);
      return REC_E_OFFSETS;
    }
    for (int g = 0; g < nb; ++g)
      if (offsets[g + 1] < offsets[g]) {
        set_error("offsets[%d] = %d < offsets[%d] = %d", g + 1, offsets[g + 1], g, offsets[g]);
        return REC_E_OFFSETS;
      }
    if (static_cast<int64_t>(offsets[nb]) != nnz) {
      set_error("offsets[T*B] = %d != nnz = %lld", offsets[nb], (long long)nnz);
      return REC_E_OFFSETS;
    }
    REC_CUDA(cudaMemcpyAsync(w.offsets, offsets, sizeof(int) * (nb + 1), cudaMemcpyHostToDevice, s));
    d_off = w.offsets;
  }
  if (!idx_dev) {
    // table-wise sharded with host offsets: only this rank's tables' indices cross PCIe (the
    // range [offsets[t0 B], offsets[(t0 + T_loc) B]) of the table-major CSR, same positions)
    int64_t i0 = 0, i1 = nnz;
    if (sharded && !off_dev) {
      i0 = offsets[static_cast<int64_t>(m->t0) * batch];
      i1 = offsets[static_cast<int64_t>(m->t0 + m->T_loc) * batch];
    }
    REC_CUDA(cudaMemcpyAsync(w.indices + i0, indices + i0, sizeof(int) * (i1 - i0), cudaMemcpyHostToDevice, s));
    d_idx = w.indices;
  }
  if (m->F > 0 && !is_device_ptr(dense)) {
    int64_t r0 = 0, r1 = batch;  // sharded: only this rank's item block of the dense rows
    if (sharded) {
      const int Bq = (batch + m->world - 1) / m->world;
      r0 = std::min<int64_t>(batch, static_cast<int64_t>(m->rank) * Bq);
      r1 = std::min<int64_t>(batch, r0 + Bq);
    }
    REC_CUDA(cudaMemcpyAsync(w.dense_f32 + r0 * m->F, dense + r0 * m->F, sizeof(float) * (r1 - r0) * m->F,
                             cudaMemcpyHostToDevice, s));
    d_dense = w.dense_f32;
  }
  const bool ctr_dev = is_device_ptr(ctr);
  // device offsets: offsets[T*B] == nnz is checked on the device (flag -> REC_E_OFFSETS at
  // rec_sync) and the SLS clamps every bag to [0, nnz), so no read leaves the indices
  if (off_dev) launch_check_offsets(d_off, nb, w.flag, s, nnz);
  if (sharded) {  // table-wise over peer memory: every rank enqueues the same global batch
    m->launches += off_dev ? 1 : 0;
    rec_status st = shard_enqueue(m, w, d_dense, d_idx, d_off, batch, nnz);
    if (st != REC_OK) return st;
    REC_CUDA(cudaMemcpyAsync(ctr, w.sh_ctr_gather, sizeof(float) * batch, cudaMemcpyDefault, s));
    return REC_OK;
  }
  launch_dense_to_bf16(d_dense, batch, m->F, m->Fpad, w.dense_bf, s);
  m->launches += off_dev ? 2 : 1;
  rec_status st = forward_enqueue(m, w, d_idx, d_off, batch, nullptr, ctr_dev ? ctr : w.ctr, w.logit,
                                  nullptr, nnz);
  if (st != REC_OK) return st;
  if (!ctr_dev)
    REC_CUDA(cudaMemcpyAsync(ctr, w.ctr, sizeof(float) * batch * m->tasks, cudaMemcpyDeviceToHost, s));
  return REC_OK;
}

rec_status rec_synth_query_async(rec_model_t m, int32_t slot, const int32_t* segs, int32_t nseg,
                                 float* ctr) {
  if (!m) {
    set_error("null argument");
    return REC_E_INVALID_ARG;
  }
  const bool sharded = m->world > 1 && m->shard != REC_SHARD_REPLICA;
  if (sharded && !(m->p2p_slots && m->ws[0].slots[0].var[0].exec)) {
    set_error("synthetic batches on a sharded model need table-wise sharding over peer memory "
              "and fixed pooling");
    return REC_E_UNSUPPORTED;
  }
  if (slot < 0 || slot >= m->nstreams) {
    set_error("slot = %d out of [0, %d)", slot, m->nstreams);
    return REC_E_INVALID_ARG;
  }
  REC_CUDA(cudaSetDevice(m->device));
  Workspace& w = m->ws[slot];
  int B = 0;
  rec_status st = synth_submit(m, w, segs, nseg, &B, nullptr);
  if (st != REC_OK) return st;
  const float* src = sharded ? w.sh_ctr_gather : w.ctr;  // sharded: every rank's CTRs, gathered
  if (ctr && ctr != src)
    REC_CUDA(cudaMemcpyAsync(ctr, src, sizeof(float) * B * m->tasks, cudaMemcpyDefault, w.stream));
  return REC_OK;
}

rec_status rec_synth_query_batches(rec_model_t m, const int32_t* segs, const int64_t* batch_start,
                                   int64_t nbatches, int32_t first_slot) {
  if (!m || !segs || !batch_start || nbatches < 0 || first_slot < 0) {
    set_error("null argument or negative count");
    return REC_E_INVALID_ARG;
  }
  if (m->world > 1 && m->shard != REC_SHARD_REPLICA && !(m->p2p_slots && m->ws[0].slots[0].var[0].exec)) {
    set_error("synthetic batches on a sharded model need table-wise sharding over peer memory "
              "and fixed pooling");
    return REC_E_UNSUPPORTED;
  }
  REC_CUDA(cudaSetDevice(m->device));
  if (!m->pipe.empty()) return pipe_submit(m, segs, batch_start, nbatches, nullptr);
  for (int64_t b = 0; b < nbatches; ++b) {
    Workspace& w = m->ws[(first_slot + b) % m->nstreams];
    const int64_t s0 = batch_start[b], s1 = batch_start[b + 1];
    int B = 0;
    rec_status st = synth_submit(m, w, segs + 3 * s0, static_cast<int>(s1 - s0), &B, nullptr);
    if (st != REC_OK) return st;
  }
  return REC_OK;
}

rec_status rec_sync(rec_model_t m, int32_t slot) {
  if (!m || slot < 0 || slot >= m->nstreams) {
    set_error("bad model or slot");
    return REC_E_INVALID_ARG;
  }
  REC_CUDA(cudaSetDevice(m->device));
  if (m->pipe_active.load()) {  // the slot's batches may run inside a lane graph
    for (auto& L : m->pipe)
      for (int k : L.ws)
        if (k == slot) REC_CUDA(cudaEventSynchronize(L.free));
  }
  return sync_ws(m->ws[slot]);
}

void* rec_stream_handle(rec_model_t m, int32_t slot) {
  if (!m || slot < 0 || slot >= m->nstreams) return nullptr;
  return m->ws[slot].stream;
}

rec_status rec_gen_batch(rec_model_t m, const int32_t* segs, int32_t nseg, int32_t* indices,
                         int32_t* offsets, float* dense) {
  if (!m || !segs || !indices || !offsets || !dense) {
    set_error("null argument");
    return REC_E_INVALID_ARG;
  }
  REC_CUDA(cudaSetDevice(m->device));
  Workspace& w = m->ws[0];
  int B = 0;
  rec_status st = synth_submit(m, w, segs, nseg, &B, w.dense_f32);
  if (st != REC_OK) return st;
  cudaStream_t s = w.stream;
  const int nb = m->T * B;
  REC_CUDA(cudaMemcpyAsync(offsets, w.offsets, sizeof(int) * (nb + 1), cudaMemcpyDefault, s));
  int nnz = 0;
  REC_CUDA(cudaMemcpyAsync(w.flag_host, w.offsets + nb, sizeof(int), cudaMemcpyDeviceToHost, s));
  REC_CUDA(cudaStreamSynchronize(s));
  nnz = *w.flag_host;
  *w.flag_host = 0;
  REC_CUDA(cudaMemcpyAsync(indices, w.indices, sizeof(int) * nnz, cudaMemcpyDefault, s));
  if (m->F > 0)
    REC_CUDA(cudaMemcpyAsync(dense, w.dense_f32, sizeof(float) * B * m->F, cudaMemcpyDefault, s));
  REC_CUDA(cudaStreamSynchronize(s));
  return REC_OK;
}

rec_status rec_bench_mlp(rec_model_t m, int32_t which, int32_t batch, int32_t iters, double* ms_per_iter) {
  if (!m || !ms_per_iter || batch < 1 || batch > m->max_batch || iters < 1 || which < 0 || which > 2) {
    set_error("bad argument");
    return REC_E_INVALID_ARG;
  }
  REC_CUDA(cudaSetDevice(m->device));
  Workspace& w = m->ws[0];
  cudaStream_t s = w.stream;
  cudaEvent_t a, b;
  REC_CUDA(cudaEventCreate(&a));
  REC_CUDA(cudaEventCreate(&b));
  const bool prof = m->prof;
  m->prof = false;
  auto once = [&]() {
    if (which == 0) enqueue_bottom(m, w, s, batch, nullptr, nullptr);
    else if (which == 1) enqueue_interact_top(m, w, s, batch, nullptr, w.ctr, w.logit, nullptr);
    else if (m->arch == REC_ARCH_MTWND)
      launch_concat(w.X, batch, nullptr, m->T, m->D, w.A_top, m->Ktop_pad, m->wide_v, m->tasks, w.wide, s);
    else launch_interact(w.X, batch, nullptr, m->T, m->D, w.A_top, m->Ktop_pad, s);
  };
  for (int i = 0; i < 3; ++i) once();
  REC_CUDA(cudaEventRecord(a, s));
  for (int i = 0; i < iters; ++i) once();
  REC_CUDA(cudaEventRecord(b, s));
  REC_CUDA(cudaEventSynchronize(b));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  *ms_per_iter = ms / iters;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  m->prof = prof;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "rec_bench_mlp");
  return REC_OK;
}

rec_status rec_bench_sls(rec_model_t m, const int32_t* segs, const int64_t* batch_start,
                         int32_t nbatches, int32_t pdl, double* ms_total) {
  if (!m || !segs || !batch_start || nbatches < 1 || !ms_total || (pdl != 0 && pdl != 1)) {
    set_error("bad argument");
    return REC_E_INVALID_ARG;
  }
  if (m->lo != m->hi || (m->world > 1 && m->shard != REC_SHARD_REPLICA)) {
    set_error("rec_bench_sls needs fixed pooling and an unsharded model");
    return REC_E_UNSUPPORTED;
  }
  // host: one batch descriptor per launch (long segment lists go to one device buffer)
  std::vector<SegBatch> sbs(nbatches + 1);
  std::vector<int4> longsegs;
  std::vector<int64_t> long_at(nbatches + 1, -1);
  for (int k = 0; k <= nbatches; ++k) {
    // k == nbatches: warm-up copy of batch 0 with disjoint query ids (rows not reused)
    const int kb = k == nbatches ? 0 : k;
    const int64_t s0 = batch_start[kb], s1 = batch_start[kb + 1];
    const int nseg = static_cast<int>(s1 - s0);
    if (nseg < 1 || nseg > m->max_batch) {
      set_error("batch %d: %d segments", kb, nseg);
      return REC_E_INVALID_ARG;
    }
    int64_t B = 0;
    std::vector<int4> v(nseg);
    for (int i = 0; i < nseg; ++i) {
      const int32_t* sg = segs + 3 * (s0 + i);
      if (sg[2] <= 0 || sg[0] < 0 || sg[1] < 0) {
        set_error("batch %d segment %d: qid/start must be >= 0 and len > 0", kb, i);
        return REC_E_INVALID_ARG;
      }
      v[i] = make_int4(k == nbatches ? (sg[0] ^ 0x40000000) : sg[0], sg[1], sg[2], static_cast<int>(B));
      B += sg[2];
    }
    if (B > m->max_batch) {
      set_error("batch %d: %lld items exceed max_batch %d", kb, (long long)B, m->max_batch);
      return REC_E_INVALID_ARG;
    }
    SegBatch& sb = sbs[k];
    sb = SegBatch{};
    sb.B = static_cast<int>(B);
    sb.nseg = nseg;
    if (nseg > kParamSegs) {
      long_at[k] = static_cast<int64_t>(longsegs.size());
      longsegs.insert(longsegs.end(), v.begin(), v.end());
    } else {
      std::copy(v.begin(), v.end(), sb.seg);
    }
  }
  REC_CUDA(cudaSetDevice(m->device));
  REC_CUDA(cudaDeviceSynchronize());
  int4* dlong = nullptr;
  if (!longsegs.empty()) {
    REC_CUDA(cudaMalloc(reinterpret_cast<void**>(&dlong), sizeof(int4) * longsegs.size()));
    REC_CUDA(cudaMemcpy(dlong, longsegs.data(), sizeof(int4) * longsegs.size(), cudaMemcpyHostToDevice));
  }
  for (int k = 0; k <= nbatches; ++k) sbs[k].gsegs = long_at[k] >= 0 ? dlong + long_at[k] : nullptr;
  Workspace& w = m->ws[0];
  SlsSynthArgs sa = w.slots[0].sa;
  sa.pdl = pdl && !sa.tma;
  cudaEvent_t a, b;
  REC_CUDA(cudaEventCreate(&a));
  REC_CUDA(cudaEventCreate(&b));
  for (int i = 0; i < 3; ++i) launch_sls_synth(sbs[nbatches], sa, w.stream);
  REC_CUDA(cudaEventRecord(a, w.stream));
  for (int k = 0; k < nbatches; ++k) launch_sls_synth(sbs[k], sa, w.stream);
  REC_CUDA(cudaEventRecord(b, w.stream));
  REC_CUDA(cudaEventSynchronize(b));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  *ms_total = ms;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (dlong) cudaFree(dlong);
  m->launches += 3 + nbatches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "rec_bench_sls");
  return REC_OK;
}

rec_status rec_bench_sls_caller(rec_model_t m, const int32_t* indices, const int32_t* offsets,
                                int32_t batch, int32_t nbatches, int64_t idx_stride, double* ms_total) {
  if (!m || !indices || !offsets || batch < 1 || batch > m->max_batch || nbatches < 1 ||
      idx_stride < 0 || !ms_total) {
    set_error("bad argument");
    return REC_E_INVALID_ARG;
  }
  if (m->world > 1 && m->shard != REC_SHARD_REPLICA) {
    set_error("rec_bench_sls_caller needs an unsharded model");
    return REC_E_UNSUPPORTED;
  }
  if (!is_device_ptr(indices) || !is_device_ptr(offsets)) {
    set_error("rec_bench_sls_caller: indices and offsets must be device memory");
    return REC_E_INVALID_ARG;
  }
  REC_CUDA(cudaSetDevice(m->device));
  REC_CUDA(cudaDeviceSynchronize());
  Workspace& w = m->ws[0];
  const int T = m->T, D = m->D;
  const int64_t ostride = static_cast<int64_t>(T) * batch + 1;
  auto one = [&](int k) {
    launch_sls(m->tables, m->d_tab_off, m->row_stride, m->d_rows, indices + k * idx_stride,
               offsets + k * ostride, batch, nullptr, T, D, w.X, (T + 1) * D, 1, w.flag, w.stream, 0,
               0x7fffffff, static_cast<int>(std::min<int64_t>(idx_stride, 0x7fffffff)));
  };
  cudaEvent_t a, b;
  REC_CUDA(cudaEventCreate(&a));
  REC_CUDA(cudaEventCreate(&b));
  for (int i = 0; i < 3; ++i) one(0);
  REC_CUDA(cudaEventRecord(a, w.stream));
  for (int k = 0; k < nbatches; ++k) one(k);
  REC_CUDA(cudaEventRecord(b, w.stream));
  REC_CUDA(cudaEventSynchronize(b));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  *ms_total = ms;
  m->launches += 3 + nbatches;
  rec_status st = sync_ws(w);  // the device error flag (OOB / offsets) of the timed launches
  if (st != REC_OK) return st;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "rec_bench_sls_caller");
  return REC_OK;
}

rec_status rec_debug_chain_timeline(rec_model_t m, int32_t which, int32_t batch, int64_t* out16) {
  if (!m || !out16 || batch < 1 || batch > m->max_batch || which < 0 || which > 1) {
    set_error("bad argument");
    return REC_E_INVALID_ARG;
  }
  if (!(which == 0 ? m->chain_bottom : m->chain_top)) {
    set_error("no fused chain for this MLP");
    return REC_E_UNSUPPORTED;
  }
  REC_CUDA(cudaSetDevice(m->device));
  Workspace& w = m->ws[0];
  unsigned long long* d = nullptr;
  REC_CUDA(cudaMalloc(reinterpret_cast<void**>(&d), 16 * sizeof(unsigned long long)));
  REC_CUDA(cudaMemset(d, 0, 16 * sizeof(unsigned long long)));
  ChainArgs a = which == 0 ? m->chain_bottom_args : m->chain_top_args;
  a.M = batch;
  a.dM = nullptr;
  a.out_f32 = w.X;
  a.ldo = (m->T + 1) * m->D;
  a.ctr = w.ctr;
  a.logit = w.logit;
  a.dbg = d;
#ifdef REC_DEBUG_KNOBS
  if (const char* e = getenv("REC_DBG_EPI")) a.dbg_mode = atoi(e);  // diagnostic build only
#endif
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0, w.stream);
    launch_mlp_chain(which == 0 ? w.chain_bottom : w.chain_top, a, w.stream);
    cudaEventRecord(e1, w.stream);
  }
  REC_CUDA(cudaStreamSynchronize(w.stream));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  unsigned long long h[16];
  REC_CUDA(cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost));
  cudaFree(d);
  for (int i = 0; i < 16; ++i) out16[i] = static_cast<int64_t>(h[i]);
  out16[14] = static_cast<int64_t>(ms * 1e6);  // event time of the last launch (ns)
  return REC_OK;
}

rec_status rec_profile(rec_model_t m, int32_t enable) {
  if (!m) {
    set_error("null model");
    return REC_E_INVALID_ARG;
  }
  for (auto& w : m->ws) REC_CUDA(cudaStreamSynchronize(w.stream));
  prof_collect(m);
  for (int k = 0; k < 4; ++k) {
    m->prof_ms[k] = 0;
    m->prof_n[k] = 0;
    for (auto& w : m->ws) w.host_ns[k] = 0;
  }
  m->prof = enable != 0;
  return REC_OK;
}

rec_status rec_profile_read(rec_model_t m, int32_t kernel, double* total_ms, int64_t* launches) {
  if (!m || kernel < 0 || kernel > 8 || !total_ms || !launches) {
    set_error("bad argument");
    return REC_E_INVALID_ARG;
  }
  if (kernel == 4) {  // all kernels launched by this handle (count only)
    *total_ms = 0.0;
    *launches = m->launches;
    return REC_OK;
  }
  if (kernel >= 5 && kernel <= 8) {  // host time of the synthetic submit path
    double ns = 0;
    for (auto& w : m->ws) ns += w.host_ns[kernel - 5];
    *total_ms = ns * 1e-6;
    *launches = 0;
    return REC_OK;
  }
  for (auto& w : m->ws) REC_CUDA(cudaStreamSynchronize(w.stream));
  prof_collect(m);
  *total_ms = m->prof_ms[kernel];
  *launches = m->prof_n[kernel];
  return REC_OK;
}

}  // extern "C"
