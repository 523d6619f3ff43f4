// pipe.cu — S-D pipeline lanes ("S-D pipeline": the
// SparseNet and DenseNet stages of consecutive batches overlap instead of running back to
// back).  B200 form: one captured graph per lane runs N batches; their SLS kernels form a
// programmatic-dependent-launch chain on the lane stream (a launch's row gathers overlap the
// previous launch's drain; the writes wait for it), each batch's dense features and bottom
// MLP run on its workspace's branch stream, and its interaction + top MLP on a third stream
// after both halves.  Lanes alternate so one lane's fill/drain overlaps the other's bulk.
//
// The per-batch arithmetic is exactly the slot-graph chain's (same kernels, same buffers of
// the batch's workspace): CTRs are bit-identical to rec_synth_query_async
// (tests/test_gpu_serving.py::test_pipeline_matches_slots).
#include <chrono>
#include <cstring>

#include "model.h"

using namespace rec;

namespace rec {

// Host segment list -> by-value batch descriptor (long lists through w's pinned staging and
// an H2D copy on `s`).  *B_out = items.
static rec_status build_segbatch(rec_model_s* m, Workspace& w, const int32_t* segs, int nseg,
                                 SegBatch& sb, cudaStream_t s, int* B_out) {
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
  sb.B = static_cast<int>(B);
  sb.nseg = nseg;
  sb.gsegs = w.gsegs;
  int4* dst = sb.seg;
  if (nseg > kParamSegs) {
    REC_CUDA(cudaEventSynchronize(w.pin_free));
    dst = reinterpret_cast<int4*>(w.pin);
  }
  int row = 0;
  for (int i = 0; i < nseg; ++i) {
    dst[i] = make_int4(segs[3 * i], segs[3 * i + 1], segs[3 * i + 2], row);
    row += segs[3 * i + 2];
  }
  if (nseg > kParamSegs) {
    REC_CUDA(cudaMemcpyAsync(w.gsegs, w.pin, sizeof(int4) * nseg, cudaMemcpyHostToDevice, s));
    REC_CUDA(cudaEventRecord(w.pin_free, s));
  }
  *B_out = static_cast<int>(B);
  return REC_OK;
}

static rec_status pipe_capture(rec_model_s* m, PipeLane& L) {
  const int N = static_cast<int>(L.ws.size());
  Workspace& head = m->ws[L.ws[0]];
  cudaStream_t S = head.stream;
  L.sls_node.assign(N, nullptr);
  L.dense_node.assign(N, nullptr);
  const int64_t before = m->launches;
  REC_CUDA(cudaStreamBeginCapture(S, cudaStreamCaptureModeThreadLocal));
  auto body = [&]() -> rec_status {
    REC_CUDA(cudaEventRecord(head.ev_fork, S));
    for (int i = 0; i < N; ++i) {
      Workspace& w = m->ws[L.ws[i]];
      REC_CUDA(cudaStreamWaitEvent(w.stream_b, head.ev_fork, 0));
      REC_CUDA(cudaStreamWaitEvent(w.stream_c, head.ev_fork, 0));
    }
    for (int i = 0; i < N; ++i) {
      Workspace& w = m->ws[L.ws[i]];
      // DenseNet half: dense features -> bottom MLP (branch stream)
      launch_gen_dense_seg(*L.sb[i], L.ga[i], w.stream_b);
      size_t n = 0;
      const cudaGraphNode_t* d = last_node(w.stream_b, &n);
      if (n != 1) {
        set_error("pipeline capture: dense node not found");
        return REC_E_CUDA;
      }
      L.dense_node[i] = d[0];
      enqueue_bottom(m, w, w.stream_b, w.cap, w.dB, nullptr);
      REC_CUDA(cudaEventRecord(w.ev_join, w.stream_b));
      // SparseNet half: SLS on the lane stream, PDL-chained to the previous batch's SLS
      launch_sls_synth(*L.sb[i], L.sa[i], S);
      d = last_node(S, &n);
      if (n != 1) {
        set_error("pipeline capture: SLS node not found");
        return REC_E_CUDA;
      }
      L.sls_node[i] = d[0];
      REC_CUDA(cudaEventRecord(w.ev_sls, S));
      m->launches += 2;
      // join: interaction + top MLP once both halves of batch i are done
      REC_CUDA(cudaStreamWaitEvent(w.stream_c, w.ev_sls, 0));
      REC_CUDA(cudaStreamWaitEvent(w.stream_c, w.ev_join, 0));
      enqueue_interact_top(m, w, w.stream_c, w.cap, w.dB, w.ctr, w.logit, nullptr);
      REC_CUDA(cudaEventRecord(w.ev_done, w.stream_c));
    }
    for (int i = 0; i < N; ++i) REC_CUDA(cudaStreamWaitEvent(S, m->ws[L.ws[i]].ev_done, 0));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "pipeline capture");
    return REC_OK;
  };
  rec_status st = body();
  cudaGraph_t g = nullptr;
  cudaError_t ce = cudaStreamEndCapture(S, &g);
  L.kernels = static_cast<int>(m->launches - before);
  m->launches = before;
  if (st != REC_OK) {
    if (g) cudaGraphDestroy(g);
    return st;
  }
  if (ce != cudaSuccess) return cuda_fail(ce, "cudaStreamEndCapture (pipeline)");
  L.graph = g;
  ce = cudaGraphInstantiate(&L.exec, g, cudaGraphInstantiateFlagUseNodePriority);
  if (ce != cudaSuccess) return cuda_fail(ce, "cudaGraphInstantiate (pipeline)");
  return REC_OK;
}

void pipe_destroy(rec_model_s* m) {
  for (auto& L : m->pipe) {
    if (L.free) cudaEventSynchronize(L.free);
    if (L.exec) cudaGraphExecDestroy(L.exec);
    if (L.graph) cudaGraphDestroy(L.graph);
    if (L.free) cudaEventDestroy(L.free);
    for (auto* p : L.sb) delete p;
  }
  m->pipe.clear();
  m->pipe_active.store(0);
}

rec_status pipe_leave(rec_model_s* m) {
  for (auto& L : m->pipe) REC_CUDA(cudaEventSynchronize(L.free));
  m->pipe_active.store(0, std::memory_order_release);
  return REC_OK;
}

static rec_status pipe_enter(rec_model_s* m) {
  if (m->pipe_active.load()) return REC_OK;
  // slot graphs and rec_query work may still use the workspaces' buffers
  for (auto& w : m->ws) {
    REC_CUDA(cudaStreamSynchronize(w.stream));
    REC_CUDA(cudaStreamSynchronize(w.stream_b));
    REC_CUDA(cudaStreamSynchronize(w.stream_c));
  }
  m->pipe_active.store(1, std::memory_order_release);
  return REC_OK;
}

rec_status pipe_submit(rec_model_s* m, const int32_t* segs, const int64_t* batch_start,
                       int64_t nbatches, float* ctr_out) {
  const int lanes = static_cast<int>(m->pipe.size());
  const int N = static_cast<int>(m->pipe[0].ws.size());
  int64_t b = 0, item0 = 0;
  if (nbatches >= N) {
    rec_status st = pipe_enter(m);
    if (st != REC_OK) return st;
  }
  for (; nbatches - b >= N; b += N) {
    PipeLane& L = m->pipe[m->pipe_next];
    m->pipe_next = (m->pipe_next + 1) % lanes;
    Workspace& head = m->ws[L.ws[0]];
    const double t0 = std::chrono::duration<double, std::nano>(
                          std::chrono::steady_clock::now().time_since_epoch()).count();
    REC_CUDA(cudaEventSynchronize(L.free));
    const double t1 = std::chrono::duration<double, std::nano>(
                          std::chrono::steady_clock::now().time_since_epoch()).count();
    int Bs[64];
    for (int i = 0; i < N; ++i) {
      const int64_t s0 = batch_start[b + i], s1 = batch_start[b + i + 1];
      rec_status st = build_segbatch(m, m->ws[L.ws[i]], segs + 3 * s0, static_cast<int>(s1 - s0),
                                     *L.sb[i], head.stream, &Bs[i]);
      if (st != REC_OK) return st;
      dim3 grid, block;
      size_t smem = 0;
      cudaKernelNodeParams kp{};
      void* args_s[2] = {L.sb[i], &L.sa[i]};
      kp.func = sls_synth_kernel(L.sa[i], &grid, &block, &smem);
      kp.gridDim = grid;
      kp.blockDim = block;
      kp.sharedMemBytes = static_cast<unsigned>(smem);
      kp.kernelParams = args_s;
      REC_CUDA(cudaGraphExecKernelNodeSetParams(L.exec, L.sls_node[i], &kp));
      cudaKernelNodeParams kd{};
      void* args_d[2] = {L.sb[i], &L.ga[i]};
      kd.func = gen_dense_seg_kernel(L.ga[i], &grid, &block);
      kd.gridDim = grid;
      kd.blockDim = block;
      kd.kernelParams = args_d;
      REC_CUDA(cudaGraphExecKernelNodeSetParams(L.exec, L.dense_node[i], &kd));
    }
    const double t2 = std::chrono::duration<double, std::nano>(
                          std::chrono::steady_clock::now().time_since_epoch()).count();
    REC_CUDA(cudaGraphLaunch(L.exec, head.stream));
    const double t3 = std::chrono::duration<double, std::nano>(
                          std::chrono::steady_clock::now().time_since_epoch()).count();
    if (ctr_out) {
      for (int i = 0; i < N; ++i) {
        REC_CUDA(cudaMemcpyAsync(ctr_out + item0 * m->tasks, m->ws[L.ws[i]].ctr,
                                 sizeof(float) * Bs[i] * m->tasks, cudaMemcpyDeviceToDevice, head.stream));
        item0 += Bs[i];
      }
    }
    REC_CUDA(cudaEventRecord(L.free, head.stream));
    head.host_ns[0] += t2 - t1;
    head.host_ns[1] += t3 - t2;
    head.host_ns[2] += t1 - t0;
    head.host_ns[3] += t3 - t0;
    m->launches += L.kernels;
  }
  // remainder (< N batches): per-stream slot graphs
  for (int64_t k = 0; b < nbatches; ++b, ++k) {
    Workspace& w = m->ws[k % m->nstreams];
    const int64_t s0 = batch_start[b], s1 = batch_start[b + 1];
    int B = 0;
    rec_status st = synth_submit(m, w, segs + 3 * s0, static_cast<int>(s1 - s0), &B, nullptr);
    if (st != REC_OK) return st;
    if (ctr_out) {
      REC_CUDA(cudaMemcpyAsync(ctr_out + item0 * m->tasks, w.ctr, sizeof(float) * B * m->tasks,
                               cudaMemcpyDeviceToDevice, w.stream));
      item0 += B;
    }
  }
  return REC_OK;
}

}  // namespace rec

rec_status rec_set_pipeline(rec_model_t m, int32_t lanes) {
  if (!m) {
    set_error("null model");
    return REC_E_INVALID_ARG;
  }
  if (lanes < 0 || (lanes > 0 && (m->nstreams % lanes != 0 || m->nstreams / lanes < 2 ||
                                  m->nstreams / lanes > 64))) {
    set_error("lanes = %d: must be 0 or divide streams = %d into groups of 2..64", lanes, m->nstreams);
    return REC_E_INVALID_ARG;
  }
  if (lanes > 0 && (m->lo != m->hi || m->F == 0 || (m->world > 1 && m->shard != REC_SHARD_REPLICA))) {
    set_error("pipeline lanes need fixed pooling, a bottom MLP and an unsharded model");
    return REC_E_UNSUPPORTED;
  }
  REC_CUDA(cudaSetDevice(m->device));
  REC_CUDA(cudaDeviceSynchronize());
  pipe_destroy(m);
  if (lanes == 0) return REC_OK;
  const int N = m->nstreams / lanes;
  const bool prof = m->prof;
  m->prof = false;  // lane graphs carry no profiling events
  m->pipe.resize(lanes);
  for (int l = 0; l < lanes; ++l) {
    PipeLane& L = m->pipe[l];
    REC_CUDA(cudaEventCreateWithFlags(&L.free, cudaEventDisableTiming));
    REC_CUDA(cudaEventRecord(L.free, m->ws[l * N].stream));
    for (int i = 0; i < N; ++i) {
      const int k = l * N + i;
      L.ws.push_back(k);
      L.sb.push_back(new SegBatch{});
      L.sb.back()->B = 1;
      L.sb.back()->nseg = 1;
      L.sb.back()->gsegs = m->ws[k].gsegs;
      L.sb.back()->seg[0] = make_int4(0, 0, 1, 0);
      L.ga.emplace_back();
      L.sa.emplace_back();
      fill_genargs(m, m->ws[k], L.ga.back(), L.sa.back(), nullptr);
      L.sa.back().dense_bf = nullptr;  // lanes generate dense features on the branch stream
    }
    rec_status st = pipe_capture(m, L);
    if (st != REC_OK) {
      m->prof = prof;
      pipe_destroy(m);
      return st;
    }
  }
  m->prof = prof;
  m->pipe_next = 0;
  return REC_OK;
}

rec_status rec_synth_query_pipeline(rec_model_t m, const int32_t* segs, const int64_t* batch_start,
                                    int64_t nbatches, float* ctr_out) {
  if (!m || !segs || !batch_start || nbatches < 0) {
    set_error("null argument or negative count");
    return REC_E_INVALID_ARG;
  }
  if (m->pipe.empty()) {
    set_error("no pipeline lanes: call rec_set_pipeline first");
    return REC_E_INVALID_ARG;
  }
  REC_CUDA(cudaSetDevice(m->device));
  return pipe_submit(m, segs, batch_start, nbatches, ctr_out);
}
