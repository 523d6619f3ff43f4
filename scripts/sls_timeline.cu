// sls_timeline.cu — diagnostic (not product): per-warp %globaltimer timeline of one
// synthetic-index SLS launch (k_sls_synth, RMC1 shapes) to split a launch into ramp
// (CTA start spread), first-round latency, bulk and drain.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DREC_SLS_TIMELINE \
//        -I include -I paper_2203_07424_b200/csrc scripts/sls_timeline.cu -o build/sls_timeline
//   build/sls_timeline B L [rows]
#include <algorithm>
#include <string>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2203_07424_b200/csrc/k_sls.cu"

using namespace rec;

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));   \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

__global__ void k_empty_big(const __grid_constant__ SegBatch sb, const SlsSynthArgs a) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && sb.B < 0) *a.dB = 1;
}
__global__ void k_empty_small(int* p, int B) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && B < 0) *p = 1;
}

static double pct(std::vector<double> v, double p) {
  if (v.empty()) return 0;
  std::sort(v.begin(), v.end());
  return v[std::min(v.size() - 1, static_cast<size_t>(p * (v.size() - 1)))];
}

int main(int argc, char** argv) {
  if (argc > 1 && std::string(argv[1]) == "gap") {  // launch-gap probe: empty kernels
    SegBatch sb{};
    SlsSynthArgs a{};
    int* p;
    CK(cudaMalloc(&p, 4));
    a.dB = p;
    sb.B = 1;
    cudaStream_t s;
    CK(cudaStreamCreate(&s));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int grid : {1, 148, 640, 2560}) {
      float ms_big = 0, ms_small = 0;
      for (int rep = 0; rep < 2; ++rep) {
        CK(cudaEventRecord(e0, s));
        for (int i = 0; i < 200; ++i) k_empty_big<<<grid, 128, 0, s>>>(sb, a);
        CK(cudaEventRecord(e1, s));
        CK(cudaStreamSynchronize(s));
        CK(cudaEventElapsedTime(&ms_big, e0, e1));
        CK(cudaEventRecord(e0, s));
        for (int i = 0; i < 200; ++i) k_empty_small<<<grid, 128, 0, s>>>(p, 1);
        CK(cudaEventRecord(e1, s));
        CK(cudaStreamSynchronize(s));
        CK(cudaEventElapsedTime(&ms_small, e0, e1));
      }
      printf("{\"grid\": %d, \"us_per_launch_2KB_params\": %.2f, \"us_per_launch_small\": %.2f}\n", grid,
             ms_big * 1e3 / 200, ms_small * 1e3 / 200);
    }
    return 0;
  }
  const int B = argc > 1 ? atoi(argv[1]) : 1024;
  const int L = argc > 2 ? atoi(argv[2]) : 80;
  const int64_t R = argc > 3 ? atoll(argv[3]) : 1000000;
  const int T = 10, D = 32;
  float* tables;
  CK(cudaMalloc(&tables, sizeof(float) * R * T * D));
  CK(cudaMemset(tables, 0, sizeof(float) * R * T * D));
  int64_t h_off[T], h_rows[T];
  for (int t = 0; t < T; ++t) {
    h_off[t] = int64_t(t) * D;
    h_rows[t] = R;
  }
  int64_t *d_off, *d_rows;
  float* X;
  int* dB;
  CK(cudaMalloc(&d_off, sizeof(h_off)));
  CK(cudaMalloc(&d_rows, sizeof(h_rows)));
  CK(cudaMalloc(&X, sizeof(float) * B * (T + 1) * D));
  CK(cudaMalloc(&dB, sizeof(int)));
  CK(cudaMemcpy(d_off, h_off, sizeof(h_off), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_rows, h_rows, sizeof(h_rows), cudaMemcpyHostToDevice));
  SegBatch sb{};
  sb.B = B;
  sb.nseg = 1;
  sb.seg[0] = make_int4(7, 0, B, 0);
  SlsSynthArgs a{};
  a.tables = tables;
  a.tab_off = d_off;
  a.row_stride = int64_t(T) * D;
  a.rows = d_rows;
  a.cap = B;
  a.T = T;
  a.D = D;
  a.L = L;
  a.index_dist = 0;
  a.k0 = 0x12345678u;
  a.k1 = 0x9abcdef0u;
  a.X = X;
  a.x_stride = (T + 1) * D;
  a.dB = dB;
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int i = 0; i < 5; ++i) launch_sls_synth(sb, a, s);
  CK(cudaEventRecord(e0, s));
  launch_sls_synth(sb, a, s);
  CK(cudaEventRecord(e1, s));
  CK(cudaStreamSynchronize(s));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  const int warps = (T * B * 8 + 31) / 32;  // LANES = 8 at D = 32
  std::vector<unsigned long long> h(4 * 65536);
  CK(cudaMemcpyFromSymbol(h.data(), g_sls_tl, sizeof(unsigned long long) * h.size()));
  unsigned long long t0 = ~0ull, tend = 0;
  for (int w = 0; w < warps; ++w) {
    t0 = std::min(t0, h[4 * w]);
    tend = std::max(tend, h[4 * w + 3]);
  }
  std::vector<double> entry, setup, first, end, span;
  for (int w = 0; w < warps; ++w) {
    entry.push_back((h[4 * w] - t0) * 1e-3);
    setup.push_back((h[4 * w + 1] - h[4 * w]) * 1e-3);
    first.push_back((h[4 * w + 2] - h[4 * w + 1]) * 1e-3);
    end.push_back((h[4 * w + 3] - t0) * 1e-3);
    span.push_back((h[4 * w + 3] - h[4 * w]) * 1e-3);
  }
  const double bytes = double(B) * T * (L * D * 4 + D * 4);
  float b2b[2] = {0, 0};
  for (int pdl = 0; pdl < 2; ++pdl) {
    a.pdl = pdl;
    for (int i = 0; i < 3; ++i) launch_sls_synth(sb, a, s);
    CK(cudaEventRecord(e0, s));
    for (int i = 0; i < 50; ++i) launch_sls_synth(sb, a, s);
    CK(cudaEventRecord(e1, s));
    CK(cudaStreamSynchronize(s));
    CK(cudaEventElapsedTime(&b2b[pdl], e0, e1));
    b2b[pdl] *= 1e3f / 50;
  }
  printf("{\"b2b_us\": %.2f, \"b2b_pdl_us\": %.2f, \"b2b_GBps\": %.1f, \"b2b_pdl_GBps\": %.1f}\n",
         b2b[0], b2b[1], bytes / (b2b[0] * 1e-6) / 1e9, bytes / (b2b[1] * 1e-6) / 1e9);
  printf("{\"B\": %d, \"L\": %d, \"rows\": %lld, \"event_us\": %.2f, \"kernel_span_us\": %.2f, "
         "\"GBps_span\": %.1f, \"warps\": %d, "
         "\"entry_us\": [%.2f, %.2f, %.2f], \"setup_us\": [%.2f, %.2f, %.2f], "
         "\"first_round_us\": [%.2f, %.2f, %.2f], \"end_us\": [%.2f, %.2f, %.2f, %.2f], "
         "\"warp_span_us\": [%.2f, %.2f, %.2f]}\n",
         B, L, (long long)R, ms * 1e3, (tend - t0) * 1e-3, bytes / ((tend - t0) * 1e-9) / 1e9, warps,
         pct(entry, 0.5), pct(entry, 0.9), pct(entry, 1.0), pct(setup, 0.5), pct(setup, 0.9),
         pct(setup, 1.0), pct(first, 0.1), pct(first, 0.5), pct(first, 0.9), pct(end, 0.0),
         pct(end, 0.5), pct(end, 0.9), pct(end, 1.0), pct(span, 0.1), pct(span, 0.5),
         pct(span, 0.9));
  return 0;
}
