// gemm2sm_test.cu — diagnostic (not product): the CTA-pair tcgen05 GEMM (k_gemm_2sm) against
// the single-CTA kernel on the same operands, launched directly (no graph), plus timing.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        -I paper_2203_07424_b200/csrc scripts/gemm2sm_test.cu -o build/gemm2sm_test -lcuda
//   build/gemm2sm_test M N K
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2203_07424_b200/csrc/k_gemm.cu"

using namespace rec;

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));   \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)


__global__ void __cluster_dims__(1, 2, 1) k_probe_y(int* p) {
  extern __shared__ int sm_[];
  if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) p[0] = sm_[0] * 0 + 1;
}
__global__ void __cluster_dims__(2, 1, 1) k_probe_x(int* p) {
  extern __shared__ int sm_[];
  if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) p[0] = sm_[0] * 0 + 2;
}

int main(int argc, char** argv) {
  {
    int* p;
    CK(cudaMalloc(&p, 4));
    for (int smem : {0, 65536, 132352}) {
      cudaFuncSetAttribute(k_probe_y, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaFuncSetAttribute(k_probe_x, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      k_probe_y<<<dim3(2, 512), 128, smem>>>(p);
      cudaError_t ey = cudaDeviceSynchronize();
      cudaGetLastError();
      k_probe_x<<<dim3(512, 2), 128, smem>>>(p);
      cudaError_t ex = cudaDeviceSynchronize();
      cudaGetLastError();
      printf("probe smem %d: y-cluster %s, x-cluster %s\n", smem, cudaGetErrorString(ey), cudaGetErrorString(ex));
    }
  }
  const int M = argc > 1 ? atoi(argv[1]) : 65536;
  const int N = argc > 2 ? atoi(argv[2]) : 512;
  const int K = argc > 3 ? atoi(argv[3]) : 2560;
  std::vector<__nv_bfloat16> hA(size_t(M) * K), hW(size_t(N) * K);
  uint32_t x = 12345;
  auto rnd = [&]() {
    x = x * 1664525u + 1013904223u;
    return static_cast<float>(static_cast<int>((x >> 24) & 0xFF) - 128) / 128.f;
  };
  for (auto& v : hA) v = __float2bfloat16(rnd());
  for (auto& v : hW) v = __float2bfloat16(rnd() * 0.0625f);
  __nv_bfloat16 *A, *Wt, *O1, *O2;
  float* bias;
  CK(cudaMalloc(&A, hA.size() * 2));
  CK(cudaMalloc(&Wt, hW.size() * 2));
  CK(cudaMalloc(&O1, size_t(M) * N * 2));
  CK(cudaMalloc(&O2, size_t(M) * N * 2));
  CK(cudaMalloc(&bias, N * 4));
  CK(cudaMemset(bias, 0, N * 4));
  CK(cudaMemcpy(A, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(Wt, hW.data(), hW.size() * 2, cudaMemcpyHostToDevice));
  CUtensorMap ta, tw, tw128;
  if (!encode_tmap_bf16(&ta, A, M, K, K, 128) || !encode_tmap_bf16(&tw, Wt, N, K, K, 256) ||
      !encode_tmap_bf16(&tw128, Wt, N, K, K, 128)) {
    fprintf(stderr, "tensor map encode failed\n");
    return 1;
  }
  gemm_prepare();
  {
    GemmArgs t{};
    t.M = M; t.N = N; t.K = K; t.mode = GEMM_OUT_BF16; t.ldo = N;
    __nv_bfloat16* Ot;
    float* bt;
    CK(cudaMalloc(&Ot, size_t(M) * N * 2));
    CK(cudaMalloc(&bt, N * 4));
    t.out_bf16 = Ot; t.bias = bt;
    for (int st : {1, 2, 4}) {
      const size_t sm = size_t(st) * 32768 + 1280;
      k_gemm_2sm<256><<<dim3(2, 2, ((M + 127) / 128 + (((M + 127) / 128) & 1)) / 2), 128, sm>>>(ta, tw128, t, st);
      cudaError_t e1 = cudaGetLastError();
      cudaError_t e2 = cudaDeviceSynchronize();
      printf("direct 2sm stages %d smem %zu: launch %s, run %s\n", st, sm, cudaGetErrorString(e1), cudaGetErrorString(e2));
      if (e2 != cudaSuccess) return 1;
    }
  }
  {
    cudaFuncAttributes fa;
    CK(cudaFuncGetAttributes(&fa, k_gemm_2sm<256>));
    printf("k_gemm_2sm: maxDynSmem %d static %zu regs %d maxThreads %d clusterDims %d,%d,%d reqd %d\n",
           fa.maxDynamicSharedSizeBytes, fa.sharedSizeBytes, fa.numRegs, fa.maxThreadsPerBlock,
           fa.requiredClusterWidth, fa.requiredClusterHeight, fa.requiredClusterDepth,
           fa.clusterDimMustBeSet);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2, 512);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = 4 * (16384 + 16384) + 1280;
    int ncl = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, k_gemm_2sm<256>, &cfg);
    printf("max active clusters: %d (%s)\n", ncl, cudaGetErrorString(e));
  }
  GemmArgs a{};
  a.M = M;
  a.N = N;
  a.K = K;
  a.bias = bias;
  a.relu = 0;
  a.mode = GEMM_OUT_BF16;
  a.ldo = N;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float ms1 = 0, ms2 = 0;
  a.out_bf16 = O1;
  g_gemm_2sm = 0;
  for (int i = 0; i < 3; ++i) launch_gemm_tc(&ta, &tw, a, 0, &tw128);
  CK(cudaEventRecord(e0));
  for (int i = 0; i < 20; ++i) launch_gemm_tc(&ta, &tw, a, 0, &tw128);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  CK(cudaGetLastError());
  CK(cudaEventElapsedTime(&ms1, e0, e1));
  a.out_bf16 = O2;
  g_gemm_2sm = argc > 4 ? atoi(argv[4]) : 1;
  launch_gemm_tc(&ta, &tw, a, 0, &tw128);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  for (int i = 0; i < 2; ++i) launch_gemm_tc(&ta, &tw, a, 0, &tw128);
  CK(cudaEventRecord(e0));
  for (int i = 0; i < 20; ++i) launch_gemm_tc(&ta, &tw, a, 0, &tw128);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  CK(cudaGetLastError());
  CK(cudaEventElapsedTime(&ms2, e0, e1));
  std::vector<__nv_bfloat16> h1(size_t(M) * N), h2(size_t(M) * N);
  CK(cudaMemcpy(h1.data(), O1, h1.size() * 2, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h2.data(), O2, h2.size() * 2, cudaMemcpyDeviceToHost));
  size_t diff = 0;
  double maxd = 0;
  for (size_t i = 0; i < h1.size(); ++i) {
    const float d = fabsf(__bfloat162float(h1[i]) - __bfloat162float(h2[i]));
    if (d != 0.f) ++diff;
    if (d > maxd) maxd = d;
  }
  const double flop = 2.0 * M * N * K;
  printf("{\"M\": %d, \"N\": %d, \"K\": %d, \"single_us\": %.2f, \"pair_us\": %.2f, "
         "\"single_tflops\": %.1f, \"pair_tflops\": %.1f, \"mismatches\": %zu, \"max_abs_diff\": %g}\n",
         M, N, K, ms1 * 1e3 / 20, ms2 * 1e3 / 20, flop / (ms1 / 20 * 1e-3) / 1e12,
         flop / (ms2 / 20 * 1e-3) / 1e12, diff, maxd);
  return 0;
}
