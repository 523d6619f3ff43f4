// k_interact.cu — pairwise dot-product feature interaction.
//
// Paper: the SparseNet / DenseNet join is shown only in Fig. rec_char(a) and by
// citing DLRM; reading R1 takes DLRM's dot interaction without self pairs:
//   X_b = [x_b; p_b,0; ...; p_b,T-1]  ((T+1) x D, fp32),  Z = X_b X_b^T,
//   A_top[b] = bf16([x_b, Z(1,0), Z(2,0), Z(2,1), ..., Z(T,T-1), 0-pad])
// which is the A operand (K-major bf16 row) of the first top-MLP GEMM.
//
// One warp per item: X_b (<= 41 x 64 fp32 for RMC2) is staged in shared memory with a
// padded row pitch (D+1 floats, conflict-free column reads); lanes own pairs; each dot is a
// sequential fp32 FMA chain.  (T+1)^2/2 * D FMAs per item is < 1 % of the item's SLS time.
#include "common.cuh"
#include "kernels.h"

namespace rec {

__global__ void k_interact(const float* __restrict__ X, int B, const int* __restrict__ dB, int T,
                           int D, __nv_bfloat16* __restrict__ A, int ld, int warps_per_cta) {
  extern __shared__ float sm[];
  if (dB) B = *dB;
  if (static_cast<int>(blockIdx.x) * warps_per_cta >= B) return;
  const int rows = T + 1, pitch = D + 1, npairs = T * (T + 1) / 2;
  uint8_t* pi = reinterpret_cast<uint8_t*>(sm);
  uint8_t* pj = pi + npairs;
  float* xs_all = sm + (2 * npairs + 15) / 4 + 4;
  for (int p = threadIdx.x; p < npairs; p += blockDim.x) {
    int i = 1, base = 0;
    while (base + i <= p) {  // row i holds pairs [i(i-1)/2, i(i+1)/2)
      base += i;
      ++i;
    }
    pi[p] = static_cast<uint8_t>(i);
    pj[p] = static_cast<uint8_t>(p - base);
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* xs = xs_all + warp * rows * pitch;
  for (int b = blockIdx.x * warps_per_cta + warp; b < B; b += gridDim.x * warps_per_cta) {
    const float* xb = X + static_cast<int64_t>(b) * rows * D;
    for (int e = lane; e < rows * D; e += 32) xs[(e / D) * pitch + (e % D)] = xb[e];
    __syncwarp();
    __nv_bfloat16* ab = A + static_cast<int64_t>(b) * ld;
    for (int k = lane; k < D; k += 32) ab[k] = __float2bfloat16_rn(xs[k]);
    for (int p = lane; p < npairs; p += 32) {
      const float* xi = xs + pi[p] * pitch;
      const float* xj = xs + pj[p] * pitch;
      float acc = 0.f;
      for (int k = 0; k < D; ++k) acc = fmaf(xi[k], xj[k], acc);
      ab[D + p] = __float2bfloat16_rn(acc);
    }
    for (int k = D + npairs + lane; k < ld; k += 32) ab[k] = __float2bfloat16_rn(0.f);
    __syncwarp();
  }
}

void launch_interact(const float* X, int B, const int* dB, int T, int D, __nv_bfloat16* A_top,
                     int ld_top, cudaStream_t s) {
  if (B <= 0) return;
  const int npairs = T * (T + 1) / 2;
  const size_t per_warp = static_cast<size_t>(T + 1) * (D + 1) * sizeof(float);
  const size_t head = ((2 * npairs + 15) / 4 + 4) * sizeof(float);
  int wpc = static_cast<int>((44 * 1024 - head) / per_warp);
  if (wpc > 8) wpc = 8;
  if (wpc < 1) wpc = 1;
  const size_t smem = head + wpc * per_warp;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_interact, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
  int blocks = (B + wpc - 1) / wpc;
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_interact<<<blocks, 32 * wpc, smem, s>>>(X, B, dB, T, D, A_top, ld_top, wpc);
}

}  // namespace rec
