// k_interact.cu — pairwise dot-product feature interaction.
//
// Paper: the SparseNet / DenseNet join is shown only in Fig. rec_char(a) and by
// citing DLRM; reading R1 takes DLRM's dot interaction without self pairs:
//   X_b = [x_b; p_b,0; ...; p_b,T-1]  ((T+1) x D, fp32),  Z = X_b X_b^T,
//   A_top[b] = bf16([x_b, Z(1,0), Z(2,0), Z(2,1), ..., Z(T,T-1), 0-pad])
// which is the A operand (K-major bf16 row) of the first top-MLP GEMM.
//
// One warp per item (see k_interact below).  (T+1)^2/2 * D FMAs per item is < 1 % of the
// item's SLS time; the kernel is latency bound, so loads and stores are vectorised.
#include "common.cuh"
#include "kernels.h"

namespace rec {

int g_interact_wpc = 8;  // warps (items) per CTA, REC_INTERACT_WPC
// rows of X_b (T + 1) from which the interaction uses 4 x 4 register blocks (REC_INTERACT_BLOCKED
// sets it; 0 = never)
int kBlockedRows = 24;
int g_interact_pf = 0;   // few-CTA prefetching interaction (REC_INTERACT_PF=1; measured slightly slower)

// Pair p of the strict lower triangle in row-major order: (i, j), 1 <= i <= T, 0 <= j < i,
// p = i(i-1)/2 + j.
__device__ __forceinline__ int2 pair_of(int p) {
  int i = static_cast<int>((1.0f + sqrtf(1.0f + 8.0f * static_cast<float>(p))) * 0.5f);
  while (i * (i - 1) / 2 > p) --i;
  while ((i + 1) * i / 2 <= p) ++i;
  return make_int2(i, p - i * (i - 1) / 2);
}

// One warp per item.  X_b arrives as 16-B vector loads issued back to back (one L2 round
// trip), rows land in shared memory with a D+4 pitch (float4-aligned, rows 4 banks apart);
// each lane forms whole pairs as sequential fp32 FMA chains over k; the bf16 output row is
// staged in shared memory and written with 16-B vector stores (ld is a multiple of 8).
__global__ void k_interact(const float* __restrict__ X, int B, const int* __restrict__ dB, int T,
                           int D, __nv_bfloat16* __restrict__ A, int ld, int warps_per_cta,
                           int blocked_rows) {
  extern __shared__ float4 sm4[];
  // the top MLP kernel that follows may be scheduled now: it sets up (barriers, TMEM, bias)
  // and waits for this grid before reading A (programmatic dependent launch)
  cudaTriggerProgrammaticLaunchCompletion();
  if (dB) B = *dB;
  if (static_cast<int>(blockIdx.x) * warps_per_cta >= B) return;
  const int rows = T + 1, pitch = D + 4, npairs = T * (T + 1) / 2, d4 = D / 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int per_warp_f = rows * pitch + ld / 2;  // floats: X rows + bf16 output row
  float* xs = reinterpret_cast<float*>(sm4) + warp * per_warp_f;
  __nv_bfloat16* outs = reinterpret_cast<__nv_bfloat16*>(xs + rows * pitch);
  const int nvec = rows * d4;
  for (int b = blockIdx.x * warps_per_cta + warp; b < B; b += gridDim.x * warps_per_cta) {
    const float4* xb = reinterpret_cast<const float4*>(X + static_cast<int64_t>(b) * rows * D);
#pragma unroll 4
    for (int e = lane; e < nvec; e += 32) {
      const float4 v = __ldg(xb + e);
      const int r = e / d4, c = e - r * d4;
      *reinterpret_cast<float4*>(xs + r * pitch + 4 * c) = v;
    }
    __syncwarp();
    for (int k = lane; k < D; k += 32) outs[k] = __float2bfloat16_rn(xs[k]);
    if (rows >= blocked_rows) {
      // many tables (RMC2: 41 rows, 820 pairs): each lane owns 4 x 4 blocks of the lower
      // triangle, so one pair of 4-row float4 loads feeds 64 FMAs instead of 4 (the per-pair
      // loop is shared-memory bound there).  Every Z(i, j) is still one fp32 FMA chain over
      // k = 0..D-1 in the same order, so the bits equal the per-pair loop's.
      const int nrb = (rows + 3) / 4, nblk = nrb * (nrb + 1) / 2;
      const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int q = lane; q < nblk; q += 32) {
        int I = static_cast<int>((sqrtf(8.f * static_cast<float>(q) + 1.f) - 1.f) * 0.5f);
        while (I * (I + 1) / 2 > q) --I;
        while ((I + 1) * (I + 2) / 2 <= q) ++I;
        const int J = q - I * (I + 1) / 2;
        float acc[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[u][v] = 0.f;
        for (int k = 0; k < d4; ++k) {
          float4 a[4], c[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int ri = 4 * I + u, rj = 4 * J + u;
            a[u] = ri < rows ? reinterpret_cast<const float4*>(xs + ri * pitch)[k] : z4;
            c[u] = rj < rows ? reinterpret_cast<const float4*>(xs + rj * pitch)[k] : z4;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              float t = acc[u][v];
              t = fmaf(a[u].x, c[v].x, t);
              t = fmaf(a[u].y, c[v].y, t);
              t = fmaf(a[u].z, c[v].z, t);
              t = fmaf(a[u].w, c[v].w, t);
              acc[u][v] = t;
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const int i = 4 * I + u, j = 4 * J + v;
            if (i < rows && j < i) outs[D + i * (i - 1) / 2 + j] = __float2bfloat16_rn(acc[u][v]);
          }
      }
    } else {
      for (int p = lane; p < npairs; p += 32) {
        const int2 ij = pair_of(p);
        const float4* xi = reinterpret_cast<const float4*>(xs + ij.x * pitch);
        const float4* xj = reinterpret_cast<const float4*>(xs + ij.y * pitch);
        float acc = 0.f;
        for (int k = 0; k < d4; ++k) {
          const float4 a = xi[k], c = xj[k];
          acc = fmaf(a.x, c.x, acc);
          acc = fmaf(a.y, c.y, acc);
          acc = fmaf(a.z, c.z, acc);
          acc = fmaf(a.w, c.w, acc);
        }
        outs[D + p] = __float2bfloat16_rn(acc);
      }
    }
    for (int k = D + npairs + lane; k < ld; k += 32) outs[k] = __float2bfloat16_rn(0.f);
    __syncwarp();
    int4* ab = reinterpret_cast<int4*>(A + static_cast<int64_t>(b) * ld);
    const int4* os = reinterpret_cast<const int4*>(outs);
    for (int v = lane; v < ld / 8; v += 32) ab[v] = os[v];
    __syncwarp();
  }
}

// Same computation, few CTAs: each warp walks ~kItemsPerWarp items and prefetches the next
// item's X rows into registers while it computes the current one, so the kernel holds ~8x
// fewer CTA-microseconds of SM residency (what co-running SLS CTAs pay for)
// at about the same duration.  PF = float4 per lane per item ((T+1)*D/4 <= 32*PF).
constexpr int kItemsPerWarp = 4;
template <int PF>
__global__ void k_interact_pf(const float* __restrict__ X, int B, const int* __restrict__ dB, int T,
                              int D, __nv_bfloat16* __restrict__ A, int ld, int warps_per_cta, int blocked_rows) {
  extern __shared__ float4 sm4[];
  if (dB) B = *dB;
  const int rows = T + 1, pitch = D + 4, npairs = T * (T + 1) / 2, d4 = D / 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int per_warp_f = rows * pitch + ld / 2;
  float* xs = reinterpret_cast<float*>(sm4) + warp * per_warp_f;
  __nv_bfloat16* outs = reinterpret_cast<__nv_bfloat16*>(xs + rows * pitch);
  const int nvec = rows * d4;
  const int stride = gridDim.x * warps_per_cta;
  int b = blockIdx.x * warps_per_cta + warp;
  float4 pf[PF];
  if (b < B) {
    const float4* xb = reinterpret_cast<const float4*>(X + static_cast<int64_t>(b) * rows * D);
#pragma unroll
    for (int q = 0; q < PF; ++q) {
      const int e = lane + 32 * q;
      if (e < nvec) pf[q] = __ldg(xb + e);
    }
  }
  for (; b < B; b += stride) {
#pragma unroll
    for (int q = 0; q < PF; ++q) {  // prefetched rows of item b -> shared memory
      const int e = lane + 32 * q;
      if (e < nvec) {
        const int r = e / d4, c = e - r * d4;
        *reinterpret_cast<float4*>(xs + r * pitch + 4 * c) = pf[q];
      }
    }
    const int bn = b + stride;
    if (bn < B) {  // next item's rows in flight during this item's math
      const float4* xb = reinterpret_cast<const float4*>(X + static_cast<int64_t>(bn) * rows * D);
#pragma unroll
      for (int q = 0; q < PF; ++q) {
        const int e = lane + 32 * q;
        if (e < nvec) pf[q] = __ldg(xb + e);
      }
    }
    __syncwarp();
    for (int k = lane; k < D; k += 32) outs[k] = __float2bfloat16_rn(xs[k]);
    if (rows >= blocked_rows) {
      // many tables (RMC2: 41 rows, 820 pairs): each lane owns 4 x 4 blocks of the lower
      // triangle, so one pair of 4-row float4 loads feeds 64 FMAs instead of 4 (the per-pair
      // loop is shared-memory bound there).  Every Z(i, j) is still one fp32 FMA chain over
      // k = 0..D-1 in the same order, so the bits equal the per-pair loop's.
      const int nrb = (rows + 3) / 4, nblk = nrb * (nrb + 1) / 2;
      const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int q = lane; q < nblk; q += 32) {
        int I = static_cast<int>((sqrtf(8.f * static_cast<float>(q) + 1.f) - 1.f) * 0.5f);
        while (I * (I + 1) / 2 > q) --I;
        while ((I + 1) * (I + 2) / 2 <= q) ++I;
        const int J = q - I * (I + 1) / 2;
        float acc[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[u][v] = 0.f;
        for (int k = 0; k < d4; ++k) {
          float4 a[4], c[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int ri = 4 * I + u, rj = 4 * J + u;
            a[u] = ri < rows ? reinterpret_cast<const float4*>(xs + ri * pitch)[k] : z4;
            c[u] = rj < rows ? reinterpret_cast<const float4*>(xs + rj * pitch)[k] : z4;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              float t = acc[u][v];
              t = fmaf(a[u].x, c[v].x, t);
              t = fmaf(a[u].y, c[v].y, t);
              t = fmaf(a[u].z, c[v].z, t);
              t = fmaf(a[u].w, c[v].w, t);
              acc[u][v] = t;
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const int i = 4 * I + u, j = 4 * J + v;
            if (i < rows && j < i) outs[D + i * (i - 1) / 2 + j] = __float2bfloat16_rn(acc[u][v]);
          }
      }
    } else {
      for (int p = lane; p < npairs; p += 32) {
        const int2 ij = pair_of(p);
        const float4* xi = reinterpret_cast<const float4*>(xs + ij.x * pitch);
        const float4* xj = reinterpret_cast<const float4*>(xs + ij.y * pitch);
        float acc = 0.f;
        for (int k = 0; k < d4; ++k) {
          const float4 a = xi[k], c = xj[k];
          acc = fmaf(a.x, c.x, acc);
          acc = fmaf(a.y, c.y, acc);
          acc = fmaf(a.z, c.z, acc);
          acc = fmaf(a.w, c.w, acc);
        }
        outs[D + p] = __float2bfloat16_rn(acc);
      }
    }
    for (int k = D + npairs + lane; k < ld; k += 32) outs[k] = __float2bfloat16_rn(0.f);
    __syncwarp();
    int4* ab = reinterpret_cast<int4*>(A + static_cast<int64_t>(b) * ld);
    const int4* os = reinterpret_cast<const int4*>(outs);
    for (int v = lane; v < ld / 8; v += 32) ab[v] = os[v];
    __syncwarp();
  }
}

void launch_interact(const float* X, int B, const int* dB, int T, int D, __nv_bfloat16* A_top,
                     int ld_top, cudaStream_t s) {
  if (B > 0 && g_interact_pf && (T + 1) * (D / 4) <= 32 * 4) {
    const size_t per_warp = (static_cast<size_t>(T + 1) * (D + 4) + ld_top / 2) * sizeof(float);
    const int wpc = 8;
    int blocks = (B + wpc * kItemsPerWarp - 1) / (wpc * kItemsPerWarp);
    if (blocks > 148) blocks = 148;
    const size_t smem = wpc * per_warp;
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(k_interact_pf<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem));
    k_interact_pf<4><<<blocks, 32 * wpc, smem, s>>>(X, B, dB, T, D, A_top, ld_top, wpc, kBlockedRows);
    return;
  }
  if (B <= 0) return;
  const size_t per_warp = (static_cast<size_t>(T + 1) * (D + 4) + ld_top / 2) * sizeof(float);
  int wpc = static_cast<int>((96 * 1024) / per_warp);
  if (wpc > g_interact_wpc) wpc = g_interact_wpc;
  if (wpc < 1) wpc = 1;
  const size_t smem = wpc * per_warp;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_interact, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
  int blocks = (B + wpc - 1) / wpc;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (g_dense_prio == 0) {
    k_interact<<<blocks, 32 * wpc, smem, s>>>(X, B, dB, T, D, A_top, ld_top, wpc, kBlockedRows);
    return;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(32 * wpc);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributePriority;
  at[0].val.priority = g_dense_prio;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_interact, X, B, dB, T, D, A_top, ld_top, wpc, kBlockedRows);
}

// MT-WnD join (R26, R28): one warp per item; the concatenated pooled vectors become the bf16
// A row of the first tower layer, and each task's wide term is an fp32 dot product whose
// lane-strided partial sums meet in a fixed xor-shuffle tree (deterministic; with int8 x 2^e
// tables and weights every product and partial sum is exact, so the order is immaterial).
__global__ void k_concat(const float* __restrict__ X, int B, const int* __restrict__ dB, int T, int D,
                         __nv_bfloat16* __restrict__ A, int ld, const float* __restrict__ v,
                         int n_tasks, float* __restrict__ wide) {
  if (dB) B = *dB;
  const int warps = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  const int K = T * D;
  for (int b = blockIdx.x * warps + (threadIdx.x >> 5); b < B; b += gridDim.x * warps) {
    const float* u = X + static_cast<int64_t>(b) * (T + 1) * D + D;  // slots 1..T
    __nv_bfloat16* a = A + static_cast<int64_t>(b) * ld;
    float part[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) part[k] = 0.f;
    for (int c = lane; c < ld; c += 32) {
      const float x = c < K ? u[c] : 0.f;
      a[c] = __float2bfloat16_rn(x);
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (k < n_tasks && c < K) part[k] = fmaf(x, __ldg(&v[static_cast<int64_t>(k) * K + c]), part[k]);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (k >= n_tasks) break;
      float p = part[k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
      if (lane == 0) wide[static_cast<int64_t>(b) * n_tasks + k] = p;
    }
  }
}

void launch_concat(const float* X, int B, const int* dB, int T, int D, __nv_bfloat16* A_top, int ld,
                   const float* v, int n_tasks, float* wide, cudaStream_t s) {
  if (B <= 0) return;
  int blocks = (B + 7) / 8;
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_concat<<<blocks, 256, 0, s>>>(X, B, dB, T, D, A_top, ld, v, n_tasks, wide);
}

}  // namespace rec
