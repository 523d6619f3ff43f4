#include <algorithm>
// k_synth.cu — synthetic parameters and batch inputs as Philox functions of counters
// (G2-G5).  Every value is bit-identical to oracle/gen.py.
#include "common.cuh"
#include "kernels.h"
#include "synth.cuh"

namespace rec {

// ------------------------------------------------------------------ tables (G4)
// Element (r, k) of table t is stored at base[r * stride + k] (base = start of row 0 of t).
__global__ void k_init_table(float* __restrict__ base, int64_t rows, int D, int64_t stride, int t,
                             uint32_t k0, uint32_t k1, int shift, int value_mode, int64_t r0) {
  const int64_t n = rows * D;
  const uint32_t c2 = (static_cast<uint32_t>(t) << 8) | DOM_TABLE;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t r = static_cast<uint32_t>(e / D), k = static_cast<uint32_t>(e % D);
    const U4 w = philox(k, static_cast<uint32_t>(r0 + r), c2, 0u, k0, k1);
    float v;
    if (value_mode == 0) {
      v = i8(w.x) * pow2f(-(7 + shift));
    } else {
      v = static_cast<float>(static_cast<int>(w.x >> 8) - (1 << 23)) * pow2f(-(23 + shift));
    }
    base[static_cast<int64_t>(r) * stride + k] = v;
  }
}

void launch_init_table(float* base, int64_t rows, int D, int64_t stride, int t, uint32_t k0,
                       uint32_t k1, int shift, int value_mode, cudaStream_t s, int64_t r0) {
  k_init_table<<<148 * 8, 256, 0, s>>>(base, rows, D, stride, t, k0, k1, shift, value_mode, r0);
}

// ------------------------------------------------------------------ weights (G5)
__global__ void k_init_layer(__nv_bfloat16* __restrict__ W, float* __restrict__ bias, int N, int K,
                             int Kpad, int layer, int e, uint32_t k0, uint32_t k1) {
  const int64_t n = (int64_t)N * Kpad;
  const uint32_t cw = (static_cast<uint32_t>(layer) << 8) | DOM_W;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int o = static_cast<int>(x / Kpad), i = static_cast<int>(x % Kpad);
    float v = 0.f;
    if (i < K) v = i8(philox(i, o, cw, 0u, k0, k1).x) * pow2f(e);
    W[x] = __float2bfloat16_rn(v);
  }
  const uint32_t cb = (static_cast<uint32_t>(layer) << 8) | DOM_B;
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < N; o += gridDim.x * blockDim.x)
    bias[o] = i8(philox(o, 0u, cb, 0u, k0, k1).x) * pow2f(e);
}

void launch_init_layer(__nv_bfloat16* W, float* bias, int N, int K, int Kpad, int layer, int e,
                       uint32_t k0, uint32_t k1, cudaStream_t s) {
  k_init_layer<<<256, 256, 0, s>>>(W, bias, N, K, Kpad, layer, e, k0, k1);
}

__global__ void k_init_final(float* __restrict__ w, float* __restrict__ b, int K, int layer, int e,
                             uint32_t k0, uint32_t k1) {
  const uint32_t cw = (static_cast<uint32_t>(layer) << 8) | DOM_W;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < K; i += gridDim.x * blockDim.x)
    w[i] = i8(philox(i, 0u, cw, 0u, k0, k1).x) * pow2f(e);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const uint32_t cb = (static_cast<uint32_t>(layer) << 8) | DOM_B;
    b[0] = i8(philox(0u, 0u, cb, 0u, k0, k1).x) * pow2f(e);
  }
}

void launch_init_final(float* w, float* b, int K, int layer, int e, uint32_t k0, uint32_t k1,
                       cudaStream_t s) {
  k_init_final<<<4, 256, 0, s>>>(w, b, K, layer, e, k0, k1);
}

// ------------------------------------------------ fused inputs, fixed pooling (a2)
// Blocks [0, nbag_blocks): one warp per bag g = t*B + b (offsets[g] = g*L, L indices);
// blocks beyond: one warp per batch row (dense features).  One launch for all of a2.
constexpr int kGenWPB = 8;

__global__ void __launch_bounds__(32 * kGenWPB) k_gen_fused(const __grid_constant__ SegBatch sb,
                                                            const GenArgs ga) {
  const int B = sb.B;
  const int lane = threadIdx.x & 31;
  if (blockIdx.x == 0 && threadIdx.x == 0) *ga.dB = B;
  const int L = ga.lo;
  if (static_cast<int>(blockIdx.x) < ga.nbag_blocks) {
    const int g = blockIdx.x * kGenWPB + (threadIdx.x >> 5);
    const int nb = ga.T * B;
    if (g == 0 && lane == 0) ga.offsets[nb] = nb * L;
    if (g >= nb) return;
    const int t = g / B, b = g - t * B;
    const int2 qi = row_item(sb, b);
    if (lane == 0) ga.offsets[g] = g * L;
    const uint64_t R = static_cast<uint64_t>(__ldg(&ga.rows[t]));
    const uint32_t c2 = (static_cast<uint32_t>(t) << 8) | DOM_INDEX;
    const double zc = ga.index_dist == 3 ? zipf_c(R) : 0.0;
    int* dst = ga.indices + static_cast<int64_t>(g) * L;
    for (int j = lane; j < L; j += 32)
      dst[j] = gen_index(j, qi.y, c2, qi.x, ga.k0, ga.k1, R, ga.index_dist, zc);
  } else {
    const int b = (blockIdx.x - ga.nbag_blocks) * kGenWPB + (threadIdx.x >> 5);
    if (b >= B) return;
    const int2 qi = row_item(sb, b);
    gen_dense_row(qi.y, qi.x, ga.k0, ga.k1, ga.F, ga.Fpad, ga.dense_bf + static_cast<int64_t>(b) * ga.Fpad,
                  ga.dense_f32 ? ga.dense_f32 + static_cast<int64_t>(b) * ga.F : nullptr, lane, 32);
  }
}

// Dense features only (fixed-pooling synthetic path, where the SLS kernel generates its own
// indices): one warp per batch row, bf16 padded row for the bottom MLP.
__global__ void __launch_bounds__(32 * kGenWPB) k_gen_dense_seg(const __grid_constant__ SegBatch sb,
                                                                const GenArgs ga) {
  if (blockIdx.x == 0 && threadIdx.x == 0) *ga.dB = sb.B;
  const int b = blockIdx.x * kGenWPB + (threadIdx.x >> 5);
  if (b >= sb.B) return;
  const int lane = threadIdx.x & 31;
  const int2 qi = row_item(sb, b);
  gen_dense_row(qi.y, qi.x, ga.k0, ga.k1, ga.F, ga.Fpad, ga.dense_bf + static_cast<int64_t>(b) * ga.Fpad,
                nullptr, lane, 32);
}

void* gen_dense_seg_kernel(const GenArgs& ga, dim3* grid, dim3* block) {
  *grid = dim3((ga.cap + kGenWPB - 1) / kGenWPB);
  *block = dim3(32 * kGenWPB);
  return reinterpret_cast<void*>(k_gen_dense_seg);
}

void launch_gen_dense_seg(const SegBatch& sb, const GenArgs& ga, cudaStream_t s) {
  dim3 grid, block;
  void* fn = gen_dense_seg_kernel(ga, &grid, &block);
  void* args[2] = {const_cast<SegBatch*>(&sb), const_cast<GenArgs*>(&ga)};
  cudaLaunchKernel(fn, grid, block, args, 0, s);
}

// Variable pooling, step 1: rows (q, item) of the batch + the device batch size.
__global__ void k_expand_rows(const __grid_constant__ SegBatch sb, const GenArgs ga) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b == 0) *ga.dB = sb.B;
  if (b >= sb.B) return;
  const int2 qi = row_item(sb, b);
  ga.rowq[b] = qi.x;
  ga.rowi[b] = qi.y;
}

void* gen_first_kernel(const GenArgs& ga, dim3* grid, dim3* block) {
  if (ga.lo == ga.hi) {
    const int nrow_blocks = (ga.cap + kGenWPB - 1) / kGenWPB;
    *grid = dim3(ga.nbag_blocks + nrow_blocks);
    *block = dim3(32 * kGenWPB);
    return reinterpret_cast<void*>(k_gen_fused);
  }
  *grid = dim3((ga.cap + 255) / 256);
  *block = dim3(256);
  return reinterpret_cast<void*>(k_expand_rows);
}

void launch_gen_first(const SegBatch& sb, const GenArgs& ga, cudaStream_t s) {
  dim3 grid, block;
  void* fn = gen_first_kernel(ga, &grid, &block);
  void* args[2] = {const_cast<SegBatch*>(&sb), const_cast<GenArgs*>(&ga)};
  cudaLaunchKernel(fn, grid, block, args, 0, s);
}

// ------------------------------------------------------------ lengths + offsets (G3)
// Variable pooling: per-bag Philox lengths, then a one-CTA exclusive scan (T*B is a few
// 10^4-10^5: a handful of microseconds).
__global__ void __launch_bounds__(1024) k_offsets_var(const int* __restrict__ rowq,
                                                      const int* __restrict__ rowi,
                                                      const int* __restrict__ dB, int T,
                                                      int lo, int hi, uint32_t k0, uint32_t k1,
                                                      int* __restrict__ off) {
  __shared__ int wsum[32];
  __shared__ int carry;
  const int B = *dB;
  const int nb = T * B;
  const uint64_t span = static_cast<uint64_t>(hi - lo + 1);
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nb; base += 1024) {
    const int g = base + threadIdx.x;
    int len = 0;
    if (g < nb) {
      const int t = g / B, b = g % B;
      const U4 w = philox(0u, static_cast<uint32_t>(rowi[b]), (static_cast<uint32_t>(t) << 8) | DOM_LEN,
                          static_cast<uint32_t>(rowq[b]), k0, k1);
      const uint64_t r = (static_cast<uint64_t>(w.y) << 32) | w.x;
      len = lo + static_cast<int>(__umul64hi(r, span));
    }
    int v = len;  // block inclusive scan
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += n;
    }
    if (lane == 31) wsum[wid] = v;
    __syncthreads();
    if (wid == 0) {
      int s2 = wsum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int n = __shfl_up_sync(0xffffffffu, s2, o);
        if (lane >= o) s2 += n;
      }
      wsum[lane] = s2;
    }
    __syncthreads();
    const int incl = v + (wid ? wsum[wid - 1] : 0) + carry;
    if (g < nb) off[g + 1] = incl;
    __syncthreads();
    if (threadIdx.x == 1023) carry = incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) off[0] = 0;
}

// One warp per bag, lanes over slots (variable pooling path).
__global__ void k_gen_indices(const int* __restrict__ rowq, const int* __restrict__ rowi,
                              const int* __restrict__ off, const int* __restrict__ dB, int T,
                              const int64_t* __restrict__ rows, int index_dist, uint32_t k0,
                              uint32_t k1, int* __restrict__ indices) {
  const int B = *dB;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; g < T * B; g += warps) {
    const int t = g / B, b = g % B;
    const uint32_t q = static_cast<uint32_t>(rowq[b]), it = static_cast<uint32_t>(rowi[b]);
    const uint64_t R = static_cast<uint64_t>(rows[t]);
    const uint32_t c2 = (static_cast<uint32_t>(t) << 8) | DOM_INDEX;
    const int s0 = off[g], e = off[g + 1];
    const double zc = index_dist == 3 ? zipf_c(R) : 0.0;
    for (int j = lane; j < e - s0; j += 32)
      indices[s0 + j] = gen_index(j, it, c2, q, k0, k1, R, index_dist, zc);
  }
}

__global__ void k_gen_dense(const int* __restrict__ rowq, const int* __restrict__ rowi,
                            const int* __restrict__ dB, int F, int Fpad, uint32_t k0, uint32_t k1,
                            __nv_bfloat16* __restrict__ dbf, float* __restrict__ df) {
  const int B = *dB;
  const int nblk = (Fpad + 15) / 16;
  const int64_t n = (int64_t)B * nblk;  // one thread per (row, 16-feature block)
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int b = static_cast<int>(x / nblk), blk = static_cast<int>(x % nblk);
    if (dbf) {
      gen_dense_row(static_cast<uint32_t>(rowi[b]), static_cast<uint32_t>(rowq[b]), k0, k1, F, Fpad,
                    dbf + (int64_t)b * Fpad, df ? df + (int64_t)b * F : nullptr, blk, nblk);  // this block only
    } else {
      float v[16];
      gen_dense16(static_cast<uint32_t>(blk), rowi[b], rowq[b], k0, k1, v);
      for (int j = 0; j < 16 && blk * 16 + j < F; ++j) df[(int64_t)b * F + blk * 16 + j] = v[j];
    }
  }
}

void launch_gen_variable_rest(const GenArgs& ga, cudaStream_t s) {
  k_offsets_var<<<1, 1024, 0, s>>>(ga.rowq, ga.rowi, ga.dB, ga.T, ga.lo, ga.hi, ga.k0, ga.k1,
                                   ga.offsets);
  int blocks = (ga.T * ga.cap + 7) / 8;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  k_gen_indices<<<blocks, 256, 0, s>>>(ga.rowq, ga.rowi, ga.offsets, ga.dB, ga.T, ga.rows,
                                       ga.index_dist, ga.k0, ga.k1, ga.indices);
  const int64_t n = (int64_t)ga.cap * ga.Fpad;
  int dblocks = static_cast<int>((n + 255) / 256);
  if (dblocks > 148 * 16) dblocks = 148 * 16;
  if (dblocks < 1) dblocks = 1;
  k_gen_dense<<<dblocks, 256, 0, s>>>(ga.rowq, ga.rowi, ga.dB, ga.F, ga.Fpad, ga.k0, ga.k1,
                                      ga.dense_bf, ga.dense_f32);
}

__global__ void k_dense_to_bf16(const float* __restrict__ d, int B, int F, int Fpad,
                                __nv_bfloat16* __restrict__ out) {
  const int64_t n = (int64_t)B * Fpad;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int b = static_cast<int>(x / Fpad), f = static_cast<int>(x % Fpad);
    out[x] = __float2bfloat16_rn(f < F ? d[(int64_t)b * F + f] : 0.f);
  }
}

void launch_dense_to_bf16(const float* dense, int B, int F, int Fpad, __nv_bfloat16* out,
                          cudaStream_t s) {
  const int64_t n = (int64_t)B * Fpad;
  if (n == 0) return;  // no dense input (MT-WnD)
  int blocks = static_cast<int>((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_dense_to_bf16<<<blocks, 256, 0, s>>>(dense, B, F, Fpad, out);
}

// ------------------------------------------------------- hot-row partition (rec_hot_remap)
__global__ void k_remap(const int* __restrict__ in, const int* __restrict__ off, int B,
                        const int* __restrict__ dB, const int64_t* __restrict__ rows,
                        const int* __restrict__ remap, const int64_t* __restrict__ remap_off,
                        int* __restrict__ out, int64_t cap, int* __restrict__ flag) {
  if (dB) B = *dB;
  const int t = blockIdx.y;
  const int lo = off[t * B], hi = off[(t + 1) * B];
  const int64_t R = rows[t];
  const int* map = remap + remap_off[t];
  bool oob = false, over = false;
  for (int i = lo + blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += gridDim.x * blockDim.x) {
    const int r = in[i];
    const bool ok = r >= 0 && r < R;
    oob |= !ok;
    if (i < cap) out[i] = ok ? __ldg(map + r) : 0;
    else over = true;
  }
  if (oob) atomicOr(flag, 1);
  if (over) atomicOr(flag, 2);
}

void launch_remap(const int* in, const int* offsets, int B, const int* dB, int T, const int64_t* rows,
                  const int* remap, const int64_t* remap_off, int* out, int64_t cap, int* flag,
                  cudaStream_t s) {
  if (T <= 0 || B <= 0) return;
  k_remap<<<dim3(32, T), 256, 0, s>>>(in, offsets, B, dB, rows, remap, remap_off, out, cap, flag);
}

__global__ void k_permute_rows(const float4* __restrict__ src, float4* __restrict__ dst,
                               const int64_t* __restrict__ tab_off, int64_t row_stride,
                               const int64_t* __restrict__ rows, int D, const int* __restrict__ inv,
                               const int64_t* __restrict__ remap_off) {
  const int t = blockIdx.y;
  const int64_t R = rows[t];
  const int d4 = D / 4;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < R * d4;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t p = e / d4;
    const int c = static_cast<int>(e - p * d4);
    const int64_t o = inv[remap_off[t] + p];
    dst[(tab_off[t] + p * row_stride) / 4 + c] = src[(tab_off[t] + o * row_stride) / 4 + c];
  }
}

void launch_permute_rows(const float* src, float* dst, const int64_t* tab_off, int64_t row_stride,
                         const int64_t* rows, int T, int D, const int* inv, const int64_t* remap_off,
                         int64_t max_rows, cudaStream_t s) {
  const int64_t n = max_rows * (D / 4);
  const int bx = static_cast<int>(std::min<int64_t>((n + 255) / 256, 4096));
  k_permute_rows<<<dim3(bx, T), 256, 0, s>>>(reinterpret_cast<const float4*>(src), reinterpret_cast<float4*>(dst),
                                             tab_off, row_stride, rows, D, inv, remap_off);
}

// ------------------------------------------------------- caller offsets validation
__global__ void k_check_offsets(const int* __restrict__ off, int nbags, int64_t nnz,
                                int* __restrict__ flag) {
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < nbags; g += gridDim.x * blockDim.x) {
    if (off[g + 1] < off[g] || (g == 0 && off[0] != 0)) atomicOr(flag, 2);
  }
  if (nnz >= 0 && blockIdx.x == 0 && threadIdx.x == 0 && static_cast<int64_t>(off[nbags]) != nnz)
    atomicOr(flag, 2);
}

void launch_check_offsets(const int* offsets, int nbags, int* flag, cudaStream_t s, int64_t nnz) {
  int blocks = (nbags + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  k_check_offsets<<<blocks, 256, 0, s>>>(offsets, nbags, nnz, flag);
}

}  // namespace rec
