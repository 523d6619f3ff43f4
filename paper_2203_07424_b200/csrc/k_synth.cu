// k_synth.cu — synthetic parameters and batch inputs as Philox functions of counters
// (G2-G5).  Every value is bit-identical to oracle/gen.py.
#include "common.cuh"
#include "kernels.h"

namespace rec {

__device__ __forceinline__ float pow2f(int e) {  // exact 2^e for e in [-126, 127]
  return __int_as_float((127 + e) << 23);
}
__device__ __forceinline__ float i8(uint32_t w) {
  return static_cast<float>(static_cast<int>(static_cast<int8_t>(w & 0xFFu)));
}

// ------------------------------------------------------------------ tables (G4)
// Element (r, k) of table t is stored at base[r * stride + k] (base = start of row 0 of t).
__global__ void k_init_table(float* __restrict__ base, int64_t rows, int D, int64_t stride, int t,
                             uint32_t k0, uint32_t k1, int shift, int value_mode) {
  const int64_t n = rows * D;
  const uint32_t c2 = (static_cast<uint32_t>(t) << 8) | DOM_TABLE;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t r = static_cast<uint32_t>(e / D), k = static_cast<uint32_t>(e % D);
    const U4 w = philox(k, r, c2, 0u, k0, k1);
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
                       uint32_t k1, int shift, int value_mode, cudaStream_t s) {
  k_init_table<<<148 * 8, 256, 0, s>>>(base, rows, D, stride, t, k0, k1, shift, value_mode);
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

// ------------------------------------------------------------ batch rows (q, item)
__global__ void k_expand_rows(const int4* __restrict__ segs, int nseg, int B, int* __restrict__ rowq,
                              int* __restrict__ rowi) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  int lo = 0, hi = nseg - 1;  // last segment with first_row <= b
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(&segs[mid].w) <= b) lo = mid; else hi = mid - 1;
  }
  const int4 sg = segs[lo];
  rowq[b] = sg.x;
  rowi[b] = sg.y + (b - sg.w);
}

void launch_expand_rows(const int4* segs4, int nseg, int B, int* rowq, int* rowi, cudaStream_t s) {
  k_expand_rows<<<(B + 255) / 256, 256, 0, s>>>(segs4, nseg, B, rowq, rowi);
}

// ------------------------------------------------------------ lengths + offsets (G3)
// Fixed pooling: offsets[g] = g*L.  Variable: per-bag Philox lengths, then one-CTA
// exclusive scan (T*B <= a few 10^5, a handful of microseconds).
__global__ void k_offsets_fixed(int* __restrict__ off, int nbags, int L) {
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g <= nbags; g += gridDim.x * blockDim.x)
    off[g] = g * L;
}

__global__ void __launch_bounds__(1024) k_offsets_var(const int* __restrict__ rowq,
                                                      const int* __restrict__ rowi, int B, int T,
                                                      int lo, int hi, uint32_t k0, uint32_t k1,
                                                      int* __restrict__ off) {
  __shared__ int wsum[32];
  __shared__ int carry;
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
    // block inclusive scan
    int v = len;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += n;
    }
    if (lane == 31) wsum[wid] = v;
    __syncthreads();
    if (wid == 0) {
      int s = wsum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int n = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += n;
      }
      wsum[lane] = s;
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

void launch_gen_offsets(const int* rowq, const int* rowi, int B, int T, int lo, int hi, uint32_t k0,
                        uint32_t k1, int* offsets, cudaStream_t s) {
  if (lo == hi) {
    const int nb = T * B;
    k_offsets_fixed<<<(nb + 1 + 255) / 256, 256, 0, s>>>(offsets, nb, lo);
  } else {
    k_offsets_var<<<1, 1024, 0, s>>>(rowq, rowi, B, T, lo, hi, k0, k1, offsets);
  }
}

// ---------------------------------------------------------------------- indices (G2)
// One warp per bag, lanes over slots.
__global__ void k_gen_indices(const int* __restrict__ rowq, const int* __restrict__ rowi,
                              const int* __restrict__ off, int B, int T,
                              const int64_t* __restrict__ rows, int index_dist, uint32_t k0,
                              uint32_t k1, int* __restrict__ indices) {
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; g < T * B; g += warps) {
    const int t = g / B, b = g % B;
    const uint32_t q = static_cast<uint32_t>(rowq[b]), it = static_cast<uint32_t>(rowi[b]);
    const uint64_t R = static_cast<uint64_t>(rows[t]);
    const uint32_t c2 = (static_cast<uint32_t>(t) << 8) | DOM_INDEX;
    const int s = off[g], e = off[g + 1];
    for (int j = lane; j < e - s; j += 32) {
      const U4 w = philox(static_cast<uint32_t>(j), it, c2, q, k0, k1);
      uint64_t r = (static_cast<uint64_t>(w.y) << 32) | w.x;
      if (index_dist == 2) r = __umul64hi(r, (static_cast<uint64_t>(w.w) << 32) | w.z);
      indices[s + j] = static_cast<int>(__umul64hi(r, R));
    }
  }
}

void launch_gen_indices(const int* rowq, const int* rowi, const int* offsets, int B, int T,
                        const int64_t* rows, int index_dist, uint32_t k0, uint32_t k1, int* indices,
                        cudaStream_t s) {
  const int bags = T * B;
  int blocks = (bags + 7) / 8;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_gen_indices<<<blocks, 256, 0, s>>>(rowq, rowi, offsets, B, T, rows, index_dist, k0, k1, indices);
}

// ------------------------------------------------------------------------ dense (G4)
__global__ void k_gen_dense(const int* __restrict__ rowq, const int* __restrict__ rowi, int B, int F,
                            int Fpad, uint32_t k0, uint32_t k1, __nv_bfloat16* __restrict__ dbf,
                            float* __restrict__ df) {
  const int64_t n = (int64_t)B * Fpad;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int b = static_cast<int>(x / Fpad), f = static_cast<int>(x % Fpad);
    float v = 0.f;
    if (f < F) {
      const U4 w = philox(static_cast<uint32_t>(f), static_cast<uint32_t>(rowi[b]), DOM_DENSE,
                          static_cast<uint32_t>(rowq[b]), k0, k1);
      v = i8(w.x) * pow2f(-7);
      if (df) df[(int64_t)b * F + f] = v;
    }
    if (dbf) dbf[x] = __float2bfloat16_rn(v);
  }
}

void launch_gen_dense(const int* rowq, const int* rowi, int B, int F, int Fpad, uint32_t k0,
                      uint32_t k1, __nv_bfloat16* dense_bf, float* dense_f32, cudaStream_t s) {
  const int64_t n = (int64_t)B * Fpad;
  int blocks = static_cast<int>((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_gen_dense<<<blocks, 256, 0, s>>>(rowq, rowi, B, F, Fpad, k0, k1, dense_bf, dense_f32);
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
  int blocks = static_cast<int>((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_dense_to_bf16<<<blocks, 256, 0, s>>>(dense, B, F, Fpad, out);
}

// ------------------------------------------------------- caller offsets validation
__global__ void k_check_offsets(const int* __restrict__ off, int nbags, int* __restrict__ flag) {
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < nbags; g += gridDim.x * blockDim.x) {
    if (off[g + 1] < off[g] || (g == 0 && off[0] != 0)) atomicOr(flag, 2);
  }
}

void launch_check_offsets(const int* offsets, int nbags, int* flag, cudaStream_t s) {
  int blocks = (nbags + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  k_check_offsets<<<blocks, 256, 0, s>>>(offsets, nbags, flag);
}

}  // namespace rec
