// k_sls.cu — SparseLengthsSum embedding-bag gather + sum-pool.
//
// out[b][1+t][:] = sum_{j = offsets[g]}^{offsets[g+1]-1} E_t[indices[j]][:],  g = t*B + b
// (PAPER.md:140 SparseNet "memory-intensive sparse operations on embeddings", P:151 pooling,
// P:933 "Gather-Reduce").  fp32 accumulate in index order (bit-comparable with the oracle's
// fp32-sequential mode).
//
// B200 mapping: a group of LANES = D/4 lanes owns one bag; each lane owns 4
// consecutive floats, so one table row (128 B at D = 32) is one fully coalesced 128-bit
// request per group.  Bag offsets of the CTA are staged in shared memory.  The group reads
// the bag's indices LANES at a time (one per lane), broadcasts them with shuffles, and keeps
// LANES independent 128-bit row loads in flight per lane (ld.global.nc.L1::no_allocate —
// rows are streamed, never reused from L1) before accumulating them in order.
#include "common.cuh"
#include "kernels.h"

namespace rec {

__device__ __forceinline__ float4 ldg_stream(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

// U = 128-bit row loads in flight per lane before they are accumulated.
template <int LANES, int THREADS, int U = 8>
__global__ void __launch_bounds__(THREADS) k_sls(const float* __restrict__ tables,
                                                 const int64_t* __restrict__ tab_off,
                                                 int64_t row_stride,
                                                 const int64_t* __restrict__ rows,
                                                 const int* __restrict__ indices,
                                                 const int* __restrict__ offsets, int B, int T,
                                                 int D, float* __restrict__ X, int x_stride,
                                                 int x_slot0, int* __restrict__ flag) {
  constexpr int GROUPS = THREADS / LANES;
  __shared__ int s_off[GROUPS + 1];
  const int nbags = T * B;
  const int g0 = blockIdx.x * GROUPS;
  for (int i = threadIdx.x; i <= GROUPS; i += THREADS) {
    const int g = min(g0 + i, nbags);
    s_off[i] = offsets[g];
  }
  __syncthreads();
  const int grp = threadIdx.x / LANES;
  const int sub = threadIdx.x % LANES;
  const int g = g0 + grp;
  if (g >= nbags) return;
  const int t = g / B, b = g - t * B;
  const int lo = s_off[grp], hi = s_off[grp + 1];
  const int64_t toff = __ldg(&tab_off[t]);
  const int64_t nrows = __ldg(&rows[t]);
  const bool active = (sub * 4) < D;
  const int col = active ? sub * 4 : 0;
  const float4* __restrict__ tab = reinterpret_cast<const float4*>(tables + toff + col);
  const int64_t row_stride4 = row_stride / 4;
  const unsigned gmask = (LANES == 32) ? 0xffffffffu
                                       : (((1u << LANES) - 1u) << ((threadIdx.x & 31) & ~(LANES - 1)));
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  bool oob = false;
  for (int base = lo; base < hi; base += LANES) {
    const int n = min(LANES, hi - base);
    int my = (sub < n) ? __ldg(&indices[base + sub]) : 0;
    if (sub < n && (my < 0 || static_cast<int64_t>(my) >= nrows)) {
      oob = true;
      my = 0;
    }
#pragma unroll
    for (int kk = 0; kk < LANES; kk += U) {
      if (kk >= n) break;
      float4 v[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int r = __shfl_sync(gmask, my, kk + k, LANES);
        if (kk + k < n) v[k] = ldg_stream(tab + static_cast<int64_t>(r) * row_stride4);
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        if (kk + k < n) {
          acc.x += v[k].x;
          acc.y += v[k].y;
          acc.z += v[k].z;
          acc.w += v[k].w;
        }
      }
    }
  }
  if (oob) atomicOr(flag, 1);
  if (active) {
    float4* dst = reinterpret_cast<float4*>(X + (static_cast<int64_t>(b) * x_stride +
                                                 static_cast<int64_t>(x_slot0 + t) * D + col));
    *dst = acc;
  }
}

void launch_sls(const float* tables, const int64_t* tab_off, int64_t row_stride,
                const int64_t* rows, const int* indices, const int* offsets, int B, int T, int D,
                float* X, int x_stride_items, int x_slot0, int* flag, cudaStream_t s) {
  const int nbags = T * B;
  if (nbags == 0) return;
  constexpr int THREADS = 256;
  const int lanes_needed = D / 4;
  if (lanes_needed <= 8) {
    constexpr int L = 8;
    k_sls<L, THREADS><<<(nbags + THREADS / L - 1) / (THREADS / L), THREADS, 0, s>>>(
        tables, tab_off, row_stride, rows, indices, offsets, B, T, D, X, x_stride_items, x_slot0, flag);
  } else if (lanes_needed <= 16) {
    constexpr int L = 16;
    k_sls<L, THREADS><<<(nbags + THREADS / L - 1) / (THREADS / L), THREADS, 0, s>>>(
        tables, tab_off, row_stride, rows, indices, offsets, B, T, D, X, x_stride_items, x_slot0, flag);
  } else {
    constexpr int L = 32;
    k_sls<L, THREADS><<<(nbags + THREADS / L - 1) / (THREADS / L), THREADS, 0, s>>>(
        tables, tab_off, row_stride, rows, indices, offsets, B, T, D, X, x_stride_items, x_slot0, flag);
  }
}

}  // namespace rec
