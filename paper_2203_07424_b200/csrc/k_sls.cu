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
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace rec {

// Streaming 128-bit load of row `row` (address = base + row * stride_bytes, formed inside the
// asm so no 64-bit address stays live per in-flight load; rows are never reused from L1).
__device__ __forceinline__ float4 ldg_row(const float4* base, uint32_t row, uint32_t stride_bytes) {
  float4 v;
  asm volatile(
      "{\n\t.reg .u64 a;\n\t"
      "mad.wide.u32 a, %4, %5, %6;\n\t"
      "ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [a];\n\t}"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "r"(row), "r"(stride_bytes), "l"(base));
  return v;
}

// ------------------------------------------------------------------------------------
// k_sls_async — the production SLS for D <= 64.  Memory-level parallelism is what bounds a
// random 128-B-row gather on B200 (ncu of the register version: 24 % warps active, 44 % of
// DRAM peak), so rows land in SHARED memory through cp.async (LDGSTS, L1-bypassing .cg):
// an in-flight row costs 16 B of smem per lane instead of 4 registers.  Each lane owns a
// private ring of P rounds x LANES rows; a round is LANES consecutive index positions (one
// index loaded per lane, broadcast by shuffles), so P*LANES rows per group are in flight
// and no CTA barrier is ever needed (each lane reads back exactly the bytes it copied).
// The grid is persistent (all CTAs resident); group i streams the contiguous bag range
// [i*k, (i+1)*k), k = ceil(T*B / groups), whose indices are contiguous in the CSR array,
// flushing a bag's sum when the stream crosses offsets[g+1].  Rows are accumulated in
// index order, exactly like the register kernel below.
__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* gptr) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(gptr) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int LANES, int P>
__global__ void __launch_bounds__(128) k_sls_async(const float* __restrict__ tables,
                                                   const int64_t* __restrict__ tab_off,
                                                   int64_t row_stride,
                                                   const int64_t* __restrict__ rows,
                                                   const int* __restrict__ indices,
                                                   const int* __restrict__ offsets, int B,
                                                   const int* __restrict__ dB, int T, int D,
                                                   float* __restrict__ X, int x_stride, int x_slot0,
                                                   int* __restrict__ flag) {
  extern __shared__ float4 ring[];  // [P][LANES][128 threads]: lanes interleaved (no bank conflicts)
  if (dB) B = *dB;
  const int nbags = T * B;
  constexpr int GPB = 128 / LANES;  // groups per block
  const int total_groups = gridDim.x * GPB;
  const int gid = blockIdx.x * GPB + threadIdx.x / LANES;
  const int k = (nbags + total_groups - 1) / total_groups;
  const int gb0 = gid * k;
  if (gb0 >= nbags) return;
  const int gb1 = min(gb0 + k, nbags);
  const int sub = threadIdx.x % LANES;
  const unsigned gmask = (LANES == 32) ? 0xffffffffu
                                       : (((1u << LANES) - 1u) << ((threadIdx.x & 31) & ~(LANES - 1)));
  const bool active = (sub * 4) < D;
  const int col = active ? sub * 4 : 0;
  const float4* slot = ring + threadIdx.x;  // element (round slot q, row j) at [(q*LANES + j)*128]
  const uint32_t saddr = static_cast<uint32_t>(__cvta_generic_to_shared(slot));

  const int p_begin = __ldg(&offsets[gb0]), p_end = __ldg(&offsets[gb1]);
  const int nrounds = (p_end - p_begin + LANES - 1) / LANES;

  // issue cursor (bag / table of the next row to fetch)
  int ib = gb0, ib_end = __ldg(&offsets[gb0 + 1]);
  int it = gb0 / B;
  const float* itab = tables + __ldg(&tab_off[it]) + col;
  int64_t inrows = __ldg(&rows[it]);
  // consume cursor (bag being summed)
  int cb = gb0, cb_end = ib_end;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  bool oob = false;

  auto flush = [&](int bag) {
    if (active) {
      const int t = bag / B, b = bag - t * B;
      *reinterpret_cast<float4*>(X + (static_cast<int64_t>(b) * x_stride +
                                      static_cast<int64_t>(x_slot0 + t) * D + col)) = acc;
    }
    acc = make_float4(0.f, 0.f, 0.f, 0.f);
  };
  auto load_idx = [&](int r) {
    const int p = p_begin + r * LANES + sub;
    return (r < nrounds && p < p_end) ? __ldg(&indices[p]) : 0;
  };
  auto issue = [&](int r, int mine) {
    const int pr = p_begin + r * LANES;
#pragma unroll
    for (int j = 0; j < LANES; ++j) {
      const int p = pr + j;
      int ri = __shfl_sync(gmask, mine, j, LANES);
      if (p < p_end) {
        while (p >= ib_end) {
          ++ib;
          ib_end = __ldg(&offsets[ib + 1]);
        }
        if (ib / B != it) {
          it = ib / B;
          itab = tables + __ldg(&tab_off[it]) + col;
          inrows = __ldg(&rows[it]);
        }
        if (ri < 0 || static_cast<int64_t>(ri) >= inrows) {
          oob = true;
          ri = 0;
        }
        if (active)
          cp_async16(saddr + static_cast<uint32_t>(((r % P) * LANES + j) * 128 * 16),
                     itab + static_cast<int64_t>(ri) * row_stride);
      }
    }
    cp_async_commit();
  };

  // prologue: P rounds in flight
#pragma unroll
  for (int r = 0; r < P; ++r) {
    const int mine = load_idx(r);
    if (r < nrounds) issue(r, mine);
    else cp_async_commit();
  }
  int nxt = load_idx(P);
  for (int r = 0; r < nrounds; ++r) {
    cp_async_wait<P - 1>();  // round r has landed (this lane's own copies)
    const int pr = p_begin + r * LANES;
    const float4* s = slot + (r % P) * LANES * 128;
#pragma unroll
    for (int j = 0; j < LANES; ++j) {
      const int p = pr + j;
      if (p >= p_end) break;
      while (p >= cb_end) {  // crossing into the next bag(s), empty ones included
        flush(cb);
        ++cb;
        cb_end = __ldg(&offsets[cb + 1]);
      }
      const float4 v = s[j * 128];
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    if (r + P < nrounds) {
      const int cur = nxt;
      nxt = load_idx(r + P + 1);
      issue(r + P, cur);
    } else {
      cp_async_commit();
    }
  }
  cp_async_wait<0>();
  while (cb < gb1) {  // last bag and any trailing empty bags
    flush(cb);
    ++cb;
  }
  if (oob) atomicOr(flag, 1);
}

// Per round a group consumes ROWS = IPL * LANES indices (IPL per lane, prefetched one round
// ahead so the index load never sits in front of the row loads) and issues the row loads in
// sub-batches of U = 8 independent 128-bit loads per lane before accumulating them in order.
template <int LANES>
struct SlsShape {
  static constexpr int IPL = 1;
  static constexpr int ROWS = IPL * LANES;
  static constexpr int U = 8;  // 8 x 16 B in flight per lane keeps ~90 regs: 5 CTAs of 128/SM
};

template <int LANES, int THREADS>
__global__ void __launch_bounds__(THREADS, 5) k_sls(const float* __restrict__ tables,
                                                    const int64_t* __restrict__ tab_off,
                                                    int64_t row_stride,
                                                    const int64_t* __restrict__ rows,
                                                    const int* __restrict__ indices,
                                                    const int* __restrict__ offsets, int B,
                                                    const int* __restrict__ dB, int T,
                                                    int D, float* __restrict__ X, int x_stride,
                                                    int x_slot0, int* __restrict__ flag) {
  using S = SlsShape<LANES>;
  constexpr int GROUPS = THREADS / LANES;
  __shared__ int s_off[GROUPS + 1];
  if (dB) B = *dB;  // device-side batch size (graph replay); grid sized for the capacity
  const int nbags = T * B;
  if (static_cast<int>(blockIdx.x) * GROUPS >= nbags) return;
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
  const uint32_t stride_bytes = static_cast<uint32_t>(row_stride * 4);
  const unsigned gmask = (LANES == 32) ? 0xffffffffu
                                       : (((1u << LANES) - 1u) << ((threadIdx.x & 31) & ~(LANES - 1)));
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  bool oob = false;
  int cur[S::IPL], nxt[S::IPL];
#pragma unroll
  for (int j = 0; j < S::IPL; ++j) {
    const int p = lo + j * LANES + sub;
    cur[j] = p < hi ? __ldg(&indices[p]) : 0;
  }
  for (int base = lo; base < hi; base += S::ROWS) {
#pragma unroll
    for (int j = 0; j < S::IPL; ++j) {  // prefetch the next round's indices
      const int p = base + S::ROWS + j * LANES + sub;
      nxt[j] = p < hi ? __ldg(&indices[p]) : 0;
    }
#pragma unroll
    for (int j = 0; j < S::IPL; ++j) {
      const int p = base + j * LANES + sub;
      if (p < hi && (cur[j] < 0 || static_cast<int64_t>(cur[j]) >= nrows)) {
        oob = true;
        cur[j] = 0;
      }
    }
    const int n = min(S::ROWS, hi - base);
#pragma unroll
    for (int kk = 0; kk < S::ROWS; kk += S::U) {
      if (kk >= n) break;
      float4 v[S::U];
#pragma unroll
      for (int k = 0; k < S::U; ++k) {
        const int r = kk + k;  // row r of the round = index position base + r
        const int rr = __shfl_sync(gmask, cur[r / LANES], r % LANES, LANES);
        if (r < n) v[k] = ldg_row(tab, static_cast<uint32_t>(rr), stride_bytes);
      }
#pragma unroll
      for (int k = 0; k < S::U; ++k) {
        if (kk + k < n) {
          acc.x += v[k].x;
          acc.y += v[k].y;
          acc.z += v[k].z;
          acc.w += v[k].w;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < S::IPL; ++j) cur[j] = nxt[j];
  }
  if (oob) atomicOr(flag, 1);
  if (active) {
    float4* dst = reinterpret_cast<float4*>(X + (static_cast<int64_t>(b) * x_stride +
                                                 static_cast<int64_t>(x_slot0 + t) * D + col));
    *dst = acc;
  }
}

template <int L>
static void launch_l(const float* tables, const int64_t* tab_off, int64_t row_stride,
                     const int64_t* rows, const int* indices, const int* offsets, int B,
                     const int* dB, int T, int D, float* X, int x_stride_items, int x_slot0, int* flag,
                     cudaStream_t s) {
  constexpr int THREADS = 128;
  const int nbags = T * B;
  k_sls<L, THREADS><<<(nbags + THREADS / L - 1) / (THREADS / L), THREADS, 0, s>>>(
      tables, tab_off, row_stride, rows, indices, offsets, B, dB, T, D, X, x_stride_items, x_slot0,
      flag);
}

void launch_sls(const float* tables, const int64_t* tab_off, int64_t row_stride,
                const int64_t* rows, const int* indices, const int* offsets, int B, const int* dB,
                int T, int D, float* X, int x_stride_items, int x_slot0, int* flag, cudaStream_t s) {
  if (T * B == 0) return;
  const int lanes_needed = D / 4;
  // REC_SLS_IMPL=reg selects the register-pipelined kernel (diagnostics / A-B profiling)
  static const int impl = [] {
    const char* e = getenv("REC_SLS_IMPL");
    return (e && e[0] == 'r') ? 1 : 0;
  }();
  if (lanes_needed <= 16 && impl == 0) {
    // persistent grid of k_sls_async: every CTA resident (smem-limited), groups stream bags
    static int grid8 = 0, grid16 = 0;
    constexpr size_t SMEM = 128 * 512;  // 512 B of ring per lane
    int& grid = lanes_needed <= 8 ? grid8 : grid16;
    if (grid == 0) {
      int dev = 0, sms = 0, per_sm = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      if (lanes_needed <= 8) {
        cudaFuncSetAttribute(k_sls_async<8, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sls_async<8, 4>, 128, SMEM);
      } else {
        cudaFuncSetAttribute(k_sls_async<16, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sls_async<16, 2>, 128, SMEM);
      }
      grid = sms * (per_sm > 0 ? per_sm : 1);
    }
    if (lanes_needed <= 8)
      k_sls_async<8, 4><<<grid, 128, SMEM, s>>>(tables, tab_off, row_stride, rows, indices, offsets,
                                                 B, dB, T, D, X, x_stride_items, x_slot0, flag);
    else
      k_sls_async<16, 2><<<grid, 128, SMEM, s>>>(tables, tab_off, row_stride, rows, indices, offsets,
                                                  B, dB, T, D, X, x_stride_items, x_slot0, flag);
  } else if (lanes_needed <= 8) {
    launch_l<8>(tables, tab_off, row_stride, rows, indices, offsets, B, dB, T, D, X, x_stride_items, x_slot0, flag, s);
  } else if (lanes_needed <= 16) {
    launch_l<16>(tables, tab_off, row_stride, rows, indices, offsets, B, dB, T, D, X, x_stride_items, x_slot0, flag, s);
  } else {
    launch_l<32>(tables, tab_off, row_stride, rows, indices, offsets, B, dB, T, D, X, x_stride_items, x_slot0, flag, s);
  }
}

}  // namespace rec
