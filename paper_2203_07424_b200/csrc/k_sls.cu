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
#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "sm100.cuh"
#include "synth.cuh"

#ifndef REC_SLS_MINB
#define REC_SLS_MINB 5  // CTAs of 128 per SM the register budget must allow (5: ~85 regs)
#endif
#ifdef REC_SLS_NO_GDC  // A/B: build without the griddepcontrol instructions
#define SLS_GDC_TRIGGER()
#define SLS_GDC_WAIT()
#else
#define SLS_GDC_TRIGGER() cudaTriggerProgrammaticLaunchCompletion()
#define SLS_GDC_WAIT() cudaGridDependencySynchronize()
#endif
#ifndef REC_SLS_RIF
#define REC_SLS_RIF 8  // independent 128-bit row loads in flight per lane
#endif

#ifdef REC_SLS_TIMELINE  // diagnostic build (scripts/sls_timeline.cu): per-warp %globaltimer
__device__ unsigned long long g_sls_tl[4 * 65536];
#define SLS_STAMP(k)                                                            \
  do {                                                                          \
    if ((threadIdx.x & 31) == 0) {                                              \
      unsigned long long t_;                                                    \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                     \
      const unsigned w_ = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;         \
      if (w_ < 65536) g_sls_tl[4 * w_ + (k)] = t_;                              \
    }                                                                           \
  } while (0)
#else
#define SLS_STAMP(k)
#endif

namespace rec {

int g_sls_prio = 0;

// Same load with an explicit L2 eviction-priority policy (createpolicy): the hot-row prefix
// is read evict_last, everything else evict_first, so hot rows stay L2-resident under the
// streaming gather (the access-policy window does not govern these non-coherent loads).
__device__ __forceinline__ float4 ldg_row_pol(const float4* base, uint32_t row, uint32_t stride_bytes,
                                              uint64_t pol) {
  float4 v;
  asm volatile(
      "{\n\t.reg .u64 a;\n\t"
      "mad.wide.u32 a, %4, %5, %6;\n\t"
      "ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [a], %7;\n\t}"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "r"(row), "r"(stride_bytes), "l"(base), "l"(pol));
  return v;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

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

// Per round a group consumes ROWS = IPL * LANES indices (IPL per lane, prefetched one round
// ahead so the index load never sits in front of the row loads) and issues the row loads in
// sub-batches of U = 8 independent 128-bit loads per lane before accumulating them in order.
template <int LANES, int RIF = REC_SLS_RIF>
struct SlsShape {
  static constexpr int IPL = RIF > LANES ? RIF / LANES : 1;
  static constexpr int ROWS = IPL * LANES;
  static constexpr int U = RIF;  // RIF x 16 B in flight per lane (8: ~90 regs, 5 CTAs of 128/SM)
};

__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Release + acquire RMW at system scope: makes this CTA's earlier stores (ordered before it by
// the CTA barrier) visible before the count, and the last CTA, which reads the final count,
// observes every CTA's stores before it raises the flags (release cumulativity) — without the
// full fence.sc.sys of __threadfence_system() in every CTA.
__device__ __forceinline__ unsigned atom_add_acq_rel_sys(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.sys.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
// LL lines: one 16-byte volatile store / load (each 8-byte {value, epoch} half is single-copy
// atomic, also over NVLink).
__device__ __forceinline__ void st_volatile_v4(uint4* p, uint4 v) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
__device__ __forceinline__ uint4 ld_volatile_v4(const uint4* p) {
  uint4 v;
  asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int LANES, int THREADS, bool P2P = false>
__global__ void __launch_bounds__(THREADS, REC_SLS_MINB) k_sls(const float* __restrict__ tables,
                                                    const int64_t* __restrict__ tab_off,
                                                    int64_t row_stride,
                                                    const int64_t* __restrict__ rows,
                                                    const int* __restrict__ indices,
                                                    const int* __restrict__ offsets, int B,
                                                    const int* __restrict__ dB, int T,
                                                    int D, float* __restrict__ X, int x_stride,
                                                    int x_slot0, int* __restrict__ flag, int row_lo,
                                                    int row_hi, int idx_limit, const P2PArgs p2p) {
  using S = SlsShape<LANES>;
  constexpr int GROUPS = THREADS / LANES;
  __shared__ int s_off[GROUPS + 1];
  if (dB) B = *dB;  // device-side batch size (graph replay); grid sized for the capacity
  const int nbags = T * B;
  if (!P2P && static_cast<int>(blockIdx.x) * GROUPS >= nbags) return;  // (P2P grids are exact)
  const int g0 = blockIdx.x * GROUPS;
  // offsets are clamped to [0, idx_limit] (the readable index count): caller offsets that
  // were flagged by k_check_offsets (REC_E_OFFSETS) can never address outside the indices
  for (int i = threadIdx.x; i <= GROUPS; i += THREADS) {
    const int g = min(g0 + i, nbags);
    s_off[i] = min(max(offsets[g], 0), idx_limit);
  }
  __syncthreads();
  const int grp = threadIdx.x / LANES;
  const int sub = threadIdx.x % LANES;
  const int g = g0 + grp;
  // groups past the last bag stay alive (P2P: every thread reaches the CTA barrier below)
  // with an empty range and no store
  const bool live = g < nbags;
  if (!P2P && !live) return;
  const int t = live ? g / B : 0, b = live ? g - t * B : 0;
  const int lo = live ? s_off[grp] : 0, hi = live ? s_off[grp + 1] : 0;
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
        // row-wise sharding: only rows in [row_lo, row_hi) live on this GPU (others add 0)
        const bool take = r < n && rr >= row_lo && rr < row_hi;
        v[k] = take ? ldg_row(tab, static_cast<uint32_t>(rr - row_lo), stride_bytes)
                    : make_float4(0.f, 0.f, 0.f, 0.f);
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
  if (!P2P) {
    if (active) {  // (live: the non-P2P kernel returned early otherwise)
      float4* dst = reinterpret_cast<float4*>(X + (static_cast<int64_t>(b) * x_stride +
                                                   static_cast<int64_t>(x_slot0 + t) * D + col));
      *dst = acc;
    }
    return;
  }
  // fused all-to-all: item b lives on rank b / Bq as local row b % Bq
  if (active && live) {
    const int p = b / p2p.Bq, bi = p2p.row_off + b - p * p2p.Bq;
    float4* dst = reinterpret_cast<float4*>(p2p.peer_X[p] + (static_cast<int64_t>(bi) * x_stride +
                                                             static_cast<int64_t>(x_slot0 + t) * D + col));
    *dst = acc;
  }
  __syncthreads();  // the CTA's peer stores happen-before thread 0's system-scope release
  if (threadIdx.x == 0) {
    unsigned prev;
    if (p2p.sc_fence) {
      __threadfence_system();
      prev = atomicAdd(p2p.counter, 1u);
    } else {
      prev = atom_add_acq_rel_sys(p2p.counter, 1u);
    }
    if (prev == gridDim.x - 1) {  // last CTA: every CTA's stores are visible
      __threadfence_system();
      for (int q = 0; q < p2p.G; ++q) st_release_sys(p2p.peer_flags[q] + p2p.rank, p2p.epoch);
      *p2p.counter = 0;  // ready for the next launch using this counter (stream-ordered)
    }
  }
}

// One thread per rank: wait until rank q's arrival flag reached this epoch.  Bounded: a peer
// that misses p2p.timeout_ns sets bit 2 of the error flag (rec_sync / rec_query report
// REC_E_NCCL) and the wait returns instead of trapping, so the CUDA context survives.
__global__ void k_p2p_wait(const P2PArgs p2p) {
  const int q = threadIdx.x;
  if (q >= p2p.G) return;
  const unsigned epoch = p2p.words ? p2p.words[0] : p2p.epoch;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (ld_acquire_sys(p2p.my_flags + q) < epoch) {
    __nanosleep(200);
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > p2p.timeout_ns) {
      if (p2p.err_flag) atomicOr(p2p.err_flag, 4);
      return;
    }
  }
}

__global__ void k_p2p_ctr_scatter(const float* __restrict__ ctr, int Bl, int item0, const P2PArgs p2p) {
  unsigned epoch = p2p.epoch;
  if (p2p.words) {  // batch of the slot (captured graphs): this rank's block of ceil(B / G)
    epoch = p2p.words[0];
    const int B = static_cast<int>(p2p.words[1]);
    const int Bq = (B + p2p.G - 1) / p2p.G;
    item0 = p2p.rank * Bq;
    Bl = max(0, min(Bq, B - item0));
  }
  for (int q = 0; q < p2p.G; ++q)
    for (int i = threadIdx.x; i < Bl; i += blockDim.x) p2p.peer_X[q][item0 + i] = ctr[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int q = 0; q < p2p.G; ++q) st_release_sys(p2p.peer_flags[q] + p2p.rank, epoch);
  }
}

__global__ void __launch_bounds__(256) k_p2p_ll_unpack(const P2PArgs p2p, const uint4* __restrict__ ll,
                                                        float* __restrict__ X, int T, int D, int t0, int TL) {
  const unsigned epoch = p2p.words[0];
  const int B = static_cast<int>(p2p.words[1]);
  const int Bq = (B + p2p.G - 1) / p2p.G;
  const int Bl = max(0, min(Bq, B - p2p.rank * Bq));
  const int D4 = D / 4, TR = T - TL;
  const int64_t n = static_cast<int64_t>(Bl) * TR * D4;
  const int64_t x_stride = static_cast<int64_t>(T + 1) * D;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % D4);
    const int64_t r = i / D4;
    const int j = static_cast<int>(r % TR), bi = static_cast<int>(r / TR);
    const int tg = j < t0 ? j : j + TL;
    const uint4* src = ll + ((static_cast<int64_t>(bi) * T + tg) * D4 + c) * 2;
    uint4 u0 = ld_volatile_v4(src), u1 = ld_volatile_v4(src + 1);
    if (u0.y != epoch || u0.w != epoch || u1.y != epoch || u1.w != epoch) {
      unsigned long long t_start;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
      for (;;) {
        __nanosleep(100);
        u0 = ld_volatile_v4(src);
        u1 = ld_volatile_v4(src + 1);
        if (u0.y == epoch && u0.w == epoch && u1.y == epoch && u1.w == epoch) break;
        unsigned long long t_now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_now));
        if (t_now - t_start > p2p.timeout_ns) {
          if (p2p.err_flag) atomicOr(p2p.err_flag, 4);
          return;
        }
      }
    }
    *reinterpret_cast<float4*>(X + bi * x_stride + static_cast<int64_t>(1 + tg) * D + 4 * c) =
        make_float4(__uint_as_float(u0.x), __uint_as_float(u0.z), __uint_as_float(u1.x), __uint_as_float(u1.z));
  }
}

void launch_p2p_ll_unpack(const P2PArgs& p2p, const uint4* ll, float* X, int T, int D, int t0, int TL,
                          int nsm, cudaStream_t s) {
  k_p2p_ll_unpack<<<2 * nsm, 256, 0, s>>>(p2p, ll, X, T, D, t0, TL);
}

void launch_p2p_ctr_scatter(const float* ctr, int Bl, int item0, const P2PArgs& p2p, cudaStream_t s) {
  k_p2p_ctr_scatter<<<1, 512, 0, s>>>(ctr, Bl, item0, p2p);
}

void launch_p2p_wait(const P2PArgs& p2p, cudaStream_t s) {
  k_p2p_wait<<<1, 32 * ((p2p.G + 31) / 32), 0, s>>>(p2p);
}

// Synthetic-index variant (device-synth serving mode, fixed pooling): identical gather /
// accumulate structure, but lane `sub` computes the index of slot base + sub with Philox
// (G2) instead of loading it, so the kernel has no predecessor in the chain and
// no dependent index load in front of its first row loads.
template <int LANES, int THREADS, int RIF, bool HOT = false, bool P2P = false>
__global__ void __launch_bounds__(THREADS, REC_SLS_MINB) k_sls_synth(const __grid_constant__ SegBatch sb,
                                                                        const SlsSynthArgs a) {
  using S = SlsShape<LANES, RIF>;
  constexpr int GROUPS = THREADS / LANES;
  SLS_STAMP(0);
  // Programmatic dependent launch: the next kernel of the stream may be scheduled as soon
  // as our CTAs retire; our reads need nothing from the predecessor grid (indices are
  // synthesised, tables constant), only the writes (X, dB) wait for it (below).
  SLS_GDC_TRIGGER();
  const int B = sb.B;
  const int nbags = a.T * B;  // >= T: a synthetic batch is never empty (block 0 writes dB)
  // Bag -> (CTA, group): blocked (g = CTA * GROUPS + group) or, with a.interleave, dealt
  // round-robin over a grid of exactly nsm x resident CTAs (g = group * gridDim + CTA), so
  // every SM holds the same number of bags and the launch ends without a tail of SMs that
  // got one CTA more (B = 1024: 640 blocked CTAs are 4.3 per SM).
  // (the same predicate as the host's grid choice, sls_interleaved)
  const bool inter = a.interleave && static_cast<int64_t>(a.nsm) * REC_SLS_MINB * GROUPS >=
                                         static_cast<int64_t>(a.T) * a.cap;
  int g = inter ? (threadIdx.x / LANES) * static_cast<int>(gridDim.x) + static_cast<int>(blockIdx.x)
                : static_cast<int>(blockIdx.x) * GROUPS + threadIdx.x / LANES;
  const int cta_has = inter ? static_cast<int>(blockIdx.x) < nbags
                            : static_cast<int>(blockIdx.x) * GROUPS < nbags;
  if (P2P) {
    // sharded: CTAs of the batch all reach the CTA barrier of the flag protocol (groups past
    // the last bag idle on bag 0 and store nothing); CTAs past the batch leave uncounted
    if (!cta_has) return;
  } else if (g >= nbags) {
    return;
  }
  const bool live = g < nbags;
  if (!live) g = 0;
  const int sub = threadIdx.x % LANES;
  const int t = g / B, b = g - t * B;
  const int2 qi = row_item(sb, b);
  const uint64_t R = static_cast<uint64_t>(__ldg(&a.rows[t]));
  const int64_t toff = __ldg(&a.tab_off[t]);
  const uint32_t c2 = (static_cast<uint32_t>(a.t0 + t) << 8) | DOM_INDEX;
  const double zc = a.index_dist == 3 ? zipf_c(R) : 0.0;
  const int* __restrict__ remap = a.remap ? a.remap + __ldg(&a.remap_off[t]) : nullptr;
  const bool active = (sub * 4) < a.D;
  const int col = active ? sub * 4 : 0;
  const float4* __restrict__ tab = reinterpret_cast<const float4*>(a.tables + toff + col);
  const uint32_t stride_bytes = static_cast<uint32_t>(a.row_stride * 4);
  const unsigned gmask = (LANES == 32) ? 0xffffffffu
                                       : (((1u << LANES) - 1u) << ((threadIdx.x & 31) & ~(LANES - 1)));
  const int L = live ? a.L : 0;  // idle groups (sharded launches) read nothing
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  uint64_t pol_hot = 0, pol_cold = 0;
  if (HOT) {
    pol_hot = l2_policy_evict_last();
    pol_cold = l2_policy_evict_first();
  }
  int cur[S::IPL];
#pragma unroll
  for (int q = 0; q < S::IPL; ++q) {
    const int j = q * LANES + sub;
    cur[q] = j < L ? gen_index(j, qi.y, c2, qi.x, a.k0, a.k1, R, a.index_dist, zc) : 0;
    if (remap) cur[q] = __ldg(remap + cur[q]);  // hot-row partition: arena row of the index
  }
  SLS_STAMP(1);
  for (int base = 0; base < L; base += S::ROWS) {
    const int n = min(S::ROWS, L - base);
#pragma unroll
    for (int kk = 0; kk < S::ROWS; kk += S::U) {
      if (kk >= n) break;
      float4 v[S::U];
#pragma unroll
      for (int k = 0; k < S::U; ++k) {
        const int r = kk + k;
        const int rr = __shfl_sync(gmask, cur[r / LANES], r % LANES, LANES);
        if (r < n)
          v[k] = HOT ? ldg_row_pol(tab, static_cast<uint32_t>(rr), stride_bytes,
                                   rr < a.hot_rows ? pol_hot : pol_cold)
                     : ldg_row(tab, static_cast<uint32_t>(rr), stride_bytes);
      }
      if (kk + S::U >= S::ROWS) {  // next round's indices, computed while the rows are in flight
#pragma unroll
        for (int q = 0; q < S::IPL; ++q) {
          const int j = base + S::ROWS + q * LANES + sub;
          cur[q] = j < L ? gen_index(j, qi.y, c2, qi.x, a.k0, a.k1, R, a.index_dist, zc) : 0;
          if (remap) cur[q] = __ldg(remap + cur[q]);
        }
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
      if (base == 0 && kk == 0) SLS_STAMP(2);
    }
  }
  if constexpr (P2P) {
    // fused all-to-all (table-wise sharding): item b lives on rank b / Bq as row b % Bq,
    // its pooled vector of local table t goes to X slot 1 + t0 + t over NVLink
    const P2PArgs& p2p = a.p2p;
    if (active && live) {
      const int Bq = (B + p2p.G - 1) / p2p.G;
      const int p = b / Bq, bi = b - p * Bq;
      if (p2p.ll && p != p2p.rank) {  // flag-in-data lines into the owner's LL buffer
        uint4* dst = p2p.peer_ll[p] + ((static_cast<int64_t>(bi) * p2p.T_all + a.t0 + t) * (a.D / 4) + sub) * 2;
        st_volatile_v4(dst, make_uint4(__float_as_uint(acc.x), p2p.epoch, __float_as_uint(acc.y), p2p.epoch));
        st_volatile_v4(dst + 1, make_uint4(__float_as_uint(acc.z), p2p.epoch, __float_as_uint(acc.w), p2p.epoch));
      } else {
        *reinterpret_cast<float4*>(p2p.peer_X[p] + static_cast<int64_t>(bi) * a.x_stride +
                                   static_cast<int64_t>(1 + a.t0 + t) * a.D + col) = acc;
      }
    }
    __syncthreads();  // the CTA's peer stores happen-before thread 0's system-scope fence
    if (threadIdx.x == 0) {
      if (blockIdx.x == 0 && p2p.words) {  // epoch + batch of this slot for the later kernels
        p2p.words[0] = p2p.epoch;
        p2p.words[1] = static_cast<unsigned>(B);
      }
      const unsigned need = inter ? static_cast<unsigned>(min(nbags, static_cast<int>(gridDim.x)))
                                         : static_cast<unsigned>((nbags + GROUPS - 1) / GROUPS);
      unsigned prev;
      if (p2p.ll) {                // data carries its own epoch: the count is only a hint
        prev = atomicAdd(p2p.counter, 1u);
      } else if (p2p.sc_fence == 1) {  // (REC_P2P_FENCE=1: the round-1 protocol)
        __threadfence_system();
        prev = atomicAdd(p2p.counter, 1u);
#ifdef REC_DEBUG_KNOBS
      } else if (p2p.sc_fence == 2) {  // diagnostic build only: no ordering (results invalid)
        prev = atomicAdd(p2p.counter, 1u);
#endif
      } else {
        prev = atom_add_acq_rel_sys(p2p.counter, 1u);
      }
      if (prev == need - 1) {  // last CTA: every CTA's stores are visible
        __threadfence_system();
        for (int q = 0; q < p2p.G; ++q) st_release_sys(p2p.peer_flags[q] + p2p.rank, p2p.epoch);
        *p2p.counter = 0;      // ready for the slot's next launch (stream-ordered)
      }
    }
    return;
  }
  SLS_GDC_WAIT();  // predecessor grid done: X / dB may be overwritten
  if (blockIdx.x == 0 && threadIdx.x == 0) *a.dB = B;
  if (active)
    *reinterpret_cast<float4*>(a.X + static_cast<int64_t>(b) * a.x_stride +
                               static_cast<int64_t>(1 + t) * a.D + col) = acc;
  if (a.dense_bf && t == 0)  // dense features of item b (same arithmetic as k_gen_dense_seg)
    gen_dense_row(qi.y, qi.x, a.k0, a.k1, a.F, a.Fpad, a.dense_bf + static_cast<int64_t>(b) * a.Fpad,
                  nullptr, sub, LANES);
  SLS_STAMP(3);
}

// TMA row-gather variant (DESIGN.md §6 "SLS via TMA gather4").  Rows travel HBM -> shared
// memory on the tensor-memory accelerator, so the bytes in flight per SM are bounded by the
// shared-memory ring (up to ~200 KB) instead of the register file (~70 KB for the register
// kernel at its occupancy): the small-batch launches of the serving path are latency bound
// on in-flight bytes, not on bandwidth.
//   * persistent grid: SLS_TMA_CTAS_PER_SM x #SM CTAs of 8 warps; warp w owns the contiguous
//     bag range [w * nbags / W, (w + 1) * nbags / W) (bag g = t * B + b, as in k_sls)
//   * a bag is read in chunks of CR = 8 rows: lanes 0..7 compute the chunk's Philox indices,
//     lanes 0..1 each issue one gather4 (4 rows) into the warp's ring slot; one mbarrier per
//     slot (expect_tx = rows x D x 4 bytes)
//   * consume: lane = (row phase ro, column group cg); rows ro, ro + 32/LANES, ... of the chunk
//     accumulate into a float4 in index order; at the end of the bag the row phases are
//     combined by a fixed xor-shuffle tree.  The summation order therefore differs from the
//     sequential register kernel; with the int8 x 2^e tables (value_mode 0, R9) all
//     partial sums are exact, so the result is bit-identical.  Models in fp32 value mode keep
//     the register kernel (model.cu).
constexpr int SLS_TMA_WARPS = 8;
constexpr int SLS_TMA_CR = 8;
constexpr int SLS_TMA_CTAS_PER_SM = 2;
constexpr int SLS_TMA_RING_BYTES = 12 * 1024;  // per warp

template <int LANES>
__global__ void __launch_bounds__(SLS_TMA_WARPS * 32, 1)
    k_sls_synth_tma(const __grid_constant__ SegBatch sb, const SlsSynthArgs a) {
  constexpr int D = LANES * 4;
  constexpr int RP = 32 / LANES;  // row phases per chunk read
  constexpr int ROWB = D * 4;
  constexpr int CHUNKB = SLS_TMA_CR * ROWB;
  extern __shared__ __align__(128) uint8_t smem[];
  const int NST = a.nst;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = smem + static_cast<size_t>(warp) * NST * CHUNKB;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(SLS_TMA_WARPS) * NST * CHUNKB) +
                  warp * NST;
  const int B = sb.B;
  if (blockIdx.x == 0 && threadIdx.x == 0) *a.dB = B;
  if (lane == 0) {
    for (int i = 0; i < NST; ++i) sm100::mbar_init(&bar[i], 1);
    sm100::fence_mbar_init();
  }
  __syncwarp();
  const int nbags = a.T * B;
  const int NW = gridDim.x * SLS_TMA_WARPS;
  const int gw = blockIdx.x * SLS_TMA_WARPS + warp;
  const int b_begin = static_cast<int>(static_cast<int64_t>(gw) * nbags / NW);
  const int b_end = static_cast<int>(static_cast<int64_t>(gw + 1) * nbags / NW);
  const int L = a.L;
  const int nch = (L + SLS_TMA_CR - 1) / SLS_TMA_CR;
  const int total = (b_end - b_begin) * nch;
  const int rs = static_cast<int>(a.row_stride / D);
  const CUtensorMap* map = a.tmap_rows;
  if (total > 0 && lane == 0) sm100::tma_prefetch_desc(map);

  // issue chunk s of this warp into slot s % NST (all lanes participate)
  auto issue = [&](int s) {
    const int g = b_begin + s / nch;
    const int c = s - (s / nch) * nch;
    const int t = g / B, b = g - t * B;
    const int n = min(SLS_TMA_CR, L - c * SLS_TMA_CR);
    int coord = 0;
    if (lane < n) {
      const int2 qi = row_item(sb, b);
      const uint64_t R = static_cast<uint64_t>(__ldg(&a.rows[t]));
      const uint32_t c2 = (static_cast<uint32_t>(t) << 8) | DOM_INDEX;
      const int idx = gen_index(c * SLS_TMA_CR + lane, qi.y, c2, qi.x, a.k0, a.k1, R, a.index_dist,
                                a.index_dist == 3 ? zipf_c(R) : 0.0);
      coord = static_cast<int>(__ldg(&a.tab_off[t]) / D) + idx * rs;
    }
    const int nops = (n + 3) >> 2;
    const int st = s % NST;
    if (lane == 0) sm100::mbar_arrive_expect_tx(&bar[st], nops * 4 * ROWB);
    // lane op (< nops) issues rows 4op..4op+3; padding rows (>= n) repeat row 4op
    const int base = (lane & 1) * 4;
    int r[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int src = base + k < n ? base + k : base;
      r[k] = __shfl_sync(0xffffffffu, coord, src & 31);
    }
    if (lane < nops)
      sm100::tma_gather4(ring + st * CHUNKB + lane * 4 * ROWB, map, &bar[st], 0, r[0], r[1], r[2], r[3]);
  };

  const int pre = min(NST, total);
  for (int s = 0; s < pre; ++s) issue(s);
  const int cg = lane % LANES, ro = lane / LANES;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int s = 0; s < total; ++s) {
    const int st = s % NST;
    sm100::mbar_wait(&bar[st], static_cast<uint32_t>((s / NST) & 1));
    const int c = s % nch;
    const int n = min(SLS_TMA_CR, L - c * SLS_TMA_CR);
    const uint8_t* chunk = ring + st * CHUNKB + cg * 16;
#pragma unroll
    for (int r = ro; r < SLS_TMA_CR; r += RP) {
      if (r < n) {
        const float4 v = *reinterpret_cast<const float4*>(chunk + r * ROWB);
        acc.x += v.x;
        acc.y += v.y;
        acc.z += v.z;
        acc.w += v.w;
      }
    }
    if (c == nch - 1) {  // bag complete: combine the row phases, store, reset
#pragma unroll
      for (int o = LANES; o < 32; o <<= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
        acc.z += __shfl_xor_sync(0xffffffffu, acc.z, o);
        acc.w += __shfl_xor_sync(0xffffffffu, acc.w, o);
      }
      const int g = b_begin + s / nch;
      const int t = g / B, b = g - t * B;
      if (ro == 0)
        *reinterpret_cast<float4*>(a.X + static_cast<int64_t>(b) * a.x_stride +
                                   static_cast<int64_t>(1 + t) * D + cg * 4) = acc;
      acc = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    sm100::fence_proxy_async_smem();
    __syncwarp();
    if (s + NST < total) issue(s + NST);
  }
}

bool sls_tma_supported(int D) { return D == 32 || D == 64 || D == 128; }

void sls_tma_configure(SlsSynthArgs& a) {
  const int chunk = SLS_TMA_CR * a.D * 4;
  a.nst = SLS_TMA_RING_BYTES / chunk < 2 ? 2 : SLS_TMA_RING_BYTES / chunk;
  const size_t smem = static_cast<size_t>(SLS_TMA_WARPS) * a.nst * (chunk + 8);
  void* fn = a.D == 32 ? reinterpret_cast<void*>(k_sls_synth_tma<8>)
             : a.D == 64 ? reinterpret_cast<void*>(k_sls_synth_tma<16>)
                         : reinterpret_cast<void*>(k_sls_synth_tma<32>);
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
}

// The interleaved bag mapping applies when one wave of nsm x REC_SLS_MINB CTAs has a group for
// every bag of the capacity (each group then handles at most one bag).
static bool sls_interleaved(const SlsSynthArgs& a) {
  const int L = a.D / 4 <= 8 ? 8 : a.D / 4 <= 16 ? 16 : 32;
  return a.interleave && static_cast<int64_t>(a.nsm) * REC_SLS_MINB * (128 / L) >=
                             static_cast<int64_t>(a.T) * a.cap;
}

void* sls_synth_kernel(const SlsSynthArgs& a, dim3* grid, dim3* block, size_t* smem) {
  if (a.tma) {
    const int chunk = SLS_TMA_CR * a.D * 4;
    *grid = dim3(a.nsm * SLS_TMA_CTAS_PER_SM);
    *block = dim3(SLS_TMA_WARPS * 32);
    if (smem) *smem = static_cast<size_t>(SLS_TMA_WARPS) * a.nst * (chunk + 8);
    if (a.D == 32) return reinterpret_cast<void*>(k_sls_synth_tma<8>);
    if (a.D == 64) return reinterpret_cast<void*>(k_sls_synth_tma<16>);
    return reinterpret_cast<void*>(k_sls_synth_tma<32>);
  }
  constexpr int THREADS = 128;
  const int L = a.D / 4 <= 8 ? 8 : a.D / 4 <= 16 ? 16 : 32;
  const int nb = a.T * a.cap;
  const int blocked = (nb + THREADS / L - 1) / (THREADS / L);
  // interleaved: one full wave of nsm x REC_SLS_MINB CTAs, each group at most one bag - only
  // when that wave covers every bag of the capacity (RMC1 / RMC3 at d = 1024: 10 240 bags,
  // 11 840 groups); larger batches keep the blocked multi-wave grid (kernel_interleaved)
  *grid = dim3(sls_interleaved(a) ? std::min(blocked, a.nsm * REC_SLS_MINB) : blocked);
  *block = dim3(THREADS);
  if (smem) *smem = 0;
  if (a.p2p.peer_X) {
    if (L == 8) return reinterpret_cast<void*>(k_sls_synth<8, THREADS, REC_SLS_RIF, false, true>);
    if (L == 16) return reinterpret_cast<void*>(k_sls_synth<16, THREADS, REC_SLS_RIF, false, true>);
    return reinterpret_cast<void*>(k_sls_synth<32, THREADS, REC_SLS_RIF, false, true>);
  }
  if (a.hot_rows > 0) {
    if (L == 8) return reinterpret_cast<void*>(k_sls_synth<8, THREADS, REC_SLS_RIF, true>);
    if (L == 16) return reinterpret_cast<void*>(k_sls_synth<16, THREADS, REC_SLS_RIF, true>);
    return reinterpret_cast<void*>(k_sls_synth<32, THREADS, REC_SLS_RIF, true>);
  }
  if (L == 8) return reinterpret_cast<void*>(k_sls_synth<8, THREADS, REC_SLS_RIF>);
  if (L == 16) return reinterpret_cast<void*>(k_sls_synth<16, THREADS, REC_SLS_RIF>);
  return reinterpret_cast<void*>(k_sls_synth<32, THREADS, REC_SLS_RIF>);
}

void launch_sls_synth(const SegBatch& sb, const SlsSynthArgs& a, cudaStream_t s) {
  dim3 grid, block;
  size_t smem = 0;
  void* fn = sls_synth_kernel(a, &grid, &block, &smem);
  void* args[2] = {const_cast<SegBatch*>(&sb), const_cast<SlsSynthArgs*>(&a)};
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = a.pdl;
  at[1].id = cudaLaunchAttributePriority;
  at[1].val.priority = g_sls_prio;
  cfg.attrs = at;
  cfg.numAttrs = g_sls_prio ? 2 : 1;
  if (a.pdl || g_sls_prio) cudaLaunchKernelExC(&cfg, fn, args);
  else cudaLaunchKernel(fn, grid, block, args, smem, s);
}

template <int L>
static void launch_l(const float* tables, const int64_t* tab_off, int64_t row_stride,
                     const int64_t* rows, const int* indices, const int* offsets, int B,
                     const int* dB, int T, int D, float* X, int x_stride_items, int x_slot0, int* flag,
                     cudaStream_t s, int row_lo, int row_hi, int idx_limit) {
  constexpr int THREADS = 128;
  const int nbags = T * B;
  k_sls<L, THREADS><<<(nbags + THREADS / L - 1) / (THREADS / L), THREADS, 0, s>>>(
      tables, tab_off, row_stride, rows, indices, offsets, B, dB, T, D, X, x_stride_items, x_slot0,
      flag, row_lo, row_hi, idx_limit, P2PArgs{});
}

// Row-wise reduction of the staged partial sums, fixed source order q = 0..G-1 (with int8 x 2^e
// tables every partial sum is exact, so the result equals any other summation order).
__global__ void k_p2p_reduce(const float4* __restrict__ stage, float4* __restrict__ X, int Bl,
                             int Bq, int T, int d4, int G) {
  const int64_t n = static_cast<int64_t>(Bl) * T * d4;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t it = e / d4;  // (i, t)
    const int c = static_cast<int>(e - it * d4);
    const int i = static_cast<int>(it / T), t = static_cast<int>(it - static_cast<int64_t>(i) * T);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int q = 0; q < G; ++q) {
      const float4 v = stage[((static_cast<int64_t>(q) * Bq + i) * T + t) * d4 + c];
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    X[(static_cast<int64_t>(i) * (T + 1) + 1 + t) * d4 + c] = acc;
  }
}

void launch_p2p_reduce(const float* stage, float* X, int Bl, int Bq, int T, int D, int G,
                       cudaStream_t s) {
  const int64_t n = static_cast<int64_t>(Bl) * T * (D / 4);
  if (n == 0) return;
  const int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 8));
  k_p2p_reduce<<<blocks, 256, 0, s>>>(reinterpret_cast<const float4*>(stage),
                                      reinterpret_cast<float4*>(X), Bl, Bq, T, D / 4, G);
}

void launch_sls_p2p(const float* tables, const int64_t* tab_off, int64_t row_stride,
                    const int64_t* rows, const int* indices, const int* offsets, int B, int T, int D,
                    int x_stride_items, int x_slot0, int* flag, const P2PArgs& p2p, cudaStream_t s,
                    int row_lo, int row_hi, int idx_limit) {
  constexpr int THREADS = 128;
  const int nbags = T * B;
  if (nbags == 0) return;
  const int L = D / 4 <= 8 ? 8 : D / 4 <= 16 ? 16 : 32;
  const int grid = (nbags + THREADS / L - 1) / (THREADS / L);
  if (L == 8)
    k_sls<8, THREADS, true><<<grid, THREADS, 0, s>>>(tables, tab_off, row_stride, rows, indices, offsets, B,
        nullptr, T, D, nullptr, x_stride_items, x_slot0, flag, row_lo, row_hi, idx_limit, p2p);
  else if (L == 16)
    k_sls<16, THREADS, true><<<grid, THREADS, 0, s>>>(tables, tab_off, row_stride, rows, indices, offsets, B,
        nullptr, T, D, nullptr, x_stride_items, x_slot0, flag, row_lo, row_hi, idx_limit, p2p);
  else
    k_sls<32, THREADS, true><<<grid, THREADS, 0, s>>>(tables, tab_off, row_stride, rows, indices, offsets, B,
        nullptr, T, D, nullptr, x_stride_items, x_slot0, flag, row_lo, row_hi, idx_limit, p2p);
}

void set_max_smem_carveout(int c) {
  cudaFuncSetAttribute(k_sls<8, 128>, cudaFuncAttributePreferredSharedMemoryCarveout, c);
  cudaFuncSetAttribute(k_sls<16, 128>, cudaFuncAttributePreferredSharedMemoryCarveout, c);
  cudaFuncSetAttribute(k_sls<32, 128>, cudaFuncAttributePreferredSharedMemoryCarveout, c);
  cudaFuncSetAttribute(k_sls_synth<8, 128, REC_SLS_RIF>, cudaFuncAttributePreferredSharedMemoryCarveout, c);
  cudaFuncSetAttribute(k_sls_synth<16, 128, REC_SLS_RIF>, cudaFuncAttributePreferredSharedMemoryCarveout, c);
  cudaFuncSetAttribute(k_sls_synth<32, 128, REC_SLS_RIF>, cudaFuncAttributePreferredSharedMemoryCarveout, c);
}

void launch_sls(const float* tables, const int64_t* tab_off, int64_t row_stride,
                const int64_t* rows, const int* indices, const int* offsets, int B, const int* dB,
                int T, int D, float* X, int x_stride_items, int x_slot0, int* flag, cudaStream_t s,
                int row_lo, int row_hi, int idx_limit) {
  if (T * B == 0) return;
  const int lanes_needed = D / 4;
  if (lanes_needed <= 8) {
    launch_l<8>(tables, tab_off, row_stride, rows, indices, offsets, B, dB, T, D, X, x_stride_items, x_slot0, flag, s, row_lo, row_hi, idx_limit);
  } else if (lanes_needed <= 16) {
    launch_l<16>(tables, tab_off, row_stride, rows, indices, offsets, B, dB, T, D, X, x_stride_items, x_slot0, flag, s, row_lo, row_hi, idx_limit);
  } else {
    launch_l<32>(tables, tab_off, row_stride, rows, indices, offsets, B, dB, T, D, X, x_stride_items, x_slot0, flag, s, row_lo, row_hi, idx_limit);
  }
}

}  // namespace rec
