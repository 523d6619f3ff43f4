#include <algorithm>
// k_mlp.cu — a whole FC stack (bottom MLP, or top MLP + width-1 output) in ONE kernel per
// 128-row tile (Table I Bottom-FC / Predict-FC).
//
// Per-layer GEMM launches are latency chains at serving batch sizes (launch, TMA descriptor
// and weight fetch, commit, epilogue: 7-10 us each for ~1 us of work, see profiles/).  Here
// the layers of a tile run back to back inside one CTA:
//   layer 0:  A = activations from global (TMA, 64-wide K boxes, SWIZZLE_128B)
//   layer l:  A = the previous layer's output, written by the epilogue warps straight into
//             shared memory in the same 128-byte-swizzled K-major layout TMA produces, so
//             tcgen05.mma reads it with the same descriptors
//   all l:    W = weight tiles streamed by TMA through an S-stage ring (<= 256 rows per
//             N-chunk), accumulators in TMEM (N <= 512 columns)
//   epilogue: + bias, ReLU -> bf16 -> smem (hidden layers); the last layer writes fp32 X
//             slot 0 (bottom) or folds the width-1 output layer + sigmoid (top -> CTR).
// Warp roles (320 threads): warp 0 TMA producer, warp 1 single-thread MMA issuer, warps 2-9
// epilogue: warp w owns TMEM lanes 32*(w%4) .. +31 (tile rows) and half (w-2)/4 of every
// layer's 64-column groups, so two warps per SM sub-partition hide each other's TMEM-load,
// math and shared-store latency.  No split-K, no atomics: an item's result is independent of
// its batch (batch invariance).
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "sm100.cuh"

namespace rec {

int g_dense_prio = 0;

constexpr int CBM = 128;
constexpr int CBK = 64;
constexpr int C_A_BYTES = CBM * CBK * 2;     // 16 KB: one A k-block (128 rows x 128 B)
// ring stage = one A k-block + one W k-block of an N-chunk (nchunk = 128 or 256 rows:
// 32 KB or 48 KB per stage; chain_configure picks the smallest ring that keeps the CTA's
// shared memory under the co-location budget, see chain_configure)

__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define STAMP(i)                                            \
  do {                                                      \
    if (args.dbg && blockIdx.x == 0) args.dbg[i] = gtimer(); \
  } while (0)

__device__ __forceinline__ const CUtensorMap* wmap(const ChainMaps& mp, int l) {
  return l == 0 ? &mp.w0 : l == 1 ? &mp.w1 : l == 2 ? &mp.w2 : &mp.w3;
}

// Epilogue probes (ChainArgs::dbg_mode) exist only in a diagnostic build (-DREC_DEBUG_KNOBS):
// the shipped library can never skip epilogue loads or stores.
#ifdef REC_DEBUG_KNOBS
constexpr bool kDbgKnobs = true;
#else
constexpr bool kDbgKnobs = false;
#endif

#ifndef REC_CHAIN_EPI_WARPS
#define REC_CHAIN_EPI_WARPS 8  // 4 or 8 (A/B: register footprint vs epilogue latency)
#endif
constexpr int C_EPI_THREADS = 32 * REC_CHAIN_EPI_WARPS;
constexpr int C_HALVES = C_EPI_THREADS / 128;  // warps per TMEM lane quarter
#ifndef REC_CHAIN_Q
#define REC_CHAIN_Q 2  // tcgen05.ld x16 in flight per wait (2: 32 columns; 4: 64 columns, +50 regs)
#endif
constexpr int C_Q = REC_CHAIN_Q;
#ifndef REC_CHAIN_MINB
#define REC_CHAIN_MINB 1
#endif
constexpr int C_THREADS = 64 + C_EPI_THREADS;

// ---------------------------------------------------------------- fused dot interaction
// Top chain only (ChainArgs::ir = T + 1): the layer-0 A operand of tile row r is the
// interaction row of item m0 + r (reading R1, k_interact.cu), computed here by the epilogue
// warps straight into the swizzled activation buffer instead of by a separate kernel and a
// TMA load.  Same arithmetic in the same order as k_interact (fp32 FMA chain over k = 0..D-1
// per pair, round-to-nearest bf16), so the fused and unfused paths are bit-identical.
__device__ __forceinline__ void act_st_bf16(uint8_t* act, int r, int col, float v) {
  uint8_t* blk = act + (col >> 6) * C_A_BYTES + r * 128;
  const int u = (col & 63) >> 3;
  *reinterpret_cast<__nv_bfloat16*>(blk + ((u ^ (r & 7)) << 4) + (col & 7) * 2) = __float2bfloat16_rn(v);
}
__device__ __forceinline__ void act_st_unit(uint8_t* act, int r, int q, float4 a, float4 b) {
  uint8_t* blk = act + (q >> 3) * C_A_BYTES + r * 128;
  const __nv_bfloat162 h0 = __floats2bfloat162_rn(a.x, a.y), h1 = __floats2bfloat162_rn(a.z, a.w);
  const __nv_bfloat162 h2 = __floats2bfloat162_rn(b.x, b.y), h3 = __floats2bfloat162_rn(b.z, b.w);
  *reinterpret_cast<uint4*>(blk + (((q & 7) ^ (r & 7)) << 4)) =
      make_uint4(*reinterpret_cast<const uint32_t*>(&h0), *reinterpret_cast<const uint32_t*>(&h1),
                 *reinterpret_cast<const uint32_t*>(&h2), *reinterpret_cast<const uint32_t*>(&h3));
}
// Pairs (i, j) with I0 <= i < I1, 0 <= j < i (p = i(i-1)/2 + j) of one item; the half with
// I0 == 1 also writes bf16(x_b) to columns 0..D-1.  xrow == nullptr: a row past M (zeros).
// Chunks of 4 k are prefetched one ahead (the row's vectors come from L2).
// Measured (RMC1, 16 co-located streams): -0.4 % against the separate kernel, and -1.2 % with
// a two-ahead prefetch (124 -> 140 registers): the chain CTA's longer residency and larger
// register file cost the co-running SLS CTAs more than the saved launch, so it is opt-in
// (REC_FUSE_INTERACT=1).
template <int D, int I0, int I1>
__device__ __forceinline__ void interact_part(const float* __restrict__ xrow, int r, uint8_t* act) {
  constexpr int C = D / 4;
  constexpr int P0 = I0 * (I0 - 1) / 2, NPP = I1 * (I1 - 1) / 2 - P0;
  float acc[NPP];
#pragma unroll
  for (int p = 0; p < NPP; ++p) acc[p] = 0.f;
  const float4* xb = reinterpret_cast<const float4*>(xrow);
  const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
  float4 cur[I1], nxt[I1];
#pragma unroll
  for (int i = 0; i < I1; ++i) cur[i] = xb ? __ldg(xb + i * C) : z4;
  float4 x0prev = z4;
#pragma unroll 1
  for (int c = 0; c < C; ++c) {
    if (c + 1 < C) {
#pragma unroll
      for (int i = 0; i < I1; ++i) nxt[i] = xb ? __ldg(xb + i * C + c + 1) : z4;
    }
#pragma unroll
    for (int i = I0; i < I1; ++i)
#pragma unroll
      for (int j = 0; j < i; ++j) {
        float& a = acc[i * (i - 1) / 2 + j - P0];
        a = fmaf(cur[i].x, cur[j].x, a);
        a = fmaf(cur[i].y, cur[j].y, a);
        a = fmaf(cur[i].z, cur[j].z, a);
        a = fmaf(cur[i].w, cur[j].w, a);
      }
    if (I0 == 1) {
      if (c & 1) act_st_unit(act, r, c >> 1, x0prev, cur[0]);
      x0prev = cur[0];
    }
#pragma unroll
    for (int i = 0; i < I1; ++i) cur[i] = nxt[i];
  }
#pragma unroll
  for (int p = 0; p < NPP; ++p) act_st_bf16(act, r, D + P0 + p, acc[p]);
}
// split point: the pairs of rows i < S and i >= S are about half each
__host__ __device__ constexpr int interact_split(int R) {
  int S = 2;
  while (S * (S - 1) < R * (R - 1) / 2) ++S;
  return S;
}

template <int IR, int ID>
__global__ void __launch_bounds__(C_THREADS, REC_CHAIN_MINB)
    k_mlp_chain(const __grid_constant__ ChainMaps maps, const ChainArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const int S = args.stages;
  const int NCH = args.nchunk;
  const int C_STAGE = C_A_BYTES + NCH * CBK * 2;
  uint8_t* ring = smem;                                   // S x C_STAGE
  uint8_t* act = smem + S * C_STAGE;                      // act_kblocks x 16 KB
  float* s_bias = reinterpret_cast<float*>(act + args.act_kblocks * C_A_BYTES);  // bias_total
  float* s_wl = s_bias + args.bias_total;                 // [N_last]
  float* s_dot = s_wl + args.wl_n + 2;                    // [128] CTR partial of half 1
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_dot + CBM);
  uint64_t* full = bars;
  uint64_t* empty = bars + S;
  // acc_full[b] MMA -> epilogue, one phase per layer of a tile using TMEM buffer b;
  // tmem_empty[b] epilogue -> MMA, one phase per tile using buffer b (its TMEM has been read);
  // act_ready epilogue -> MMA, one phase per hidden layer (its activations are in smem).
  // Persistent launches alternate two TMEM accumulators (args.dbuf), so tile j + 1's MMAs run
  // while the epilogue still reads tile j; one-tile launches only use buffer 0.
  uint64_t* acc_full = bars + 2 * S;        // [2]
  uint64_t* tmem_empty = bars + 2 * S + 2;  // [2]
  uint64_t* act_ready = bars + 2 * S + 4;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2 * S + 5);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * CBM;
  // With PDL (args.pdl) this read precedes cudaGridDependencySynchronize().  It is safe
  // because of a launch-order invariant (enqueue_interact_top): the PDL predecessor of a
  // chain is always k_interact, which never writes *dM; *dM is written by the batch's first
  // kernel (k_sls_synth / k_gen_*), which completed before k_interact started (a plain
  // stream / graph dependency).  A chain must never be PDL-launched directly after a kernel
  // that writes *dM.
  const int M = args.dM ? *args.dM : args.M;
  if (m0 >= M) return;
  const int nl = args.nlayers;
  if (threadIdx.x == 0) STAMP(0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      sm100::mbar_init(&full[s], 1);
      sm100::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      sm100::mbar_init(&acc_full[b], 1);
      sm100::mbar_init(&tmem_empty[b], C_EPI_THREADS);
    }
    sm100::mbar_init(act_ready, C_EPI_THREADS);
    sm100::fence_mbar_init();
    sm100::tma_prefetch_desc(&maps.a0);
    for (int l = 0; l < nl; ++l) sm100::tma_prefetch_desc(wmap(maps, l));
  }
  const int tcols = args.tmem_cols * (args.dbuf ? 2 : 1);
  if (warp == 0) sm100::tmem_alloc(tslot, tcols);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tslot;
  if (threadIdx.x == 0) STAMP(1);

  if (warp == 0) {
    // ------------------------------------------------ TMA producer: (layer, n-chunk, k-block)
    // With PDL, the weight tiles of the first ring fill do not depend on the predecessor
    // grid: issue them before waiting for it, then only the A tiles wait (pre stages).
    int pre = 0;
    if (IR == 0 && args.pdl) {
      const int nkb0 = (args.K[0] + CBK - 1) / CBK;
      pre = min(S, nkb0 * ((args.N[0] + NCH - 1) / NCH));
      if (lane == 0) {
        for (int i = 0; i < pre; ++i) {
          uint8_t* st = ring + i * C_STAGE;
          sm100::mbar_arrive_expect_tx(&full[i], C_A_BYTES + args.wbox[0] * CBK * 2);
          sm100::tma_load_2d(st + C_A_BYTES, wmap(maps, 0), &full[i], (i % nkb0) * CBK, (i / nkb0) * NCH);
        }
      }
      __syncwarp();
      cudaGridDependencySynchronize();  // A written by the predecessor grid
    }
    int it = 0;
    // persistent launches (grid < tiles, large batches): this CTA's tiles m0, m0 + grid * 128, ..
    // — the ring keeps streaming across tiles, so the next tile's loads overlap this epilogue
    for (int mt = m0; mt < M; mt += gridDim.x * CBM) {
    for (int l = 0; l < nl; ++l) {
      const int K = args.K[l], N = args.N[l];
      const int nkb = (K + CBK - 1) / CBK;
      for (int n0 = 0; n0 < N; n0 += NCH) {
        const int box_rows = args.wbox[l];
        const bool a_tma = l == 0 && IR == 0;  // fused interaction: layer-0 A is built in smem
        const uint32_t bytes = (a_tma ? C_A_BYTES : 0) + box_rows * CBK * 2;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % S, use = it / S;
          if (use > 0) sm100::mbar_wait(&empty[s], (use - 1) & 1);
          if (lane == 0) {
            uint8_t* st = ring + s * C_STAGE;
            if (it >= pre) sm100::mbar_arrive_expect_tx(&full[s], bytes);
            if (a_tma) sm100::tma_load_2d(st, &maps.a0, &full[s], kb * CBK, mt);
            if (it >= pre) sm100::tma_load_2d(st + C_A_BYTES, wmap(maps, l), &full[s], kb * CBK, n0);
            if (it == 0) STAMP(2);
          }
          __syncwarp();
        }
      }
    }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ single-thread MMA issuer
    int it = 0, tile = 0;
    for (int mt = m0; mt < M; mt += gridDim.x * CBM, ++tile) {
    for (int l = 0; l < nl; ++l) {
      const int K = args.K[l], N = args.N[l];
      const int nkb = (K + CBK - 1) / CBK;
      const int buf = args.dbuf ? (tile & 1) : 0;
      const int use = args.dbuf ? (tile >> 1) : tile;   // earlier tiles on this buffer
      if (l == 0 && use > 0) {  // the epilogue has read this buffer's previous tile
        sm100::mbar_wait(&tmem_empty[buf], (use - 1) & 1);
        sm100::tc_fence_after();
      }
      if (l > 0 || IR) {  // the previous layer's activations (or the interaction) are in smem
        sm100::mbar_wait(act_ready, (IR ? l : tile * (nl - 1) + l - 1) & 1);
        sm100::tc_fence_after();
      }
      const uint32_t tbase = tmem + static_cast<uint32_t>(buf * args.tmem_cols);
      for (int n0 = 0; n0 < N; n0 += NCH) {
        const int nc = min(NCH, args.wbox[l]);
        const uint32_t idesc = sm100::idesc_bf16_f32(CBM, nc);
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % S, use = it / S;
          sm100::mbar_wait(&full[s], use & 1);
          sm100::tc_fence_after();
          if (lane == 0) {
            if (it == 0) STAMP(3);
            const uint32_t st = sm100::smem_u32(ring + s * C_STAGE);
            const uint64_t da = sm100::umma_desc_sw128(l == 0 && IR == 0 ? st : sm100::smem_u32(act + kb * C_A_BYTES));
            const uint64_t db = sm100::umma_desc_sw128(st + C_A_BYTES);
#pragma unroll
            for (int k = 0; k < CBK / 16; ++k)
              sm100::mma_bf16_ss(tbase + n0, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
            sm100::mma_commit(&empty[s]);
            if (kb == nkb - 1 && n0 + NCH >= N) {
              sm100::mma_commit(&acc_full[buf]);
              STAMP(4 + l);
            }
          }
          __syncwarp();
        }
      }
    }
    }
  } else {
    // ------------------------------------------------ epilogue warps 2..9
    const int et = threadIdx.x - 64;                 // 0..255
    const int half = et >> 7;                        // column-group half of this warp
    for (int i = et; i < args.bias_total; i += C_EPI_THREADS) s_bias[i] = __ldg(&args.bias_all[i]);
    if (args.mode_last == GEMM_OUT_CTR)
      for (int i = et; i < args.wl_n; i += C_EPI_THREADS) s_wl[i] = __ldg(&args.w_last[i]);
    asm volatile("bar.sync 1, %0;" ::"n"(C_EPI_THREADS) : "memory");   // epilogue warps only
    const int qw = warp & 3;                         // TMEM lane quarter of this warp
    const int r = qw * 32 + lane;                    // tile row
    int tile = 0;
    for (int mt = m0; mt < M; mt += gridDim.x * CBM, ++tile) {
    const int row = mt + r;
    const bool row_ok = row < M;
    const int buf = args.dbuf ? (tile & 1) : 0;
    const int use = args.dbuf ? (tile >> 1) : tile;
    const uint32_t trow = tmem + (static_cast<uint32_t>(qw * 32) << 16) +
                          static_cast<uint32_t>(buf * args.tmem_cols);
    if constexpr (IR > 0) {
      if (args.pdl) cudaGridDependencySynchronize();  // X written by the predecessor grids
      const float* xrow = row_ok ? args.ix + static_cast<int64_t>(row) * IR * ID : nullptr;
      constexpr int SP = interact_split(IR);
      if (C_HALVES == 1 || half == 0) interact_part<ID, 1, SP>(xrow, r, act);
      if (C_HALVES == 1 || half == 1) {
        interact_part<ID, SP, IR>(xrow, r, act);
        for (int c = ID + IR * (IR - 1) / 2; c < args.K[0]; ++c) act_st_bf16(act, r, c, 0.f);
      }
      fence_async_smem();
      sm100::tc_fence_before();
      sm100::mbar_arrive(act_ready);
    }
    int boff = 0;
    for (int l = 0; l < nl; ++l) {
      const int N = args.N[l];
      const bool last = l == nl - 1;
      sm100::mbar_wait(&acc_full[buf], (use * nl + l) & 1);
      sm100::tc_fence_after();
      if (et == 0) STAMP(8 + 2 * l);
      float dot = 0.f;
      const int cols = last ? N : ((N + CBK - 1) / CBK) * CBK;  // hidden: zero the K padding
      // 64 columns per round: four tcgen05.ld (16 columns each) in flight, ONE wait, then the
      // math / stores of all four (a wait per 16 columns serialised the epilogue).
#pragma unroll 1
      for (int gg = 64 * half; gg < cols; gg += 64 * C_HALVES) {
#pragma unroll 1
      for (int g0 = gg; g0 < gg + 64 && g0 < cols; g0 += 16 * C_Q) {
        uint32_t rr[C_Q][16];
        if (kDbgKnobs && (args.dbg_mode & 1)) {
#pragma unroll
          for (int q = 0; q < C_Q; ++q)
#pragma unroll
            for (int j = 0; j < 16; ++j) rr[q][j] = 0u;
        } else {
#pragma unroll
          for (int q = 0; q < C_Q; ++q)
            if (g0 + 16 * q < N) sm100::tmem_ld_32x32b_x16(trow + g0 + 16 * q, rr[q]);
          sm100::tmem_ld_wait();
        }
#pragma unroll
        for (int q = 0; q < C_Q; ++q) {
          const int c0 = g0 + 16 * q;
          if (c0 >= cols) break;
          float v[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int c = c0 + j;
            float x = 0.f;
            if (c < N) x = fmaxf(__uint_as_float(rr[q][j]) + s_bias[boff + c], 0.f);
            v[j] = x;
          }
          if (kDbgKnobs && !last && (args.dbg_mode & 2)) {
            dot += v[0];  // keep the math alive, skip the stores
          } else if (!last) {
            // bf16 into the swizzled K-major A operand of layer l+1: column c0 lies in k-block
            // c0/64, 16-byte unit (c0%64)/8 (and the next one), XOR-swizzled by row % 8.
            uint32_t p[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
              p[j] = *reinterpret_cast<uint32_t*>(&h);
            }
            uint8_t* blk = act + (c0 / CBK) * C_A_BYTES + r * 128;
            const int u = (c0 % CBK) / 8;
            *reinterpret_cast<uint4*>(blk + ((u ^ (r & 7)) << 4)) = make_uint4(p[0], p[1], p[2], p[3]);
            *reinterpret_cast<uint4*>(blk + (((u + 1) ^ (r & 7)) << 4)) = make_uint4(p[4], p[5], p[6], p[7]);
          } else if (args.mode_last == GEMM_OUT_X_F32) {
            if (row_ok) {
              float* dst = args.out_f32 + static_cast<int64_t>(row) * args.ldo + c0;
              if (c0 + 16 <= N) {
                float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
                for (int j = 0; j < 4; ++j) d4[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
              } else {
#pragma unroll
                for (int j = 0; j < 16; ++j)
                  if (c0 + j < N) dst[j] = v[j];
              }
            }
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (c0 + j < N) dot = fmaf(v[j], s_wl[c0 + j], dot);
          }
        }
      }
      }
      boff += N;
      if (et == 0) STAMP(9 + 2 * l);
      if (!last) {
        fence_async_smem();          // generic-proxy smem writes -> visible to tcgen05.mma
        sm100::tc_fence_before();    // our tcgen05.ld of this layer are complete
        sm100::mbar_arrive(act_ready);
      } else if (args.mode_last == GEMM_OUT_CTR) {
        // the two halves' partial dots meet in smem: CTR = sigmoid(d_half0 + d_half1 + b)
        if (C_HALVES > 1) {
          if (half == 1) s_dot[r] = dot;
          asm volatile("bar.sync 1, %0;" ::"n"(C_EPI_THREADS) : "memory");
        }
        if (half == 0 && row_ok) {
          const float logit = (C_HALVES > 1 ? dot + s_dot[r] : dot) + args.b_last;
          args.ctr[row] = 1.f / (1.f + __expf(-logit));
          if (args.logit) args.logit[row] = logit;
        }
      }
    }
    if (IR == 0) {  // this tile's TMEM has been read: a later tile may overwrite the buffer
      sm100::tc_fence_before();
      sm100::mbar_arrive(&tmem_empty[buf]);
    }
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc(tmem, tcols);
  if (threadIdx.x == 0) STAMP(15);
}

size_t chain_smem_bytes(const ChainArgs& a) {
  return 1024 + static_cast<size_t>(a.stages) * (C_A_BYTES + a.nchunk * CBK * 2) +
         static_cast<size_t>(a.act_kblocks) * C_A_BYTES +
         sizeof(float) * (a.bias_total + a.wl_n + 2 + CBM) + 8 * (2 * a.stages + 8);
}

bool chain_configure(ChainArgs& a) {
  // Shared-memory budget: a chain CTA co-resides with SLS CTAs of other co-located streams;
  // every KB of shared memory it takes is carved out of those SMs' L1, which the SLS gathers
  // need for their in-flight rows (measured: 208 KB chains cost 7 % RMC1 throughput vs
  // <= 160 KB).  Pick the fastest ring within REC_CHAIN_SMEM KB (default 132).
  int budget = 132;
  if (const char* e = getenv("REC_CHAIN_SMEM")) budget = atoi(e);
  int smax = 4;
  if (const char* e = getenv("REC_CHAIN_STAGES")) smax = atoi(e) < 2 ? 2 : atoi(e) > 4 ? 4 : atoi(e);
  for (int nch : {256, 128}) {
    for (int s = smax; s >= 2; --s) {
      a.stages = s;
      a.nchunk = nch;
      if (chain_smem_bytes(a) <= static_cast<size_t>(budget) * 1024) return true;
    }
  }
  // Over budget: per-layer GEMMs instead (measured on RMC3: a 192-KB bottom chain with the
  // 2560-wide layer runs 8 CTAs for 80 us at B = 1024 and costs 13 % co-located throughput
  // against the per-layer kernels).
  return false;
}

using ChainKernel = void (*)(const ChainMaps, const ChainArgs);
static ChainKernel chain_kernel(int ir) {
  switch (ir) {
    case 9: return k_mlp_chain<9, 32>;
    case 11: return k_mlp_chain<11, 32>;
    default: return k_mlp_chain<0, 0>;
  }
}

bool chain_interact_supported(int T, int D) { return D == 32 && (T + 1 == 9 || T + 1 == 11); }

void chain_prepare() {
  for (int ir : {0, 9, 11})
    cudaFuncSetAttribute(chain_kernel(ir), cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
}

extern int g_chain_persistent;

// Grid of a chain launch: one CTA per 128-row tile, or — when the tiles exceed one wave of
// resident CTAs (large batches) and the interaction is not fused — one wave of persistent CTAs
// that each walk tiles blockIdx, blockIdx + grid, ... (the ring streams across tiles, so a
// tile's operand loads overlap the previous tile's epilogue; every tile is computed exactly as
// by a CTA of its own, so the bits do not depend on the grid).
static int chain_grid(const ChainArgs& a, size_t smem) {
  static int nsm = [] {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  const int tiles = (a.M + CBM - 1) / CBM;
  if (a.ix || g_chain_persistent == 0) return tiles;
  const int tc = std::max(a.tmem_cols, 32) * (a.tmem_cols <= 256 ? 2 : 1);  // double-buffered
  const int per_sm = std::max(1, std::min(512 / tc, static_cast<int>((228 * 1024) / (smem + 1024))));
  return std::min(tiles, nsm * per_sm);
}

int g_chain_persistent = 1;  // REC_CHAIN_PERSISTENT=0: one CTA per tile at every batch size

void launch_mlp_chain(const ChainMaps& maps, const ChainArgs& a0, cudaStream_t s) {
  if (a0.M <= 0) return;
  const size_t smem = chain_smem_bytes(a0);
  const ChainKernel k = chain_kernel(a0.ix ? a0.ir : 0);
  const int grid = chain_grid(a0, smem);
  ChainArgs a = a0;
  // two TMEM accumulators when CTAs walk several tiles (tiles > grid) and they fit
  a.dbuf = grid < (a.M + CBM - 1) / CBM && a.tmem_cols <= 256 && !a.ix;
  if (g_dense_prio == 0 && !a.pdl) {
    k<<<grid, C_THREADS, smem, s>>>(maps, a);
    return;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(C_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (g_dense_prio != 0) {
    at[na].id = cudaLaunchAttributePriority;
    at[na++].val.priority = g_dense_prio;
  }
  if (a.pdl) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na++].val.programmaticStreamSerializationAllowed = 1;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  cudaLaunchKernelEx(&cfg, k, maps, a);
}

}  // namespace rec
