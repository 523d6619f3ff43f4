// k_gemm.cu — FC layers of the bottom and top MLP on the 5th-generation tensor cores
// (Table I Bottom-FC / Predict-FC).
//
//   D[M x N] = A[M x K] . W[N x K]^T   (bf16 operands, fp32 accumulation in TMEM)
//   epilogue: + bias, ReLU, then one of
//     GEMM_OUT_BF16  hidden activation -> bf16 [M][ldo] (A operand of the next layer)
//     GEMM_OUT_X_F32 last bottom layer -> fp32 X slot 0 (interaction input)
//     GEMM_OUT_CTR   last top hidden layer -> per-row fp32 dot with the width-1 output
//                    layer + bias -> sigmoid -> CTR (Predict-FC "...-1")
//
// One CTA (128 threads) per 128 x BN output tile.  Warp 0 lane 0: TMA producer
// (cp.async.bulk.tensor.2d, SWIZZLE_128B, 64-element K boxes) into an S-stage smem ring
// guarded by full/empty mbarriers.  Warp 1 lane 0: single-thread tcgen05.mma issuer
// (M = 128, N = BN, K = 16 per instruction) accumulating in TMEM; tcgen05.commit frees
// each stage and finally signals the epilogue.  Epilogue: all 4 warps, thread = output
// row (TMEM lane), tcgen05.ld 16 columns at a time.  No split-K and no atomics, so an
// item's output bits do not depend on the batch it rides in (batch invariance).
#include <cudaTypedefs.h>

#include <mutex>

#include "common.cuh"
#include "kernels.h"
#include "sm100.cuh"

namespace rec {

int g_gemm_stages = 0;  // cap on the per-layer GEMM ring depth (0 = kernel maximum)

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int A_STAGE_BYTES = BM * BK * 2;  // 16 KB

// MT = 128-row M tiles per CTA sharing every weight stage (MT = 2 halves the weight bytes
// each MMA needs from L2, which is what bounds large-batch GEMMs such as RMC3's 2560x512).
template <int BN, int MT>
__device__ __forceinline__ void gemm_tile(const CUtensorMap* ta, const CUtensorMap* tw,
                                          const GemmArgs& args, int stages) {
  constexpr int B_STAGE_BYTES = BN * BK * 2;
  constexpr int STAGE_BYTES = MT * A_STAGE_BYTES + B_STAGE_BYTES;
  constexpr uint32_t TMEM_COLS = (BN < 32 ? 32 : BN) * MT;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + stages * STAGE_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + stages;
  uint64_t* done = bars + 2 * stages;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2 * stages + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // grid.x runs over N blocks (fastest): the CTAs sharing an A tile are co-scheduled, so the
  // second N block reads A from L2 instead of DRAM
  const int m0 = blockIdx.y * BM * MT, n0 = blockIdx.x * BN;
  const int nkb = (args.K + BK - 1) / BK;
  const int M = args.dM ? *args.dM : args.M;  // device-side batch (graph replay)
  if (m0 >= M) return;                        // whole CTA beyond the batch: nothing to do
  __shared__ float s_bias[BN];                // epilogue operands, staged by warps 2-3
  __shared__ float s_wl[BN];

  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      sm100::mbar_init(&full[s], 1);
      sm100::mbar_init(&empty[s], 1);
    }
    sm100::mbar_init(done, 1);
    sm100::fence_mbar_init();
    sm100::tma_prefetch_desc(ta);
    sm100::tma_prefetch_desc(tw);
  }
  if (warp == 0) sm100::tmem_alloc(tslot, TMEM_COLS);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tslot;

  // Whole warps run the role loops (lane 0 issues), so no lane of a role warp spins on a
  // barrier while its issuing lane still has work (divergent spinning stalls the issuer).
  if (warp == 0) {
    // ---------------- TMA producer
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % stages, it = kb / stages;
      if (it > 0) sm100::mbar_wait(&empty[s], (it - 1) & 1);
      if (lane == 0) {
        uint8_t* sa = smem + s * STAGE_BYTES;
        sm100::mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
#pragma unroll
        for (int h = 0; h < MT; ++h)
          sm100::tma_load_2d(sa + h * A_STAGE_BYTES, ta, &full[s], kb * BK, m0 + h * BM);
        sm100::tma_load_2d(sa + MT * A_STAGE_BYTES, tw, &full[s], kb * BK, n0);
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ---------------- single-thread MMA issuer
    constexpr uint32_t idesc = sm100::idesc_bf16_f32(BM, BN);
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % stages, it = kb / stages;
      sm100::mbar_wait(&full[s], it & 1);
      sm100::tc_fence_after();
      if (lane == 0) {
        const uint32_t sa = sm100::smem_u32(smem + s * STAGE_BYTES);
        const uint64_t db = sm100::umma_desc_sw128(sa + MT * A_STAGE_BYTES);
#pragma unroll
        for (int h = 0; h < MT; ++h) {
          const uint64_t da = sm100::umma_desc_sw128(sa + h * A_STAGE_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // advance 16 bf16 = 32 B along K inside the 128-B swizzled row: +2 in addr>>4
            sm100::mma_bf16_ss(tmem + h * BN, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
          }
        }
        sm100::mma_commit(&empty[s]);
        if (kb == nkb - 1) sm100::mma_commit(done);
      }
      __syncwarp();
    }
  } else {
    // ---------------- warps 2-3: stage bias (and the width-1 layer) while the MMA runs
    for (int c = threadIdx.x - 64; c < BN; c += 64) {
      const int n = n0 + c;
      s_bias[c] = n < args.N ? __ldg(&args.bias[n]) : 0.f;
      if (args.mode == GEMM_OUT_CTR) s_wl[c] = n < args.N ? __ldg(&args.w_last[n]) : 0.f;
    }
  }

  // ---------------- epilogue: thread = row (TMEM lane warp*32 + lane)
  sm100::mbar_wait(done, 0);
  __syncthreads();  // s_bias / s_wl visible to every epilogue thread
  sm100::tc_fence_after();
#pragma unroll 1
  for (int h = 0; h < MT; ++h) {
  const int row = m0 + h * BM + warp * 32 + lane;
  const bool row_ok = row < M;
  const uint32_t trow = tmem + (static_cast<uint32_t>(warp * 32) << 16) + h * BN;
  float dot = 0.f;
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += 16) {
    const int cbase = n0 + c0;
    if (cbase >= args.N) break;  // warp-uniform
    uint32_t r[16];
    sm100::tmem_ld_32x32b_x16(trow + c0, r);
    sm100::tmem_ld_wait();
    float v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      float x = __uint_as_float(r[j]) + s_bias[c0 + j];
      if (args.relu) x = fmaxf(x, 0.f);
      v[j] = x;
    }
    if (!row_ok) continue;
    if (args.mode == GEMM_OUT_BF16) {
      __nv_bfloat16* dst = args.out_bf16 + static_cast<int64_t>(row) * args.ldo + cbase;
      if (cbase + 16 <= args.N) {
        uint32_t p[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
          p[j] = *reinterpret_cast<uint32_t*>(&h);
        }
        uint4* d4 = reinterpret_cast<uint4*>(dst);
        d4[0] = make_uint4(p[0], p[1], p[2], p[3]);
        d4[1] = make_uint4(p[4], p[5], p[6], p[7]);
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (cbase + j < args.N) dst[j] = __float2bfloat16_rn(v[j]);
      }
    } else if (args.mode == GEMM_OUT_X_F32) {
      float* dst = args.out_f32 + static_cast<int64_t>(row) * args.ldo + cbase;
      if (cbase + 16 <= args.N) {
        float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
        for (int j = 0; j < 4; ++j) d4[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (cbase + j < args.N) dst[j] = v[j];
      }
    } else {  // GEMM_OUT_CTR: width-1 output layer folded into the epilogue
#pragma unroll
      for (int j = 0; j < 16; ++j) dot = fmaf(v[j], s_wl[c0 + j], dot);
    }
  }
  if (args.mode == GEMM_OUT_CTR && row_ok) {
    float logit = dot + args.b_last;
    if (args.logit_add) logit += args.logit_add[static_cast<int64_t>(row) * args.add_stride];
    const int64_t o = static_cast<int64_t>(row) * (args.ctr_stride > 0 ? args.ctr_stride : 1);
    args.ctr[o] = 1.f / (1.f + __expf(-logit));
    if (args.logit) args.logit[o] = logit;
  }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc(tmem, TMEM_COLS);
}

// CTA-pair variant (tcgen05 cta_group::2): a cluster of two CTAs computes a
// 256 x BN tile; each CTA stages its own 128 A rows and HALF of the BN weight rows, the
// leader's single thread issues M = 256 MMAs that read both CTAs' shared memory and write
// both CTAs' TMEM (128 lanes x BN columns each), and both CTAs run the epilogue on their rows.
// Per 256 x BN x 64 step the pair loads 2 x (16 + BN/2 * 128 B): half the weight bytes per
// FLOP of a single-CTA 128 x BN tile, with BN TMEM columns per CTA.
template <int BN>
__device__ __forceinline__ void gemm_tile_2sm(const CUtensorMap* ta, const CUtensorMap* tw,
                                              const GemmArgs& args, int stages) {
  constexpr int MT = 1;
  constexpr int B_STAGE_BYTES = (BN / 2) * BK * 2;  // this CTA's half of the weight rows
  constexpr int STAGE_BYTES = MT * A_STAGE_BYTES + B_STAGE_BYTES;
  constexpr uint32_t TMEM_COLS = BN;
  const uint32_t rank = sm100::cluster_ctarank();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + stages * STAGE_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + stages;
  uint64_t* done = bars + 2 * stages;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2 * stages + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // grid.x runs over N blocks (fastest): the CTAs sharing an A tile are co-scheduled, so the
  // second N block reads A from L2 instead of DRAM
  // grid (2, N blocks, M pairs), cluster (2, 1, 1): the pair's CTAs are x = 0 / 1; the N
  // blocks of one M pair are launched next to each other (A tiles re-read from L2)
  const int m0 = (blockIdx.z * 2 + blockIdx.x) * BM, n0 = blockIdx.y * BN;
  const int nkb = (args.K + BK - 1) / BK;
  const int M = args.dM ? *args.dM : args.M;  // device-side batch (graph replay)
  if (static_cast<int>(blockIdx.z * 2) * BM >= M) return;  // whole PAIR beyond the batch
  __shared__ float s_bias[BN];                // epilogue operands, staged by warps 2-3
  __shared__ float s_wl[BN];

  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      sm100::mbar_init(&full[s], 1);
      sm100::mbar_init(&empty[s], 1);
    }
    sm100::mbar_init(done, 1);
    sm100::fence_mbar_init();
    sm100::tma_prefetch_desc(ta);
    sm100::tma_prefetch_desc(tw);
  }
  if (warp == 0) sm100::tmem_alloc_2sm(tslot, TMEM_COLS);
  sm100::tc_fence_before();
  sm100::cluster_sync();  // both CTAs' barriers initialised before any TMA signals the leader's
  sm100::tc_fence_after();
  const uint32_t tmem = *tslot;

  // Whole warps run the role loops (lane 0 issues), so no lane of a role warp spins on a
  // barrier while its issuing lane still has work (divergent spinning stalls the issuer).
  if (warp == 0) {
    // ---------------- TMA producer (both CTAs; completion counted on the leader's barrier)
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % stages, it = kb / stages;
      if (it > 0) sm100::mbar_wait(&empty[s], (it - 1) & 1);
      if (lane == 0) {
        uint8_t* sa = smem + s * STAGE_BYTES;
        if (rank == 0) sm100::mbar_arrive_expect_tx(&full[s], 2 * STAGE_BYTES);
        sm100::tma_load_2d_2sm(sa, ta, &full[s], kb * BK, m0);
        sm100::tma_load_2d_2sm(sa + A_STAGE_BYTES, tw, &full[s], kb * BK,
                               n0 + static_cast<int>(rank) * (BN / 2));
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ---------------- single-thread MMA issuer of the pair (leader CTA only)
    if (rank == 0) {
      constexpr uint32_t idesc = sm100::idesc_bf16_f32(2 * BM, BN);
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % stages, it = kb / stages;
        sm100::mbar_wait(&full[s], it & 1);
        sm100::tc_fence_after();
        if (lane == 0) {
          const uint32_t sa = sm100::smem_u32(smem + s * STAGE_BYTES);
          const uint64_t da = sm100::umma_desc_sw128(sa);
          const uint64_t db = sm100::umma_desc_sw128(sa + A_STAGE_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            sm100::mma_bf16_ss_2sm(tmem, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
          sm100::mma_commit_2sm_mc(&empty[s], 0x3);
          if (kb == nkb - 1) sm100::mma_commit_2sm_mc(done, 0x3);
        }
        __syncwarp();
      }
    }
  } else {
    // ---------------- warps 2-3: stage bias (and the width-1 layer) while the MMA runs
    for (int c = threadIdx.x - 64; c < BN; c += 64) {
      const int n = n0 + c;
      s_bias[c] = n < args.N ? __ldg(&args.bias[n]) : 0.f;
      if (args.mode == GEMM_OUT_CTR) s_wl[c] = n < args.N ? __ldg(&args.w_last[n]) : 0.f;
    }
  }

  // ---------------- epilogue: thread = row (TMEM lane warp*32 + lane)
  sm100::mbar_wait(done, 0);
  __syncthreads();  // s_bias / s_wl visible to every epilogue thread
  sm100::tc_fence_after();
#pragma unroll 1
  for (int h = 0; h < MT; ++h) {
  const int row = m0 + h * BM + warp * 32 + lane;
  const bool row_ok = row < M;
  const uint32_t trow = tmem + (static_cast<uint32_t>(warp * 32) << 16) + h * BN;
  float dot = 0.f;
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += 16) {
    const int cbase = n0 + c0;
    if (cbase >= args.N) break;  // warp-uniform
    uint32_t r[16];
    sm100::tmem_ld_32x32b_x16(trow + c0, r);
    sm100::tmem_ld_wait();
    float v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      float x = __uint_as_float(r[j]) + s_bias[c0 + j];
      if (args.relu) x = fmaxf(x, 0.f);
      v[j] = x;
    }
    if (!row_ok) continue;
    if (args.mode == GEMM_OUT_BF16) {
      __nv_bfloat16* dst = args.out_bf16 + static_cast<int64_t>(row) * args.ldo + cbase;
      if (cbase + 16 <= args.N) {
        uint32_t p[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
          p[j] = *reinterpret_cast<uint32_t*>(&h);
        }
        uint4* d4 = reinterpret_cast<uint4*>(dst);
        d4[0] = make_uint4(p[0], p[1], p[2], p[3]);
        d4[1] = make_uint4(p[4], p[5], p[6], p[7]);
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (cbase + j < args.N) dst[j] = __float2bfloat16_rn(v[j]);
      }
    } else if (args.mode == GEMM_OUT_X_F32) {
      float* dst = args.out_f32 + static_cast<int64_t>(row) * args.ldo + cbase;
      if (cbase + 16 <= args.N) {
        float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
        for (int j = 0; j < 4; ++j) d4[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (cbase + j < args.N) dst[j] = v[j];
      }
    } else {  // GEMM_OUT_CTR: width-1 output layer folded into the epilogue
#pragma unroll
      for (int j = 0; j < 16; ++j) dot = fmaf(v[j], s_wl[c0 + j], dot);
    }
  }
  if (args.mode == GEMM_OUT_CTR && row_ok) {
    float logit = dot + args.b_last;
    if (args.logit_add) logit += args.logit_add[static_cast<int64_t>(row) * args.add_stride];
    const int64_t o = static_cast<int64_t>(row) * (args.ctr_stride > 0 ? args.ctr_stride : 1);
    args.ctr[o] = 1.f / (1.f + __expf(-logit));
    if (args.logit) args.logit[o] = logit;
  }
  }
  sm100::tc_fence_before();
  sm100::cluster_sync();
  if (warp == 0) sm100::tmem_dealloc_2sm(tmem, TMEM_COLS);
}


template <int BN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    k_gemm_2sm(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_w,
               const __grid_constant__ GemmArgs args, int stages) {
  gemm_tile_2sm<BN>(&tmap_a, &tmap_w, args, stages);
}

// tmap_w must have a BN/2-row box (Layer::tmap_w128 for BN = 256).
template <int BN>
static void launch_2sm(const CUtensorMap* ta, const CUtensorMap* tw, const GemmArgs& a, cudaStream_t s,
                       int ring = 0) {
  constexpr int STAGE = A_STAGE_BYTES + (BN / 2) * BK * 2;
  const int nkb = (a.K + BK - 1) / BK;
  const int smax = ring > 0 ? ring : g_gemm_2sm > 1 ? g_gemm_2sm : 4;  // REC_GEMM_2SM=n > 1: n-stage ring
  const int stages = nkb < smax ? (nkb < 1 ? 1 : nkb) : smax;
  const size_t smem = static_cast<size_t>(stages) * STAGE + 1024 + 256;
  int mblocks = (a.M + BM - 1) / BM;
  mblocks += mblocks & 1;  // whole pairs
  k_gemm_2sm<BN><<<dim3(2, (a.N + BN - 1) / BN, mblocks / 2), 128, smem, s>>>(*ta, *tw, a, stages);
}

// Ring depth: a launch with fewer CTAs than SMs is a serving-batch GEMM that co-runs with the
// other co-located streams' kernels; its shared memory is carved out of those SMs' L1, so it
// keeps a 2-stage ring (measured: MT-WnD towers 486k -> 611k QPS, same launch latency); a
// launch that fills the GPU (large batches) takes the deep ring the tensor pipe needs.
// REC_GEMM_STAGES overrides.
static int ring_depth(int smax, int ctas) {
  if (g_gemm_stages > 0) return g_gemm_stages < smax ? g_gemm_stages : smax;
  return ctas < 148 ? (smax < 2 ? smax : 2) : smax;
}

template <int BN, int MT>
__global__ void __launch_bounds__(128, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_w,
              const __grid_constant__ GemmArgs args, int stages) {
  gemm_tile<BN, MT>(&tmap_a, &tmap_w, args, stages);
}

// Grouped launch: blockIdx.z selects one of g.n GEMMs of identical shape (MT-WnD: the same
// layer of every task tower), each with its own A / W tensor maps and epilogue arguments.
template <int BN, int MT>
__global__ void __launch_bounds__(128, 1) k_gemm_group(const __grid_constant__ GemmGroup g, int stages) {
  // 128-wide tiles read the 128-row-box weight maps (a 256-wide tile needs the full box)
  gemm_tile<BN, MT>(&g.ta[blockIdx.z], BN == 128 && g.a[0].N > 128 ? &g.tw_half[blockIdx.z] : &g.tw[blockIdx.z],
                    g.a[blockIdx.z], stages);
}

template <int BN, int MT>
static void launch_group_bn(const GemmGroup& g, cudaStream_t s) {
  constexpr int STAGE = MT * A_STAGE_BYTES + BN * BK * 2;
  constexpr int SMAX = (MT == 1 ? 4 : 3);
  const GemmArgs& a = g.a[0];
  const int nkb = (a.K + BK - 1) / BK;
  const int ctas = ((a.N + BN - 1) / BN) * ((a.M + BM * MT - 1) / (BM * MT)) * g.n;
  const int smax = ring_depth(SMAX, ctas);
  const int stages = nkb < smax ? (nkb < 1 ? 1 : nkb) : smax;
  const size_t smem = static_cast<size_t>(stages) * STAGE + 1024 + 256;
  dim3 grid((a.N + BN - 1) / BN, (a.M + BM * MT - 1) / (BM * MT), g.n);
  k_gemm_group<BN, MT><<<grid, 128, smem, s>>>(g, stages);
}

template <int BN, int MT>
static void launch_bn(const CUtensorMap* ta, const CUtensorMap* tw, const GemmArgs& a,
                      cudaStream_t s, bool deep = false) {
  constexpr int STAGE = MT * A_STAGE_BYTES + BN * BK * 2;
  constexpr int SMAX = (MT == 1 ? 4 : 3);
  const int nkb = (a.K + BK - 1) / BK;
  const int smax = deep && g_gemm_stages == 0
                       ? SMAX
                       : ring_depth(SMAX, ((a.N + BN - 1) / BN) * ((a.M + BM * MT - 1) / (BM * MT)));
  const int stages = nkb < smax ? (nkb < 1 ? 1 : nkb) : smax;
  const size_t smem = static_cast<size_t>(stages) * STAGE + 1024 + 256;
  dim3 grid((a.N + BN - 1) / BN, (a.M + BM * MT - 1) / (BM * MT));
  k_gemm_tc<BN, MT><<<grid, 128, smem, s>>>(*ta, *tw, a, stages);
}

int gemm_bn(int N) { return N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256; }

template <int BN, int MT>
static void prep_bn() {
  constexpr int STAGE = MT * A_STAGE_BYTES + BN * BK * 2;
  constexpr int SMAX = (MT == 1 ? 4 : 3);
  cudaFuncSetAttribute(k_gemm_tc<BN, MT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       SMAX * STAGE + 1024 + 256);
  cudaFuncSetAttribute(k_gemm_group<BN, MT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       SMAX * STAGE + 1024 + 256);
}

void gemm_prepare() {
  cudaFuncSetAttribute(k_gemm_2sm<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       6 * (A_STAGE_BYTES + 128 * BK * 2) + 1024 + 256);
  prep_bn<32, 1>();
  prep_bn<64, 1>();
  prep_bn<128, 1>();
  prep_bn<256, 1>();
  prep_bn<256, 2>();
}

int g_gemm_2sm = 0;     // REC_GEMM_2SM: CTA-pair GEMM for full-GPU launches (experimental)
int g_gemm_2sm_serve = 0;  // REC_GEMM_2SM_SERVE=n: CTA-pair GEMM (n-stage ring) for serving launches (opt-in, see DESIGN)
int g_gemm_mt1 = 0;     // REC_GEMM_MT1=1: 128x256 tiles (one M tile per CTA) for full-GPU launches too (A/B)
int g_gemm_narrow = 0;  // REC_GEMM_NARROW=n: 128-wide N tiles below n 128x256 tiles (measured: RMC2/3 +0.5-1 %, MT-WnD -7 %)
int g_gemm_mt2 = 0;     // REC_GEMM_MT2=1: 256 x 256 weight-sharing tiles also for serving batches
int g_gemm_bn64 = 0;    // REC_GEMM_BN64=1: 64-wide serving tiles (below; measured: RMC3 -4 % at 16
                        // co-located streams, -11 % at 32, RMC2 +2 %: off by default)

void launch_gemm_tc(const CUtensorMap* tmap_a, const CUtensorMap* tmap_w, const GemmArgs& a,
                    cudaStream_t s, const CUtensorMap* tmap_w_half, const CUtensorMap* tmap_w64) {
  if (a.M <= 0) return;
  // Serving-batch launch of a wide, deep layer (e.g. RMC3's 2560 -> 512 at B <= 1024): with
  // 128 x 256 tiles it runs 16 CTAs whose 2-stage rings keep ~1.5 MB in flight, so the layer
  // is bound by bytes in flight x L2 latency (~25 us).  64-wide N tiles give 4x the CTAs and,
  // at the same shared memory per CTA (4 stages x 24 KB), twice the k-blocks in flight each.
  // (Measured: the single-stream GEMM time of an RMC3 batch drops 70 -> 65 us, but the extra
  // CTAs and deeper rings cost the co-running kernels more, see g_gemm_bn64.)
  // Every output element still accumulates over K in the same order, so the bits do not
  // depend on the tiling (batch invariance; tests/test_gpu_variants.py).  The width-1 CTR
  // epilogue needs whole rows, so CTR layers keep their tiles.
  const int m_tiles = (a.M + BM - 1) / BM;
  if (g_gemm_bn64 && tmap_w64 && a.mode != GEMM_OUT_CTR && a.N >= 128 && a.K >= 512 &&
      m_tiles * ((a.N + 255) / 256) < 74 && m_tiles * ((a.N + 63) / 64) <= 148) {
    launch_bn<64, 1>(tmap_a, tmap_w64, a, s, true);
    return;
  }
  if (a.N <= 32) launch_bn<32, 1>(tmap_a, tmap_w, a, s);
  else if (a.N <= 64) launch_bn<64, 1>(tmap_a, tmap_w, a, s);
  else if (a.N <= 128) launch_bn<128, 1>(tmap_a, tmap_w, a, s);
  else if ((((a.M + 255) / 256) * ((a.N + 255) / 256) >= 148 || g_gemm_mt2) && a.K >= 512) {
    if (g_gemm_2sm && tmap_w_half) launch_2sm<256>(tmap_a, tmap_w_half, a, s);  // CTA pairs
    else if (g_gemm_mt1) launch_bn<256, 1>(tmap_a, tmap_w, a, s);
    else launch_bn<256, 2>(tmap_a, tmap_w, a, s);  // enough 256-row tiles to fill the GPU: share W
  } else if (g_gemm_2sm_serve && tmap_w_half && a.K >= 512) {
    // serving batch on CTA pairs: each CTA of a pair loads its own 128 A rows and half of the
    // 256-wide W tile, the pair's MMA reads both halves (1.5 x the flops per delivered byte)
    launch_2sm<256>(tmap_a, tmap_w_half, a, s, g_gemm_2sm_serve);
  } else if (g_gemm_narrow && tmap_w_half && a.mode != GEMM_OUT_CTR &&
             ((a.M + 127) / 128) * ((a.N + 255) / 256) < g_gemm_narrow) {
    // serving batch, few 128x256 tiles: 128-wide N tiles double the CTAs working on the layer
    // (lower latency; every output element keeps the same K-ordered accumulation, so the
    // result bits do not depend on the tiling)
    launch_bn<128, 1>(tmap_a, tmap_w_half, a, s);
  } else {
    launch_bn<256, 1>(tmap_a, tmap_w, a, s);
  }
}

void launch_gemm_group(const GemmGroup& g, cudaStream_t s) {
  const GemmArgs& a = g.a[0];
  if (a.M <= 0 || g.n <= 0) return;
  if (a.N <= 32) launch_group_bn<32, 1>(g, s);
  else if (a.N <= 64) launch_group_bn<64, 1>(g, s);
  else if (a.N <= 128) launch_group_bn<128, 1>(g, s);
  else if (((a.M + 255) / 256) * ((a.N + 255) / 256) * g.n >= 148 && a.K >= 512)
    launch_group_bn<256, 2>(g, s);
  else if (g_gemm_narrow && a.mode != GEMM_OUT_CTR &&  // the CTR epilogue needs the whole row
           ((a.M + 127) / 128) * ((a.N + 255) / 256) * g.n < g_gemm_narrow)
    launch_group_bn<128, 1>(g, s);
  else launch_group_bn<256, 1>(g, s);
}

// ---------------------------------------------------------------- tensor maps
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

bool encode_tmap_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t K, uint64_t ldk,
                      uint32_t box_rows) {
  auto fn = get_encode();
  if (!fn) return false;
  cuuint64_t dims[2] = {K, rows};
  cuuint64_t strides[1] = {ldk * 2};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(BK), box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Row-gather map over an fp32 row arena: dims {width, rows}, box {width, 1} (TMA gather4
// fetches 4 arbitrary rows of `width` floats per instruction).
bool encode_tmap_rows_f32(CUtensorMap* map, const void* base, uint64_t rows, uint32_t width) {
  auto fn = get_encode();
  if (!fn || width > 256 || (width * 4) % 16 != 0) return false;
  cuuint64_t dims[2] = {width, rows};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(width) * 4};
  cuuint32_t box[2] = {width, 1};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace rec
