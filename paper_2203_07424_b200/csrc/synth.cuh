// synth.cuh — device-side synthetic values shared by the input generator and the fused
// synthetic-index SLS (G2-G4).  Bit-identical to oracle/gen.py (separate code).
#pragma once
#include "common.cuh"
#include "kernels.h"

namespace rec {

__device__ __forceinline__ float pow2f(int e) {  // exact 2^e for e in [-126, 127]
  return __int_as_float((127 + e) << 23);
}
__device__ __forceinline__ float i8(uint32_t w) {
  return static_cast<float>(static_cast<int>(static_cast<int8_t>(w & 0xFFu)));
}

// ------------------------------------------------------------ batch rows (q, item)
__device__ __forceinline__ int2 row_item(const SegBatch& sb, int b) {
  const int4* segs = sb.nseg > kParamSegs ? sb.gsegs : sb.seg;
  int lo = 0, hi = sb.nseg - 1;  // last segment with first_row <= b
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (segs[mid].w <= b) lo = mid; else hi = mid - 1;
  }
  const int4 sg = segs[lo];
  return make_int2(sg.x, sg.y + (b - sg.w));
}

// ------------------------------------------------------------ Zipf(0.9) rows (G2z)
// Continuous inverse CDF of Zipf(0.9) from exactly rounded fp64 operations only (__dmul_rn /
// __dadd_rn are never contracted into FMAs), so the rows are bit-identical to oracle/gen.py:
// c = largest double with (c^10) <= R (60 bisection steps), x = 1 + u (c - 1), y = x^10,
// rank = min(floor(y) - 1, R - 1), row = (rank * 2654435761 + 7919 t) mod R.
__device__ __forceinline__ double pow10_rn(double x) {
  const double x2 = __dmul_rn(x, x), x4 = __dmul_rn(x2, x2), x8 = __dmul_rn(x4, x4);
  return __dmul_rn(x8, x2);
}
__device__ inline double zipf_c(uint64_t R) {
  double lo = 1.0, hi = 16.0;
  const double Rd = static_cast<double>(R);
  for (int i = 0; i < 60; ++i) {
    const double mid = __dmul_rn(__dadd_rn(lo, hi), 0.5);
    if (pow10_rn(mid) <= Rd) lo = mid;
    else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ int zipf_row(uint64_t r, uint64_t R, double zc, uint32_t t) {
  const double u = __dmul_rn(static_cast<double>(r >> 11), 0x1p-53);
  const double x = __dadd_rn(1.0, __dmul_rn(u, __dadd_rn(zc, -1.0)));
  uint64_t rank = static_cast<uint64_t>(floor(pow10_rn(x))) - 1;  // x >= 1: floor >= 1
  if (rank > R - 1) rank = R - 1;
  return static_cast<int>((rank * 2654435761ull + 7919ull * t) % R);
}

// ---------------------------------------------------------------------- indices (G2)
// zc: zipf_c(R) of the table (index_dist 3 only; computed once per thread by the caller).
__device__ __forceinline__ int gen_index(uint32_t j, uint32_t it, uint32_t c2, uint32_t q,
                                         uint32_t k0, uint32_t k1, uint64_t R, int index_dist,
                                         double zc = 0.0) {
  const U4 w = philox(j, it, c2, q, k0, k1);
  uint64_t r = (static_cast<uint64_t>(w.y) << 32) | w.x;
  if (index_dist == 3) return zipf_row(r, R, zc, c2 >> 8);
  if (index_dist == 2) r = __umul64hi(r, (static_cast<uint64_t>(w.w) << 32) | w.z);
  return static_cast<int>(__umul64hi(r, R));
}

// Dense features (G4, round 2): feature f of (q, item) is byte f mod 16 of the 16-byte
// little-endian output (w0, w1, w2, w3) of philox((f / 16, item, 3, q)), as int8 * 2^-7 — one
// Philox evaluation per 16 features (RMC3's 2560 features per item cost one Philox each in
// round 1, as much ALU as the whole SLS).  gen_dense16 returns the 16 values of block blk.
__device__ __forceinline__ void gen_dense16(uint32_t blk, uint32_t it, uint32_t q, uint32_t k0,
                                            uint32_t k1, float v[16]) {
  const U4 w = philox(blk, it, DOM_DENSE, q, k0, k1);
  const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = i8(ws[j >> 2] >> (8 * (j & 3))) * pow2f(-7);
}
__device__ __forceinline__ float gen_dense(uint32_t f, uint32_t it, uint32_t q, uint32_t k0,
                                           uint32_t k1) {
  const U4 w = philox(f >> 4, it, DOM_DENSE, q, k0, k1);
  const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
  const int j = static_cast<int>(f & 15);
  return i8(ws[j >> 2] >> (8 * (j & 3))) * pow2f(-7);
}
// Row b of bf16 [.][Fpad] (and optionally fp32 [.][F]) for (q, item): lanes `lane`, `lane +
// nl`, ... of a group of nl threads each own 16-feature blocks.
__device__ __forceinline__ void gen_dense_row(uint32_t it, uint32_t q, uint32_t k0, uint32_t k1, int F,
                                              int Fpad, __nv_bfloat16* __restrict__ bf,
                                              float* __restrict__ f32, int lane, int nl) {
  const int nblk = (Fpad + 15) / 16;
  for (int blk = lane; blk < nblk; blk += nl) {  // (no blk * 16 in the bound: nl may be huge)
    float v[16];
    gen_dense16(static_cast<uint32_t>(blk), it, q, k0, k1, v);
    const int f0 = blk * 16;
    if (f0 + 16 <= F && f0 + 16 <= Fpad) {
      // whole block: two 16-byte stores (bf rows start 16-byte aligned: Fpad % 8 == 0), so a
      // warp writes contiguous 512-byte runs instead of 2-byte scalars at a 32-byte stride
      uint32_t p[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
        p[j] = *reinterpret_cast<uint32_t*>(&h);
      }
      uint4* d = reinterpret_cast<uint4*>(bf + f0);
      d[0] = make_uint4(p[0], p[1], p[2], p[3]);
      d[1] = make_uint4(p[4], p[5], p[6], p[7]);
      if (f32) {
        float4* o = reinterpret_cast<float4*>(f32 + f0);  // (rec_gen_batch only; F % 4 alignment
#pragma unroll                                          //  not guaranteed -> scalar below if not)
        for (int j = 0; j < 4; ++j)
          if ((reinterpret_cast<uintptr_t>(o) & 15) == 0) o[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          else for (int k = 0; k < 4; ++k) f32[f0 + 4 * j + k] = v[4 * j + k];
      }
      continue;
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int f = f0 + j;
      if (f >= Fpad) break;
      const float x = f < F ? v[j] : 0.f;
      bf[f] = __float2bfloat16_rn(x);
      if (f32 && f < F) f32[f] = x;
    }
  }
}

}  // namespace rec
