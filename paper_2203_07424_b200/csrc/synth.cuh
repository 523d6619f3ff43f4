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

// ---------------------------------------------------------------------- indices (G2)
__device__ __forceinline__ int gen_index(uint32_t j, uint32_t it, uint32_t c2, uint32_t q,
                                         uint32_t k0, uint32_t k1, uint64_t R, int index_dist) {
  const U4 w = philox(j, it, c2, q, k0, k1);
  uint64_t r = (static_cast<uint64_t>(w.y) << 32) | w.x;
  if (index_dist == 2) r = __umul64hi(r, (static_cast<uint64_t>(w.w) << 32) | w.z);
  return static_cast<int>(__umul64hi(r, R));
}

__device__ __forceinline__ float gen_dense(uint32_t f, uint32_t it, uint32_t q, uint32_t k0,
                                           uint32_t k1) {
  return i8(philox(f, it, DOM_DENSE, q, k0, k1).x) * pow2f(-7);
}

}  // namespace rec
