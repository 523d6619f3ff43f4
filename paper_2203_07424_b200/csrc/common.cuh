// common.cuh — shared device helpers of the CUDA path (NOT shared with the oracle).
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace rec {

// Philox4x32-10 (Salmon et al., SC'11), G1.  Key bumped before rounds 2..10.
struct U4 {
  uint32_t x, y, z, w;
};
__device__ __forceinline__ U4 philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                     uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  return U4{c0, c1, c2, c3};
}

__device__ __forceinline__ float int8_scaled(uint32_t w, int e) {
  // int8(low byte) * 2^e, exact in fp32 and bf16
  const int v = static_cast<int>(static_cast<int8_t>(w & 0xFFu));
  return ldexpf(static_cast<float>(v), e);
}

// Domains of the synthetic-value counters (G2-G5).
enum : uint32_t { DOM_INDEX = 1, DOM_LEN = 2, DOM_DENSE = 3, DOM_TABLE = 4, DOM_W = 5, DOM_B = 6 };
constexpr int TOP_LAYER_BASE = 64;

}  // namespace rec
