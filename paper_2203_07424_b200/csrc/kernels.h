// kernels.h — host-side launchers of the sm_100a kernels (one translation unit each).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace rec {

// ---------------------------------------------------------------- parameters (G4, G5)
void launch_init_table(float* base, int64_t rows, int D, int64_t stride, int t, uint32_t k0,
                       uint32_t k1, int shift, int value_mode, cudaStream_t s);
void launch_init_layer(__nv_bfloat16* W, float* bias, int N, int K, int Kpad, int layer,
                       int e, uint32_t k0, uint32_t k1, cudaStream_t s);
void launch_init_final(float* w, float* b, int K, int layer, int e, uint32_t k0, uint32_t k1,
                       cudaStream_t s);

// ------------------------------------------------------------ batch inputs (G2, G3)
// segs4[nseg] = (qid, start, len, first_row)
// hdr = {B, nseg, 0, 0} then segments (device); rows for the capacity grid `cap`
void launch_expand_rows(const int4* hdr, int cap, int* rowq, int* rowi, cudaStream_t s);
void launch_gen_offsets(const int* rowq, const int* rowi, const int* dB, int T, int lo, int hi,
                        uint32_t k0, uint32_t k1, int* offsets, cudaStream_t s);
void launch_gen_indices(const int* rowq, const int* rowi, const int* offsets, int cap, const int* dB,
                        int T, const int64_t* rows, int index_dist, uint32_t k0, uint32_t k1,
                        int* indices, cudaStream_t s);
void launch_gen_dense(const int* rowq, const int* rowi, int cap, const int* dB, int F, int Fpad,
                      uint32_t k0, uint32_t k1, __nv_bfloat16* dense_bf, float* dense_f32,
                      cudaStream_t s);
void launch_dense_to_bf16(const float* dense, int B, int F, int Fpad, __nv_bfloat16* out,
                          cudaStream_t s);
void launch_check_offsets(const int* offsets, int nbags, int* flag, cudaStream_t s);

// ------------------------------------------------------------------------- SLS (a3)
// Row r of table t lives at tables + tab_off[t] + r * row_stride (floats).
// B: batch (or capacity when dB != nullptr: then the kernels read the batch from *dB,
// which lets one captured CUDA graph serve every batch size).
void launch_sls(const float* tables, const int64_t* tab_off, int64_t row_stride,
                const int64_t* rows, const int* indices, const int* offsets, int B, const int* dB,
                int T, int D, float* X, int x_stride_items, int x_slot0, int* flag, cudaStream_t s);

// ----------------------------------------------------------- tcgen05 GEMM (a4, a6)
enum GemmMode : int { GEMM_OUT_BF16 = 0, GEMM_OUT_X_F32 = 1, GEMM_OUT_CTR = 2 };
struct GemmArgs {
  int M, N, K;              // A [M][K] (bf16, K-major via tmap_a), W [N][K] (tmap_w)
  const int* dM;            // optional device-side M (grid sized for M = capacity)
  const float* bias;        // [N]
  int relu;                 // apply ReLU after bias
  int mode;                 // GemmMode
  __nv_bfloat16* out_bf16;  // mode 0: [M][ldo]
  int ldo;
  float* out_f32;           // mode 1: X base; row r col c -> out_f32[r*ldo + c]
  const float* w_last;      // mode 2: [N] final width-1 layer
  float b_last;
  float* ctr;               // mode 2: [M]
  float* logit;             // mode 2: [M] optional
};
int gemm_bn(int N);                  // tile width used for a layer of width N (W tmap box)
void gemm_prepare();                 // per-device one-time kernel attributes
void launch_gemm_tc(const CUtensorMap* tmap_a, const CUtensorMap* tmap_w, const GemmArgs& a,
                    cudaStream_t s);
// Encode a 2D bf16 K-major tensor map [rows][K] (row pitch ldk elements) with a
// 64 x box_rows box and 128-byte swizzle.  Returns false on failure.
bool encode_tmap_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t K,
                      uint64_t ldk, uint32_t box_rows);

// --------------------------------------------------------------- interaction (a5)
void launch_interact(const float* X, int B, const int* dB, int T, int D, __nv_bfloat16* A_top,
                     int ld_top, cudaStream_t s);

// Fused synthetic inputs for FIXED pooling: hdr = {B, nseg, 0, 0} followed by nseg segments
// (qid, start, len, first_row) in device memory; writes offsets (g*L), indices and dense
// (bf16 padded, optional fp32).  cap = grid capacity in items.
void launch_gen_fused(const int4* hdr, int cap, int T, int L, const int64_t* rows, int index_dist,
                      int F, int Fpad, uint32_t k0, uint32_t k1, int* offsets, int* indices,
                      __nv_bfloat16* dense_bf, float* dense_f32, cudaStream_t s);

}  // namespace rec
