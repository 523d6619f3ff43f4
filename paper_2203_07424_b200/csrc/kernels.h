// kernels.h — host-side launchers of the sm_100a kernels (one translation unit each).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace rec {

// ---------------------------------------------------------------- parameters (G4, G5)
// rows [r0, r0 + rows) of table t (global Philox counters) into base[(r - r0) * stride + k]
void launch_init_table(float* base, int64_t rows, int D, int64_t stride, int t, uint32_t k0,
                       uint32_t k1, int shift, int value_mode, cudaStream_t s, int64_t r0 = 0);
void launch_init_layer(__nv_bfloat16* W, float* bias, int N, int K, int Kpad, int layer,
                       int e, uint32_t k0, uint32_t k1, cudaStream_t s);
void launch_init_final(float* w, float* b, int K, int layer, int e, uint32_t k0, uint32_t k1,
                       cudaStream_t s);

// ------------------------------------------------------------ batch inputs (G2, G3)
// A fused batch as segments (qid, start, len, first_row).  Passed BY VALUE as a
// __grid_constant__ kernel parameter, so a captured CUDA graph is re-pointed at a new batch
// with one kernel-node parameter update (no host->device copy per batch).  Batches with more
// than kParamSegs segments read them from `gsegs` (device memory) instead.
constexpr int kParamSegs = 120;
struct SegBatch {
  int B, nseg;
  const int4* gsegs;
  int4 seg[kParamSegs];
};
struct GenArgs {
  int cap, T, lo, hi, index_dist, F, Fpad, nbag_blocks;
  uint32_t k0, k1;
  const int64_t* rows;
  int* offsets;
  int* indices;
  __nv_bfloat16* dense_bf;
  float* dense_f32;  // optional fp32 copy (rec_gen_batch)
  int* rowq;         // variable pooling path
  int* rowi;
  int* dB;           // device batch size, written by the first input kernel
};
// The first kernel of the input chain (fused fixed-pooling generator, or row expansion for
// variable pooling).  Both take (SegBatch, GenArgs) so graph updates are uniform.
void* gen_first_kernel(const GenArgs& ga, dim3* grid, dim3* block);
void launch_gen_first(const SegBatch& sb, const GenArgs& ga, cudaStream_t s);
// Fixed pooling, fused path: dense features only (indices are generated inside the SLS).
void* gen_dense_seg_kernel(const GenArgs& ga, dim3* grid, dim3* block);
void launch_gen_dense_seg(const SegBatch& sb, const GenArgs& ga, cudaStream_t s);
// Variable pooling only (after launch_gen_first): lengths + scan, indices, dense.
void launch_gen_variable_rest(const GenArgs& ga, cudaStream_t s);
void launch_dense_to_bf16(const float* dense, int B, int F, int Fpad, __nv_bfloat16* out,
                          cudaStream_t s);
// Flags bit 1 when offsets[0] != 0, offsets decrease, or (nnz >= 0) offsets[nbags] != nnz.
void launch_check_offsets(const int* offsets, int nbags, int* flag, cudaStream_t s, int64_t nnz = -1);
// Hot-row partition (rec_hot_remap): out[i] = remap[remap_off[t] + in[i]] for every index of
// the table-major CSR batch (t from the offsets); indices outside [0, rows_t) set flag bit 0
// and map to 0; positions >= cap are not written (flag bit 1).  B from *dB when dB != nullptr.
void launch_remap(const int* in, const int* offsets, int B, const int* dB, int T, const int64_t* rows,
                  const int* remap, const int64_t* remap_off, int* out, int64_t cap, int* flag,
                  cudaStream_t s);
// Arena row permutation: new arena row p of table t = old row inv[remap_off[t] + p] (interleaved
// or table-major arena: row r of table t at tab_off[t] + r * row_stride).
void launch_permute_rows(const float* src, float* dst, const int64_t* tab_off, int64_t row_stride,
                         const int64_t* rows, int T, int D, const int* inv, const int64_t* remap_off,
                         int64_t max_rows, cudaStream_t s);
void set_max_smem_carveout(int percent);  // SLS kernels' preferred shared-memory carveout (0..100)

// ------------------------------------------------------------------------- SLS (a3)
// Row r of table t lives at tables + tab_off[t] + r * row_stride (floats).
// B: batch (or capacity when dB != nullptr: then the kernels read the batch from *dB,
// which lets one captured CUDA graph serve every batch size).
// Table-wise sharding with the all-to-all fused into the SLS (dist.cu): the
// pooled vector of bag (t, b) is stored straight into the X buffer of the rank that owns item
// b (peer memory over NVLink, CUDA IPC mappings), then the grid's last CTA raises this rank's
// arrival flag on every peer (system-scope release).
struct P2PArgs {
  float* const* peer_X;         // [G] device array: every rank's X (table-wise) or partial-sum
                                // staging [G][Bq][T][D] (row-wise); own rank: local buffer
  int row_off;                  // destination row offset: 0 (table-wise) or rank * Bq (row-wise)
  unsigned* const* peer_flags;  // [G] device array: every rank's arrival-flag array [G]
  unsigned* counter;            // CTA completion counter of this launch (zeroed before it)
  unsigned* my_flags;           // this rank's arrival flags [G] (written by the peers)
  int Bq, G, rank;              // items per rank block, world size, this rank
  unsigned epoch;               // query sequence number (flags reach it when the data landed)
  int* err_flag;                // k_p2p_wait: bit 2 (value 4) set when a peer missed the timeout
  unsigned long long timeout_ns;  // k_p2p_wait bound (REC_P2P_TIMEOUT_S, default 60 s)
  // Async slot exchange (captured graphs): [0] epoch, [1] global batch B of the batch in
  // flight on this slot, written by the slot's SLS kernel; when non-null the later kernels of
  // the chain (wait, CTR scatter) read epoch / B from here instead of the fields above.
  unsigned* words;
  int sc_fence;  // 1: fence.sc.sys + relaxed atomic per CTA; 0: one acq_rel.sys atomic per CTA
  // Flag-in-data exchange (k_sls_synth, REC_P2P_LL, default on): pooled vectors of items owned
  // by another rank go to that rank's LL buffer as 16-byte stores {v0, epoch, v1, epoch}
  // (8-byte halves land atomically over NVLink), so no CTA waits on a system-scope fence; the
  // owner's k_p2p_ll_unpack validates every half's epoch and writes X.  The flags raised by
  // the last CTA are then only a hint that the data is (mostly) in flight or landed.
  // Layout per rank: [ceil(cap / G)][T][D / 4][2] uint4, item row bi, global table tg.
  uint4* const* peer_ll;  // [G] every rank's LL buffer of this slot
  int ll;                 // 1: LL stores for remote items (own items go straight into X)
  int T_all;              // global table count (LL row pitch)
};
void launch_sls_p2p(const float* tables, const int64_t* tab_off, int64_t row_stride,
                    const int64_t* rows, const int* indices, const int* offsets, int B, int T, int D,
                    int x_stride_items, int x_slot0, int* flag, const P2PArgs& p2p, cudaStream_t s,
                    int row_lo = 0, int row_hi = 0x7fffffff, int idx_limit = 0x7fffffff);
// Row-wise: X[i][1 + t] = sum over source ranks q (in order) of stage[q][i][t] for i < Bl.
void launch_p2p_reduce(const float* stage, float* X, int Bl, int Bq, int T, int D, int G,
                       cudaStream_t s);
// Block the stream until every rank's SLS of this epoch has landed in this rank's X.
void launch_p2p_wait(const P2PArgs& p2p, cudaStream_t s);
// LL exchange: X[bi][1 + tg] of this rank's item block for every table tg outside the own
// range [t0, t0 + TL), read from this rank's LL buffer `ll` once both epoch words of each
// 16-byte line equal the slot epoch (p2p.words[0]; batch p2p.words[1]).  Bounded spin: a line
// that misses p2p.timeout_ns sets bit 2 of p2p.err_flag.  Grid: nsm x 2 CTAs (grid-stride).
void launch_p2p_ll_unpack(const P2PArgs& p2p, const uint4* ll, float* X, int T, int D, int t0, int TL,
                          int nsm, cudaStream_t s);
// All-gather of the CTRs over peer memory: this rank's ctr[0..Bl) goes to every rank's
// gather buffer at [item0, item0 + Bl), then this rank's flag is raised on every peer
// (p2p.peer_X = the ranks' gather buffers, p2p.peer_flags = their CTR-flag arrays).
void launch_p2p_ctr_scatter(const float* ctr, int Bl, int item0, const P2PArgs& p2p, cudaStream_t s);

// row_lo/row_hi: row-wise sharding keeps rows [row_lo, row_hi) of every table on this GPU
// (arena row r - row_lo); other rows add nothing.  Replicated / table-wise: 0, INT32_MAX.
// idx_limit: number of readable entries of `indices`; offsets are clamped to [0, idx_limit]
// so inconsistent caller offsets (flagged separately) never read past the array.
void launch_sls(const float* tables, const int64_t* tab_off, int64_t row_stride,
                const int64_t* rows, const int* indices, const int* offsets, int B, const int* dB,
                int T, int D, float* X, int x_stride_items, int x_slot0, int* flag, cudaStream_t s,
                int row_lo = 0, int row_hi = 0x7fffffff, int idx_limit = 0x7fffffff);

// SLS over device-synthesised indices (fixed pooling L): each index is the Philox value of
// (slot, item, table, qid) computed where it is consumed (a2 fused into a3): no index array,
// no dependency on an input kernel.  Writes X slots 1..T and *dB = batch.
struct SlsSynthArgs {
  const float* tables;
  const int64_t* tab_off;
  int64_t row_stride;
  const int64_t* rows;
  int cap, T, D, L, index_dist;
  uint32_t k0, k1;
  float* X;
  int x_stride;
  int* dB;
  // hot-row residency: rows r < hot_rows of every table are loaded with an L2 evict_last
  // policy, all others evict_first (0 = plain loads); the interleaved arena makes these rows
  // one contiguous prefix of hot_rows * T * D * 4 bytes
  int hot_rows;
  // optional fused dense-feature generation (a2 for the bottom MLP): bf16 [cap][Fpad] rows,
  // written by the table-0 bag groups at the end of the kernel (nullptr: not fused)
  __nv_bfloat16* dense_bf;
  int F, Fpad;
  // TMA row-gather variant (REC_SLS=tma): map over the arena as [rows_total][D] fp32 rows
  // (device copy, 64-B aligned), arena row of (t, r) = tab_off[t] / D + r * row_stride / D.
  const CUtensorMap* tmap_rows;
  int pdl;        // launch with programmatic stream serialization (kernel waits before writes)
  // table-wise sharded serving (dist.cu): local tables are global tables t0 .. t0 + T - 1
  // (Philox counters use the global id); p2p.peer_X != nullptr stores every pooled vector into
  // the X of the rank owning the item (blocks of ceil(B / G)) and raises this rank's flags
  int t0;
  P2PArgs p2p;
  // hot-row partition (rec_hot_remap): synthesised row r of table t is stored at arena row
  // remap[remap_off[t] + r] (rows sorted by profiled frequency); nullptr = identity
  const int* remap;
  const int64_t* remap_off;
  int tma;     // 1: k_sls_synth_tma
  int nsm;     // SMs (persistent grid)
  int interleave;  // bags dealt round-robin over one wave of nsm x resident CTAs (k_sls_synth)
  int nst;     // ring chunks per warp
};
// Returns the kernel for this configuration; grid / block / dynamic smem are written back.
void* sls_synth_kernel(const SlsSynthArgs& a, dim3* grid, dim3* block, size_t* smem = nullptr);
bool sls_tma_supported(int D);
void sls_tma_configure(SlsSynthArgs& a);
void launch_sls_synth(const SegBatch& sb, const SlsSynthArgs& a, cudaStream_t s);

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
  float* ctr;               // mode 2: [M] (element r * ctr_stride)
  float* logit;             // mode 2: [M] optional (same stride)
  int ctr_stride;           // mode 2: 0 or 1 = dense; MT-WnD: n_tasks (item-major [M][N])
  const float* logit_add;   // mode 2: optional per-row addend (MT-WnD wide part) ...
  int add_stride;           // ... at logit_add[r * add_stride]
};
// Up to kMaxGroup GEMMs of one shape in ONE launch (grid.z = member): MT-WnD task towers.
constexpr int kMaxGroup = 4;
struct GemmGroup {
  CUtensorMap ta[kMaxGroup], tw[kMaxGroup];  // 64-B aligned members (CUtensorMap alignment)
  CUtensorMap tw_half[kMaxGroup];            // same weights, 128-row box (narrow N tiles)
  GemmArgs a[kMaxGroup];
  int n;
};
void launch_gemm_group(const GemmGroup& g, cudaStream_t s);
int gemm_bn(int N);                  // tile width used for a layer of width N (W tmap box)
void gemm_prepare();                 // per-device one-time kernel attributes
// tmap_w_half (optional): the same weights with a 128-row box, enabling the CTA-pair kernel.
// tmap_w64 (optional): 64-row box, enabling 64-wide N tiles for few-CTA serving launches.
void launch_gemm_tc(const CUtensorMap* tmap_a, const CUtensorMap* tmap_w, const GemmArgs& a,
                    cudaStream_t s, const CUtensorMap* tmap_w_half = nullptr,
                    const CUtensorMap* tmap_w64 = nullptr);
extern int g_gemm_2sm;
extern int g_gemm_2sm_serve;  // REC_GEMM_2SM_SERVE=n: CTA-pair GEMM for serving launches (n-stage ring)
extern int g_gemm_bn64;
extern int g_gemm_mt2;
extern int g_chain_persistent;  // REC_CHAIN_PERSISTENT (k_mlp.cu)
extern int g_gemm_narrow;
// Encode a 2D bf16 K-major tensor map [rows][K] (row pitch ldk elements) with a
// 64 x box_rows box and 128-byte swizzle.  Returns false on failure.
bool encode_tmap_rows_f32(CUtensorMap* map, const void* base, uint64_t rows, uint32_t width);
bool encode_tmap_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t K,
                      uint64_t ldk, uint32_t box_rows);

// ------------------------------------------- fused FC stack, one CTA per 128 rows (k_mlp.cu)
struct ChainMaps {
  CUtensorMap a0;  // layer-0 activations [M][K0] (box 64 x 128)
  CUtensorMap w0, w1, w2, w3;  // weights of layer l [N_l][K_l] (box 64 x wbox[l])
};
struct ChainArgs {
  int pdl;                // launched with programmatic dependent launch: the TMA producer waits
                          // for the predecessor grid before reading layer-0 activations
  int M;
  const int* dM;          // optional device-side M (grid sized for M = capacity)
  int nlayers;            // <= 4 GEMM layers, ReLU after every one
  int K[4], N[4], wbox[4];
  const float* bias_all;  // concatenated biases of all layers
  int bias_total;
  int mode_last;          // GEMM_OUT_X_F32 (bottom) | GEMM_OUT_CTR (top)
  float* out_f32;         // X slot 0, row stride ldo
  int ldo;
  const float* w_last;    // width-1 output layer [N_last] + b_last (top)
  int wl_n;
  float b_last;
  float* ctr;
  float* logit;
  int act_kblocks;        // 64-column blocks of the widest hidden activation
  int tmem_cols;          // power of two >= 32 and >= max N
  int stages;             // set by chain_configure
  int nchunk;             // N-chunk rows per MMA / weight box (128 or 256), set by chain_configure
  unsigned long long* dbg;  // diagnostic: %globaltimer stamps of CTA 0 (nullptr = off)
  int dbg_mode;             // diagnostic: bit0 skip TMEM loads, bit1 skip hidden smem stores
  const float* ix;          // top chain with the dot interaction fused (nullptr = A by TMA):
  int ir;                   //   X [M][ir][32] fp32, ir = T + 1 (chain_interact_supported)
  int dbuf;                 // set by launch_mlp_chain: two TMEM accumulators (persistent CTAs)
};
bool chain_interact_supported(int T, int D);
size_t chain_smem_bytes(const ChainArgs& a);
bool chain_configure(ChainArgs& a);   // false: does not fit in shared memory
void chain_prepare();                 // per-device kernel attribute
void launch_mlp_chain(const ChainMaps& maps, const ChainArgs& a, cudaStream_t s);
// Scheduling priority given to the dense-stage kernels (fused MLPs, interaction) through the
// launch attribute (0 = stream default).  Experiment knob (REC_PRIO).
extern int g_dense_prio;
extern int g_sls_prio;  // same for the synthetic-index SLS
extern int g_gemm_stages;
extern int g_gemm_mt1;
extern int g_interact_wpc;  // interaction warps per CTA (REC_INTERACT_WPC)
extern int g_interact_pf;   // few-CTA prefetching interaction kernel (REC_INTERACT_PF)
extern int kBlockedRows;    // interaction register blocking from this many rows (REC_INTERACT_BLOCKED)  // per-layer GEMM ring depth cap (REC_GEMM_STAGES; 0 = maximum)

// --------------------------------------------------------------- interaction (a5)
// MT-WnD (R26, R28): A_top[b] = bf16(X[b][1..T] concatenated) ++ 0-pad (ld = Ktop_pad) and
// wide[b][k] = sum_c u[c] v_k[c] (fp32) for the n_tasks wide vectors v [n_tasks][T*D].
void launch_concat(const float* X, int B, const int* dB, int T, int D, __nv_bfloat16* A_top, int ld,
                   const float* v, int n_tasks, float* wide, cudaStream_t s);
void launch_interact(const float* X, int B, const int* dB, int T, int D, __nv_bfloat16* A_top,
                     int ld_top, cudaStream_t s);


}  // namespace rec
