// Internal interface of the persistent tcgen05 GEMM (C = A . B^T, bf16 in, f32
// accumulate in TMEM) with the fused epilogues of the decoder layer.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace nf {

enum GemmEpiMode : int {
  EPI_STORE = 0,   // out = bf16(acc * row_scale)
  EPI_RESID = 1,   // out = bf16(resid + acc); optional sum-of-squares partials of out
  EPI_SILU = 2,    // tile = [gate 128 | up 128]: out = bf16(silu(g*s) * (u*s))
  EPI_QKV = 3,     // q/k RoPE at pos, q -> q_out, k/v -> paged KV pool slots
  EPI_ARGMAX = 4,  // per (n-tile,row) partial (max, argmax) of acc
  EPI_F32 = 5,     // outf = acc * row_scale (f32, for TP partial sums)
  EPI_PEER = 6,    // bf16(acc * row_scale) partial 128x256 blocks into their owner ranks' staging (peer.cuh)
};

constexpr int GEMM_BM = 128;
constexpr int GEMM_BN = 256;
constexpr int GEMM_BK = 64;
constexpr int GEMM_STAGES = 4;      // default ring depth; 3 when co-resident with attention CTAs
constexpr int GEMM_THREADS = 256;  // warp0 TMA, warp1 MMA, warp2 TMEM alloc, warps 4-7 epilogue
constexpr int GEMM_SK_LD = 256;    // stream-K partial tile row stride (floats)
constexpr int gemm_smem_bn(int stages, int bn) { return stages * (GEMM_BM + bn) * GEMM_BK * 2 + 1024 + 512; }
constexpr int GEMM_NORM_COLS = 128;  // columns per RMS sum-of-squares partial (EPI_RESID)

struct GemmArgs {
  int epi;
  int stages;           // smem ring depth: 4 (default) or 3 (co-resident with attention)
  int M, N, K;          // rows of A in this launch, rows of B (packed output columns), reduction dim
  int n_valid;          // valid output columns (EPI_SILU: F; else N)
  // outputs (row-indexed pointers are pre-offset to the launch's first row)
  __nv_bfloat16* out;
  int64_t ldo;
  float* outf;
  const __nv_bfloat16* resid;
  int64_t ldr;
  // row scale from RMS partials: s = rsqrt(sum_p norm_part[p*norm_stride + r] * inv_d + eps)
  const float* norm_part;
  int norm_nparts;
  int64_t norm_stride;
  float inv_d, eps;
  // sum-of-squares partial output per 128 columns: sq_out[(col / 128) * sq_stride + r]
  float* sq_out;
  int64_t sq_stride;
  // EPI_QKV
  int qh, kh, hd, page_size;
  float log2_theta;
  const int* tok_pos;    // [M]
  const int* tok_slot;   // [M] page*page_size + offset
  __nv_bfloat16* q_out;  // [M, qh, hd]
  __nv_bfloat16* kv_pool;
  // stream-K scratch (null: data-parallel tiles only): fp32 partial tile per CTA
  // [grid][128][256], arrival counters per tile (zero at launch, self-resetting)
  float* sk_part;
  int* sk_flag;
  int sk_slots;         // partial slots available in sk_part (split-K=2 needs one per tile)
  int split;            // set by the launcher: 1 or 2 (split-K=2 schedule)
  int tail_split;       // set by the launcher: K splits of the partial last wave's tiles (1 = none)
  int stream_k;         // set by the launcher: 1 = stream-K over the (tile, k-block) space (sub-wave GEMMs)
  // EPI_ARGMAX
  float* am_val;
  int* am_idx;
  int64_t am_stride;
  // per-row output scale (multiplies the RMS row scale): MoE routing weights / 1/rms of gathered rows
  const float* row_scale;
  // Grouped GEMM (MoE experts, reading A-23): A rows are expert segments starting at
  // grp_off[g] (device, multiples of GEMM_BM, grp_off[n_groups] = rows in use); rows
  // [grp_end[g], grp_off[g+1]) are padding (not stored).  B holds n_groups blocks of N
  // rows; the m-tile's group selects its block.  Data-parallel single-CTA tiles only.
  const int* grp_off;
  const int* grp_end;
  int n_groups;
  // EPI_PEER (peer.cuh): block (bm, bn) of 128 rows x 256 columns belongs to
  // rank (bm + bn * peer_mb) % peer_n; the partial goes to that rank's buffer at
  // peer_site_off + peer_stage_off + [peer_rank][owned index][128][256], then the owner's flag
  // at peer_site_off + peer_flags_off + 256 + 4 * (owned index * peer_n + peer_rank) is bumped by BN/64
  // (release, sys scope)
  uint8_t* const* peer_bases;  // device array [peer_n]: every rank's symmetric buffer
  int64_t peer_site_off, peer_stage_off, peer_flags_off, peer_result_off;
  int peer_n, peer_rank, peer_maxown, peer_mb;
  // peer_mode 1 (EPI_RESID, the O column-parallel projection): the output slice goes to every
  // rank's all-gather region [peer_n][M][N] at peer_site_off + peer_result_off instead of `out`,
  // then every rank's site `done` counter grows by the unit's 64-column chunks (release, sys)
  int peer_mode;
  // A in slot layout (a_slots > 1): A[m][s * a_slot_w + j] is stored at A + (s * M + m) * a_slot_w + j,
  // the layout an AllGather of a_slots row blocks [M][a_slot_w] leaves (TP: the attention output
  // feeding the O column-parallel projection); loaded by a 3-D TMA box per k-block, no interleave pass
  int a_slots, a_slot_w;
  int sk_smem;          // set by the launcher: the owner of a split tile stages a partial in smem
};

// Bytes of stream-K scratch for a GEMM with this many tiles at this grid.
inline size_t gemm_sk_bytes(int slots, int tiles) { return (size_t)slots * GEMM_BM * 256 * 4 + (size_t)tiles * 4 + 256; }

// A: [M, K] row-major (lda elements), B: [N, K] row-major (ldb elements).
// grid = min(tiles, sm_budget) persistent CTAs, one per SM.
cudaError_t launch_gemm(const __nv_bfloat16* A, int64_t lda, const __nv_bfloat16* B, int64_t ldb,
                        const GemmArgs& args, int sm_budget, cudaStream_t stream);

}  // namespace nf
