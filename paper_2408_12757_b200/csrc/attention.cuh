// Internal interface of the paged attention kernels.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace nf {

// One decode work item: query token row t attends with its R = qh/kh query
// heads of KV group `kvh` over kv_len keys listed from page_ids[page_start].
struct DecodeItem {
  int t, kvh, kv_len, page_start;
};
// One prefill work item: query rows [t0, t0+n) of one request (positions
// prefix+i0 ..), query head h; keys 0..prefix+i0+n-1 causal.
struct PrefillItem {
  int t0, n, pos0, h;   // first token row, rows in tile (<=64), position of row 0, query head
  int kv_total, page_start, pad0, pad1;
};

struct AttnArgs {
  const __nv_bfloat16* q;   // [T, qh, hd]
  __nv_bfloat16* o;         // [T, qh*hd]
  const int* page_ids;
  int qh, kh, hd, page_size;
  float scale_log2;         // log2(e)/sqrt(hd)
  int dec_warps;            // decode CTA size: 8 (own SMs) or 4 (co-resident with a GEMM CTA)
  int n_rows;               // T: rows of q / o (bound of the prefill kernel's q tensor map)
  int pf_dist;              // decode: L2 prefetch distance in pages within an item (0 = off); set by the launcher
  // decode row streams (optional): per consumer warp gw the TMA rows of all pages of its items in
  // order, dec_rows[dec_wstart[gw] .. dec_wstart[gw+1]) (built by launch_build_dec_rows)
  const int* dec_rows;
  const int* dec_wstart;
};

// Decode launch geometry shared by the row-stream builder and the kernel.
int decode_warps(int hd, int dec_warps_arg);
int decode_grid(int n_items, int sm_budget, int warps);
// Row streams of one decode launch (items sorted as the kernel takes them, `grid` CTAs of
// `warps` consumer warps): rows [sum of the items' pages] and wstart [grid * warps + 1].
cudaError_t launch_build_dec_rows(const DecodeItem* items, int n_items, int grid, int warps, const int* page_ids, int kh,
                                  int* rows, int* wstart, cudaStream_t st);

cudaError_t make_page_tmap(CUtensorMap* m, const void* pool, int64_t n_pages, int kh, int hd, int page_size);
// q [T, qh, hd] as a 3-D map {hd, qh, T}: box {64, 1, 128} = 128 token rows of one head, 128B-swizzled
cudaError_t make_q_tmap(CUtensorMap* m, const void* q, int64_t T, int qh, int hd);
cudaError_t make_pool_tmap(CUtensorMap* m, const void* pool, int64_t n_pages, int kh, int hd, int page_size);

cudaError_t launch_decode_attention(const CUtensorMap& pool_map, const CUtensorMap& page_map, const AttnArgs& a, const DecodeItem* items,
                                    int n_items, int sm_budget, cudaStream_t stream);
// stream decode attention (decode_stream.cu; needs a.dec_rows / a.dec_wstart built for a
// 12-warp geometry by launch_build_dec_rows): head_dim 64/128, page 16, GQA group <= 8
bool decode_stream_supported(const AttnArgs& a);
int decode_stream_warps();  // consumer warps per CTA of the stream kernel (row-stream geometry)
cudaError_t launch_decode_attention_stream(const CUtensorMap& page_map, const AttnArgs& a, const DecodeItem* items,
                                           int n_items, int sm_budget, cudaStream_t stream);
// warp-specialised decode attention (one producer warp drives every consumer warp's TMA ring); decode_ws.cu
cudaError_t launch_decode_attention_ws(const CUtensorMap& page_map, const AttnArgs& a, const DecodeItem* items,
                                       int n_items, int sm_budget, cudaStream_t stream);
// tcgen05 decode attention (head_dim 128, GQA group <= 8); decode_tc.cu
cudaError_t launch_decode_attention_tc(const CUtensorMap& pool_map, const AttnArgs& a, const DecodeItem* items,
                                       int n_items, int sm_budget, cudaStream_t stream);
// tcgen05 prefill attention (head_dim 128, 128-row items); prefill_tc.cu
cudaError_t launch_prefill_attention_tc(const CUtensorMap& pool_map, const AttnArgs& a, const PrefillItem* items,
                                        int n_items, int sm_budget, cudaStream_t stream);
// Query rows per prefill work item for this head_dim (128: tcgen05 kernel; 64: mma.sync kernel,
// also for head_dim 128 with NF_PREFILL_IMPL=mma).
int prefill_rows(int head_dim);
cudaError_t launch_prefill_attention(const CUtensorMap& pool_map, const AttnArgs& a, const PrefillItem* items,
                                     int n_items, int sm_budget, cudaStream_t stream);

}  // namespace nf
