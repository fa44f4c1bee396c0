#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace nf {
cudaError_t launch_gather_rows(const __nv_bfloat16* src, const int* idx, int rows, int D, __nv_bfloat16* dst,
                               float* part, cudaStream_t st);
cudaError_t launch_resid_add_rows(__nv_bfloat16* acc, const __nv_bfloat16* resid, int rows, int D, float* part,
                                  cudaStream_t st);
// out = bf16(src + resid) (src written by peers: read through L2), part = row sums of squares
cudaError_t launch_resid_add_rows_from(__nv_bfloat16* out, const __nv_bfloat16* src, const __nv_bfloat16* resid, int rows,
                                       int D, float* part, cudaStream_t st);
cudaError_t launch_gather_ids_embed(const __nv_bfloat16* embed, const int* token_ids, const int* tok_src, int rows, int D,
                                    int vocab, __nv_bfloat16* dst, float* part, cudaStream_t st);
cudaError_t launch_argmax_pairs(const float* val, const int* idx, int ntiles, int64_t stride, int rows, int idx_off,
                                float* pairs, cudaStream_t st);
cudaError_t launch_argmax_merge(const float* pairs, int n, int rows, const int* row_req, int* next_ids, cudaStream_t st);
cudaError_t launch_scatter_rows(const __nv_bfloat16* src, const int* idx, int rows, int D, __nv_bfloat16* dst,
                                cudaStream_t st);
cudaError_t launch_argmax_reduce(const float* val, const int* idx, int ntiles, int64_t stride, int rows,
                                 const int* row_req, int* next_ids, cudaStream_t st);
cudaError_t launch_interleave(const __nv_bfloat16* src, int n, int rows, int C, __nv_bfloat16* dst, float* part,
                              cudaStream_t st);
// launch_interleave reading a region other GPUs wrote (the fused all-gather): loads through L2
cudaError_t launch_interleave_from_peers(const __nv_bfloat16* src, int n, int rows, int C, __nv_bfloat16* dst,
                                         float* part, cudaStream_t st);
cudaError_t launch_sum_bf16(const void* const* in, int n, __nv_bfloat16* out, size_t count, bool ring, cudaStream_t st);
cudaError_t launch_fill_i32(int* p, int n, int v, cudaStream_t st);
cudaError_t launch_smid_probe(int* counts, int ctas, cudaStream_t st);
cudaError_t launch_assemble_tokens(const int* src, const int* prev, int* out, int T, cudaStream_t st);
cudaError_t launch_scale_cols(const __nv_bfloat16* src, const __nv_bfloat16* gamma, int64_t rows, int cols,
                              __nv_bfloat16* dst, cudaStream_t st);
cudaError_t launch_pack_gate_up(const __nv_bfloat16* gate, const __nv_bfloat16* up, const __nv_bfloat16* gamma, int F,
                                int D, __nv_bfloat16* dst, cudaStream_t st);
}  // namespace nf
