// MoE FFN kernels around the grouped tcgen05 GEMMs ("gating
// inserted into the pipeline"; readings A-20..A-23 in DESIGN.md).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace nf {

constexpr int MOE_MAX_EXPERTS = 16;
constexpr int MOE_MAX_TOPK = 4;

// Router (A-20, A-21): for each of T rows of h1 [T, D] bf16: inv_rms = 1/sqrt(mean(h1^2)+eps),
// logits[e] = inv_rms * sum_i h1_i * router[e, i] (router = gamma_ffn * W_r, fp32 [E, D]),
// top-k by logit (ties: lowest expert), weights = softmax over the k selected logits.
// ids/wts: [T, k]; inv_rms: [T].
cudaError_t launch_moe_route(const __nv_bfloat16* h1, int T, int D, const float* router, int E, int k, float eps,
                             int* ids, float* wts, float* inv_rms, cudaStream_t st);
// Token grouping (A-23), one CTA: grp_off [E+1] (segments padded to `tile` rows), grp_end [E],
// dst [T*k], and per grouped row p < grp_off[E]: row_tok (-1 = padding), row_w (routing weight),
// row_inv (1/rms of its token).
cudaError_t launch_moe_group(const int* ids, const float* wts, const float* inv_rms, int T, int k, int E, int tile,
                             int* grp_off, int* grp_end, int* dst, int* row_tok, float* row_w, float* row_inv,
                             cudaStream_t st);
// xg[p] = h1[row_tok[p]] (zeros for padding rows), p < grp_off[E] <= cap.
cudaError_t launch_moe_gather(const __nv_bfloat16* h1, int D, const int* row_tok, const int* grp_off_end, int cap,
                              __nv_bfloat16* xg, cudaStream_t st);
// Weighted combine (y: bf16 weighted expert outputs of the grouped rows):
// out[t] = bf16(resid[t] + sum_j y[dst[t*k+j]]) in fp32 (resid may be null: the
// bf16 partial of a TP rank) with RMS sum-of-squares partials of out per 128 columns
// part[(c/128)*part_stride + t] (part may be null); outf != null: outf[t] = sum_j y[...] in fp32 instead.
cudaError_t launch_moe_combine(const __nv_bfloat16* y, const int* dst, int T, int k, int D, const __nv_bfloat16* resid,
                               __nv_bfloat16* out, float* part, int64_t part_stride, float* outf, cudaStream_t st);
// router_packed[e, i] = W_r[e, i] * gamma[i] in fp32 (exact: a product of two bf16 values).
cudaError_t launch_pack_router(const __nv_bfloat16* w_router, const __nv_bfloat16* gamma, int E, int D, float* dst,
                               cudaStream_t st);

}  // namespace nf
