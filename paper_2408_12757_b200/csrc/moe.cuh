// MoE FFN kernels around the grouped tcgen05 GEMMs ("gating
// inserted into the pipeline"; readings A-20..A-23 in DESIGN.md).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace nf {

constexpr int MOE_MAX_EXPERTS = 16;
constexpr int MOE_MAX_TOPK = 4;
constexpr int MOE_ROUTE_TOK = 4;  // tokens per router CTA (and per scatter CTA)

// Token grouping state (reading A-23) shared by the router's fused grouping epilogue and
// the scatter kernel.  cta_cnt / cta_base: [ceil(T / MOE_ROUTE_TOK)][E]; counter: one int,
// zero before the first launch (self-resetting); grp_off [E+1], grp_end [E]; row_tok /
// row_w / row_inv: [rows capacity] (padding rows get -1 / 0 / 0).
struct MoeGroupArgs {
  int* cta_cnt;
  int* cta_base;
  int* counter;
  int* grp_off;
  int* grp_end;
  int* row_tok;
  float* row_w;
  float* row_inv;
  int tile;
};
inline size_t moe_group_ints(int64_t T, int E) { return 2 * (size_t)((T + MOE_ROUTE_TOK - 1) / MOE_ROUTE_TOK) * E; }

// Router (A-20, A-21): for each of T rows of h1 [T, D] bf16: inv_rms = 1/sqrt(mean(h1^2)+eps),
// logits[e] = inv_rms * sum_i h1_i * router[e, i] (router = gamma_ffn * W_r, fp32 [E, D]),
// top-k by logit (ties: lowest expert), weights = softmax over the k selected logits.
// ids/wts: [T, k]; inv_rms: [T].
// With g.cta_cnt != null the router also groups (see MoeGroupArgs); then
// launch_moe_scatter places the assignments (dst [T*k], row_* of every grouped row)
// and copies the h1 rows into xg (xg may be null).
cudaError_t launch_moe_route(const __nv_bfloat16* h1, int T, int D, const float* router, int E, int k, float eps,
                             int* ids, float* wts, float* inv_rms, const MoeGroupArgs& g, cudaStream_t st);
cudaError_t launch_moe_scatter(const __nv_bfloat16* h1, int T, int D, int k, int E, const int* ids, const float* wts,
                               const float* inv_rms, const MoeGroupArgs& g, int* dst, __nv_bfloat16* xg,
                               cudaStream_t st);
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
