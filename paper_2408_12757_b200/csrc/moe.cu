// MoE FFN (Mixtral-8x7B shape) around the grouped tcgen05 GEMMs:
//
//   route   : RMS statistics + router logits + top-k + renormalised softmax (A-20, A-21)
//   route also groups: per-CTA expert counts, scanned over CTAs by the last CTA into
//            128-row padded expert segments (A-23)
//   scatter : each assignment's grouped row + its h1 row copied into the grouped A operand
//   [grouped Up/Gate GEMM, SiLU*up, 1/rms row scale]    gemm.cu, EPI_SILU
//   [grouped Down GEMM, routing-weight row scale, bf16] gemm.cu, EPI_STORE
//   combine : out = h1 + sum_j y[dst(t, j)] (fp32 sum, one rounding) + RMS partials
//
// All of these are HBM/L2-bound and small next to the expert GEMMs; their bytes
// per token are in DESIGN.md §7.
#include "common.cuh"
#include "profile.h"
#include "moe.cuh"

namespace nf {

namespace {

template <int EMAX, int TOK>
NF_DEV void route_token(float (&red)[8][TOK][EMAX + 1], int j, int t, int D, int E, int k, float eps,
                        int* __restrict__ ids, float* __restrict__ wts, float* __restrict__ inv_rms,
                        int (&sel_out)[MOE_MAX_TOPK]);
template <int TOK>
NF_DEV void group_epilogue(const int (&sel_s)[TOK][MOE_MAX_TOPK], int t0, int T, int k, int E, const MoeGroupArgs& g);

// One CTA of 8 warps per TOK (4) tokens: warp w accumulates the RMS sum of squares and
// the E router dot products of all TOK tokens over its D/8 slice (each router
// element read once per CTA, reused TOK times), the CTA reduces over warps in
// smem, and thread t < TOK runs the top-k of token t.
template <int EMAX, int TOK>
__global__ void __launch_bounds__(256) moe_route_kernel(const __nv_bfloat16* __restrict__ h1, int T, int D,
                                                        const float* __restrict__ router, int E, int k, float eps,
                                                        int* __restrict__ ids, float* __restrict__ wts,
                                                        float* __restrict__ inv_rms, MoeGroupArgs g) {
  __shared__ float red[8][TOK][EMAX + 1];
  __shared__ int sel_s[TOK][MOE_MAX_TOPK];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t0 = blockIdx.x * TOK;
  const int d0 = warp * (D / 8), d1 = d0 + D / 8;
  float acc[TOK][EMAX], sq[TOK];
#pragma unroll
  for (int j = 0; j < TOK; ++j) {
    sq[j] = 0.f;
#pragma unroll
    for (int e = 0; e < EMAX; ++e) acc[j][e] = 0.f;
  }
  for (int i = d0 + lane * 8; i < d1; i += 256) {
    float x[TOK][8];
#pragma unroll
    for (int j = 0; j < TOK; ++j) {
      uint4 u = make_uint4(0, 0, 0, 0);
      if (t0 + j < T) u = *reinterpret_cast<const uint4*>(h1 + (int64_t)(t0 + j) * D + i);
      const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = unpack_bf16x2(w4[q]);
        x[j][2 * q] = f.x;
        x[j][2 * q + 1] = f.y;
        sq[j] = fmaf(f.x, f.x, sq[j]);
        sq[j] = fmaf(f.y, f.y, sq[j]);
      }
    }
#pragma unroll
    for (int e = 0; e < EMAX; ++e) {
      if (e < E) {
        const float4 a = *reinterpret_cast<const float4*>(router + (int64_t)e * D + i);
        const float4 b = *reinterpret_cast<const float4*>(router + (int64_t)e * D + i + 4);
#pragma unroll
        for (int j = 0; j < TOK; ++j) {
          float s = acc[j][e];
          s = fmaf(x[j][0], a.x, s); s = fmaf(x[j][1], a.y, s); s = fmaf(x[j][2], a.z, s); s = fmaf(x[j][3], a.w, s);
          s = fmaf(x[j][4], b.x, s); s = fmaf(x[j][5], b.y, s); s = fmaf(x[j][6], b.z, s); s = fmaf(x[j][7], b.w, s);
          acc[j][e] = s;
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < TOK; ++j) {
#pragma unroll
    for (int o = 16; o; o >>= 1) sq[j] += __shfl_xor_sync(0xffffffffu, sq[j], o);
#pragma unroll
    for (int e = 0; e < EMAX; ++e)
#pragma unroll
      for (int o = 16; o; o >>= 1) acc[j][e] += __shfl_xor_sync(0xffffffffu, acc[j][e], o);
  }
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < TOK; ++j) {
      red[warp][j][EMAX] = sq[j];
#pragma unroll
      for (int e = 0; e < EMAX; ++e) red[warp][j][e] = acc[j][e];
    }
  }
  __syncthreads();
  const int j = threadIdx.x, t = t0 + j;
  if (j < TOK && t < T) route_token<EMAX, TOK>(red, j, t, D, E, k, eps, ids, wts, inv_rms, sel_s[j]);
  if (g.cta_cnt != nullptr) group_epilogue<TOK>(sel_s, t0, T, k, E, g);
}

// top-k of token t (thread j of its CTA) from the CTA's per-warp partial sums
template <int EMAX, int TOK>
NF_DEV void route_token(float (&red)[8][TOK][EMAX + 1], int j, int t, int D, int E, int k, float eps,
                        int* __restrict__ ids, float* __restrict__ wts, float* __restrict__ inv_rms,
                        int (&sel_out)[MOE_MAX_TOPK]) {
  // fixed summation order over the 8 D-slices (deterministic)
  float ssq = 0.f, l[EMAX];
#pragma unroll
  for (int e = 0; e < EMAX; ++e) l[e] = 0.f;
  for (int w = 0; w < 8; ++w) {
    ssq += red[w][j][EMAX];
#pragma unroll
    for (int e = 0; e < EMAX; ++e) l[e] += red[w][j][e];
  }
  const float inv = rsqrtf(ssq / (float)D + eps);
#pragma unroll
  for (int e = 0; e < EMAX; ++e) l[e] *= inv;
  // top-k: largest logit, lowest index on ties (strict > over ascending e)
  int sel[MOE_MAX_TOPK];
  float sl[MOE_MAX_TOPK];
  uint32_t used = 0;
  for (int q = 0; q < k; ++q) {
    int bi = -1;
    float bv = -INFINITY;
#pragma unroll
    for (int e = 0; e < EMAX; ++e)
      if (e < E && !((used >> e) & 1u) && (bi < 0 || l[e] > bv)) { bv = l[e]; bi = e; }
    used |= 1u << bi;
    sel[q] = bi;
    sl[q] = bv;
  }
  float p[MOE_MAX_TOPK], z = 0.f;
  for (int q = 0; q < k; ++q) { p[q] = expf(sl[q] - sl[0]); z += p[q]; }
  for (int q = 0; q < k; ++q) {
    ids[(int64_t)t * k + q] = sel[q];
    wts[(int64_t)t * k + q] = p[q] / z;
    sel_out[q] = sel[q];
  }
  inv_rms[t] = inv;
}

// Grouping fused into the router (reading A-23): every CTA publishes its per-expert
// assignment counts; the last CTA to finish (atomic ticket) scans them over CTAs in
// CTA order (= token order), lays out the 128-row padded expert segments, writes each
// CTA's base rank per expert and marks the padding rows.  moe_scatter_kernel then
// places every assignment without a separate single-CTA grouping pass.
template <int TOK>
NF_DEV void group_epilogue(const int (&sel_s)[TOK][MOE_MAX_TOPK], int t0, int T, int k, int E, const MoeGroupArgs& g) {
  __shared__ bool is_last;
  __shared__ int tot[MOE_MAX_EXPERTS], off[MOE_MAX_EXPERTS + 1];
  __syncthreads();
  const int cta = blockIdx.x, nb = gridDim.x;
  if (threadIdx.x < E) {
    int c = 0;
    for (int j = 0; j < TOK; ++j)
      if (t0 + j < T)
        for (int q = 0; q < k; ++q) c += sel_s[j][q] == (int)threadIdx.x;
    g.cta_cnt[(int64_t)cta * E + threadIdx.x] = c;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) is_last = atomicAdd(g.counter, 1) == nb - 1;
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  // exclusive scan over CTAs, all experts at once: thread i owns CTAs [i*per, (i+1)*per)
  const int per = (nb + blockDim.x - 1) / blockDim.x;
  const int c0 = threadIdx.x * per, c1 = min(nb, c0 + per);
  int local[MOE_MAX_EXPERTS];
  for (int e = 0; e < E; ++e) local[e] = 0;
  for (int c = c0; c < c1; ++c)
    for (int e = 0; e < E; ++e) local[e] += __ldcg(g.cta_cnt + (int64_t)c * E + e);
  __shared__ int wsum[8][MOE_MAX_EXPERTS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl[MOE_MAX_EXPERTS];
  for (int e = 0; e < E; ++e) {
    int v = local[e];
    for (int o = 1; o < 32; o <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += n;
    }
    incl[e] = v;
    if (lane == 31) wsum[warp][e] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int e = 0; e < E; ++e) {
      int run = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
        const int v = wsum[w][e];
        wsum[w][e] = run;
        run += v;
      }
      tot[e] = run;
    }
    off[0] = 0;
    for (int e = 0; e < E; ++e) off[e + 1] = off[e] + (tot[e] + g.tile - 1) / g.tile * g.tile;
    for (int e = 0; e <= E; ++e) g.grp_off[e] = off[e];
    for (int e = 0; e < E; ++e) g.grp_end[e] = off[e] + tot[e];
    *g.counter = 0;  // self-reset for the next launch
  }
  __syncthreads();
  for (int e = 0; e < E; ++e) {
    int base = wsum[warp][e] + incl[e] - local[e];  // exclusive prefix of this thread's first CTA
    for (int c = c0; c < c1; ++c) {
      g.cta_base[(int64_t)c * E + e] = base;
      base += __ldcg(g.cta_cnt + (int64_t)c * E + e);
    }
  }
  // padding rows of every segment
  for (int e = 0; e < E; ++e)
    for (int p = off[e] + tot[e] + threadIdx.x; p < off[e + 1]; p += blockDim.x) {
      g.row_tok[p] = -1;
      g.row_w[p] = 0.f;
      g.row_inv[p] = 0.f;
    }
}

// Places the assignments of one route CTA's TOK tokens (A-23 ranks: segment offset +
// the CTA's base + rank inside the CTA in assignment order) and copies their h1 rows
// into the grouped A operand (xg may be null: placement only).
template <int TOK>
__global__ void __launch_bounds__(256) moe_scatter_kernel(const __nv_bfloat16* __restrict__ h1, int T, int D, int k,
                                                          int E, const int* __restrict__ ids,
                                                          const float* __restrict__ wts,
                                                          const float* __restrict__ inv_rms, MoeGroupArgs g,
                                                          int* __restrict__ dst, __nv_bfloat16* __restrict__ xg) {
  __shared__ int pos[TOK * MOE_MAX_TOPK];
  const int t0 = blockIdx.x * TOK;
  const int n = min(TOK, T - t0) * k;
  if ((int)threadIdx.x < n) {
    const int a = t0 * k + threadIdx.x;
    const int e = ids[a];
    int r = 0;
    for (int b = t0 * k; b < a; ++b) r += ids[b] == e;
    const int p = g.grp_off[e] + g.cta_base[(int64_t)blockIdx.x * E + e] + r;
    const int t = a / k;
    pos[threadIdx.x] = p;
    dst[a] = p;
    g.row_tok[p] = t;
    g.row_w[p] = wts[a];
    g.row_inv[p] = inv_rms[t];
  }
  if (xg == nullptr) return;
  __syncthreads();
  const int n16 = D / 8;
  for (int i = threadIdx.x; i < n * n16; i += blockDim.x) {
    const int q = i / n16, c = i - q * n16;
    const int t = t0 + q / k;
    reinterpret_cast<uint4*>(xg + (int64_t)pos[q] * D)[c] = reinterpret_cast<const uint4*>(h1 + (int64_t)t * D)[c];
  }
}

// Flat elementwise form: one thread per 8 columns of one token; a warp covers 256
// columns of a token (D % 256 == 0), so the RMS partial of each 128-column unit is a
// reduction over 16 lanes.
template <int KMAX>
__global__ void __launch_bounds__(256) moe_combine_kernel(const __nv_bfloat16* __restrict__ y, const int* __restrict__ dst,
                                                          int T, int k, int D,
                                                          const __nv_bfloat16* __restrict__ resid,
                                                          __nv_bfloat16* __restrict__ out, float* __restrict__ part,
                                                          int64_t part_stride, float* __restrict__ outf) {
  const int n8 = D / 8;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)T * n8) return;  // whole warps exit together (n8 % 32 == 0)
  const int t = (int)(i / n8), c = (int)(i - (int64_t)t * n8) * 8;
  float s[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) s[q] = 0.f;
#pragma unroll
  for (int j = 0; j < KMAX; ++j) {
    if (j < k) {
      const uint4 v = *reinterpret_cast<const uint4*>(y + (int64_t)dst[(int64_t)t * k + j] * D + c);
      const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = unpack_bf16x2(w4[q]);
        s[2 * q] += f.x;
        s[2 * q + 1] += f.y;
      }
    }
  }
  if (outf != nullptr) {
    float4* o = reinterpret_cast<float4*>(outf + (int64_t)t * D + c);
    o[0] = make_float4(s[0], s[1], s[2], s[3]);
    o[1] = make_float4(s[4], s[5], s[6], s[7]);
    return;
  }
  float r[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) r[q] = 0.f;
  if (resid != nullptr) {
    const uint4 v = *reinterpret_cast<const uint4*>(resid + (int64_t)t * D + c);
    const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 f = unpack_bf16x2(w4[q]);
      r[2 * q] = f.x;
      r[2 * q + 1] = f.y;
    }
  }
  float o[8], sq = 0.f;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    o[q] = round_bf16(r[q] + s[q]);
    sq = fmaf(o[q], o[q], sq);
  }
  *reinterpret_cast<uint4*>(out + (int64_t)t * D + c) =
      make_uint4(pack_bf16x2(o[0], o[1]), pack_bf16x2(o[2], o[3]), pack_bf16x2(o[4], o[5]), pack_bf16x2(o[6], o[7]));
  if (part != nullptr) {
#pragma unroll
    for (int m = 8; m; m >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, m);
    if ((threadIdx.x & 15) == 0) part[(int64_t)(c >> 7) * part_stride + t] = sq;
  }
}

__global__ void pack_router_kernel(const __nv_bfloat16* __restrict__ w, const __nv_bfloat16* __restrict__ g, int E,
                                   int D, float* __restrict__ dst) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)E * D) return;
  dst[i] = __bfloat162float(w[i]) * __bfloat162float(g[i % D]);
}

}  // namespace

cudaError_t launch_moe_route(const __nv_bfloat16* h1, int T, int D, const float* router, int E, int k, float eps,
                             int* ids, float* wts, float* inv_rms, const MoeGroupArgs& g, cudaStream_t st) {
  if (T <= 0) return cudaSuccess;
  if (E > MOE_MAX_EXPERTS || k > MOE_MAX_TOPK || D % 8 != 0) return cudaErrorInvalidValue;
  if (D % 64 != 0) return cudaErrorInvalidValue;  // 8 warps x 8-element lanes
  const int blocks = (T + MOE_ROUTE_TOK - 1) / MOE_ROUTE_TOK;
  if (E <= 8)
    moe_route_kernel<8, MOE_ROUTE_TOK><<<blocks, 256, 0, st>>>(h1, T, D, router, E, k, eps, ids, wts, inv_rms, g);
  else
    moe_route_kernel<16, MOE_ROUTE_TOK><<<blocks, 256, 0, st>>>(h1, T, D, router, E, k, eps, ids, wts, inv_rms, g);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_moe_scatter(const __nv_bfloat16* h1, int T, int D, int k, int E, const int* ids, const float* wts,
                               const float* inv_rms, const MoeGroupArgs& g, int* dst, __nv_bfloat16* xg,
                               cudaStream_t st) {
  if (T <= 0) return cudaSuccess;
  const int blocks = (T + MOE_ROUTE_TOK - 1) / MOE_ROUTE_TOK;
  moe_scatter_kernel<MOE_ROUTE_TOK><<<blocks, 256, 0, st>>>(h1, T, D, k, E, ids, wts, inv_rms, g, dst, xg);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_moe_combine(const __nv_bfloat16* y, const int* dst, int T, int k, int D, const __nv_bfloat16* resid,
                               __nv_bfloat16* out, float* part, int64_t part_stride, float* outf, cudaStream_t st) {
  if (T <= 0) return cudaSuccess;
  if (D % 256 != 0 || k > MOE_MAX_TOPK) return cudaErrorInvalidValue;
  const int blocks = (int)(((int64_t)T * (D / 8) + 255) / 256);
  if (k <= 2)
    moe_combine_kernel<2><<<blocks, 256, 0, st>>>(y, dst, T, k, D, resid, out, part, part_stride, outf);
  else
    moe_combine_kernel<MOE_MAX_TOPK><<<blocks, 256, 0, st>>>(y, dst, T, k, D, resid, out, part, part_stride, outf);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_pack_router(const __nv_bfloat16* w_router, const __nv_bfloat16* gamma, int E, int D, float* dst,
                               cudaStream_t st) {
  const int64_t n = (int64_t)E * D;
  pack_router_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(w_router, gamma, E, D, dst);
  count_launch();
  return cudaGetLastError();
}

// One kernel of this translation unit (preload_all_kernels: its module is loaded eagerly).
const void* kernel_anchor_moe() { return reinterpret_cast<const void*>(pack_router_kernel); }

}  // namespace nf
