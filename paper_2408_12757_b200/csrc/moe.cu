// MoE FFN (Mixtral-8x7B shape) around the grouped tcgen05 GEMMs:
//
//   route   : RMS statistics + router logits + top-k + renormalised softmax (A-20, A-21)
//   group   : counting sort of the T*k assignments into 128-row expert segments (A-23)
//   gather  : h1 rows -> grouped A operand (one row per assignment)
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

// One CTA of 8 warps per TOK (4) tokens: warp w accumulates the RMS sum of squares and
// the E router dot products of all TOK tokens over its D/8 slice (each router
// element read once per CTA, reused TOK times), the CTA reduces over warps in
// smem, and thread t < TOK runs the top-k of token t.
template <int EMAX, int TOK>
__global__ void __launch_bounds__(256) moe_route_kernel(const __nv_bfloat16* __restrict__ h1, int T, int D,
                                                        const float* __restrict__ router, int E, int k, float eps,
                                                        int* __restrict__ ids, float* __restrict__ wts,
                                                        float* __restrict__ inv_rms) {
  __shared__ float red[8][TOK][EMAX + 1];
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
  if (j >= TOK || t >= T) return;
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
  }
  inv_rms[t] = inv;
}

// One CTA of 1024 threads.  Pass 1 counts assignments per expert; thread 0 lays out
// the padded segments; pass 2 ranks assignments chunk by chunk in increasing
// assignment order (warp ballots + a per-expert scan over the 32 warps), so each
// expert's rows are in token-major order (A-23).
__global__ void __launch_bounds__(1024) moe_group_kernel(const int* __restrict__ ids, const float* __restrict__ wts,
                                                         const float* __restrict__ inv_rms, int T, int k, int E,
                                                         int tile, int* __restrict__ grp_off,
                                                         int* __restrict__ grp_end, int* __restrict__ dst,
                                                         int* __restrict__ row_tok, float* __restrict__ row_w,
                                                         float* __restrict__ row_inv) {
  __shared__ int cnt[MOE_MAX_EXPERTS], off[MOE_MAX_EXPERTS + 1], run[MOE_MAX_EXPERTS];
  __shared__ int wcnt[32][MOE_MAX_EXPERTS];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = T * k;
  if (tid < MOE_MAX_EXPERTS) { cnt[tid] = 0; run[tid] = 0; }
  __syncthreads();
  for (int a = tid; a < n; a += 1024) atomicAdd(&cnt[ids[a]], 1);
  __syncthreads();
  if (tid == 0) {
    off[0] = 0;
    for (int e = 0; e < E; ++e) off[e + 1] = off[e] + (cnt[e] + tile - 1) / tile * tile;
    for (int e = 0; e <= E; ++e) grp_off[e] = off[e];
    for (int e = 0; e < E; ++e) grp_end[e] = off[e] + cnt[e];
  }
  __syncthreads();
  // padding rows of every segment
  for (int e = 0; e < E; ++e)
    for (int p = off[e] + cnt[e] + tid; p < off[e + 1]; p += 1024) {
      row_tok[p] = -1;
      row_w[p] = 0.f;
      row_inv[p] = 0.f;
    }
  const uint32_t lt = (1u << lane) - 1u;
  for (int base = 0; base < n; base += 1024) {
    const int a = base + tid;
    const int e = a < n ? ids[a] : -1;
    int rank = 0;
    for (int q = 0; q < E; ++q) {
      const uint32_t m = __ballot_sync(0xffffffffu, e == q);
      if (e == q) rank = __popc(m & lt);
      if (lane == 0) wcnt[warp][q] = __popc(m);
    }
    __syncthreads();
    if (tid < E) {  // exclusive scan over warps for expert tid, continuing from earlier chunks
      int s = run[tid];
      for (int w = 0; w < 32; ++w) {
        const int c = wcnt[w][tid];
        wcnt[w][tid] = s;
        s += c;
      }
      run[tid] = s;
    }
    __syncthreads();
    if (e >= 0) {
      const int p = off[e] + wcnt[warp][e] + rank;
      const int t = a / k;
      dst[a] = p;
      row_tok[p] = t;
      row_w[p] = wts[a];
      row_inv[p] = inv_rms[t];
    }
    __syncthreads();
  }
}

// Flat elementwise form: one thread per 16 bytes (8 bf16) of a grouped row, so the
// whole copy is in flight at once (the per-warp row loop was latency-bound).
__global__ void moe_gather_kernel(const __nv_bfloat16* __restrict__ h1, int D, const int* __restrict__ row_tok,
                                  const int* __restrict__ grp_off_end, int cap, __nv_bfloat16* __restrict__ xg) {
  const int rows = min(*grp_off_end, cap);
  const int n16 = D / 8;
  const int64_t total = (int64_t)rows * n16;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int p = (int)(i / n16), c = (int)(i - (int64_t)p * n16);
    const int t = row_tok[p];
    uint4 v = make_uint4(0, 0, 0, 0);
    if (t >= 0) v = reinterpret_cast<const uint4*>(h1 + (int64_t)t * D)[c];
    reinterpret_cast<uint4*>(xg + (int64_t)p * D)[c] = v;
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
                             int* ids, float* wts, float* inv_rms, cudaStream_t st) {
  if (T <= 0) return cudaSuccess;
  if (E > MOE_MAX_EXPERTS || k > MOE_MAX_TOPK || D % 8 != 0) return cudaErrorInvalidValue;
  if (D % 64 != 0) return cudaErrorInvalidValue;  // 8 warps x 8-element lanes
  constexpr int TOK = 4;  // 4 tokens per CTA: ~2 waves of small CTAs keep enough loads in flight
  const int blocks = (T + TOK - 1) / TOK;
  if (E <= 8)
    moe_route_kernel<8, TOK><<<blocks, 256, 0, st>>>(h1, T, D, router, E, k, eps, ids, wts, inv_rms);
  else
    moe_route_kernel<16, TOK><<<blocks, 256, 0, st>>>(h1, T, D, router, E, k, eps, ids, wts, inv_rms);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_moe_group(const int* ids, const float* wts, const float* inv_rms, int T, int k, int E, int tile,
                             int* grp_off, int* grp_end, int* dst, int* row_tok, float* row_w, float* row_inv,
                             cudaStream_t st) {
  if (T <= 0) return cudaSuccess;
  if (E > MOE_MAX_EXPERTS) return cudaErrorInvalidValue;
  moe_group_kernel<<<1, 1024, 0, st>>>(ids, wts, inv_rms, T, k, E, tile, grp_off, grp_end, dst, row_tok, row_w,
                                       row_inv);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_moe_gather(const __nv_bfloat16* h1, int D, const int* row_tok, const int* grp_off_end, int cap,
                              __nv_bfloat16* xg, cudaStream_t st) {
  if (cap <= 0) return cudaSuccess;
  const int64_t total = (int64_t)cap * (D / 8);
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  moe_gather_kernel<<<blocks, 256, 0, st>>>(h1, D, row_tok, grp_off_end, cap, xg);
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

}  // namespace nf
