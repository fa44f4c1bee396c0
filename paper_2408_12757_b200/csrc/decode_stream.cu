// Paged GQA decode attention, "stream" formulation (default for head_dim 64/128,
// GQA group R <= 8, "decode attention ... memory
// bound", :626 (paged KV)).
//
// Same arithmetic as decode_attn_kernel (attention.cu: transposed S^T = K.Q^T with
// the page's 16 keys as the MMA M rows and the group's query heads as N columns,
// P^T moved into a B fragment with movmatrix, O^T += V^T.P^T), rebuilt around a
// short per-page instruction chain, because that kernel is issue-bound on small SM
// partitions (profiles/r2_ncu_decode.md: ~220 issued instructions per 8 KB page, of
// which 32 are the ldmatrix / MMA work):
//  * the TMA loader walks a flat per-warp stream of page rows (a.dec_rows, built once
//    per step by build_dec_rows_kernel in the kernel's own item order): one TMA and
//    one uniform row load per page, no item headers or page-id windows;
//  * the softmax denominator l comes out of the tensor pipe: one extra MMA per page
//    with an all-ones A fragment sums the bf16 P^T columns (the same rounded P the
//    numerator uses), replacing the per-page FADDs and the final cross-lane sum;
//  * S^T accumulates in two chains (two FADDs per score instead of three);
//  * masking of keys past kv_len (scores -> -inf, V elements -> 0 in registers, no
//    shared-memory zeroing) runs only on an item's last page;
//  * ldmatrix lane offsets (swizzle included) are computed once per warp.
// Per warp: an NS-deep ring of whole pages (K and V of one KV head, one 4-D TMA box),
// a page's K and V fragments are pulled into registers and the slot is refilled
// before any softmax math (a slot is busy for the load latency only).
#include <algorithm>
#include <cstdlib>

#include "attention.cuh"
#include "common.cuh"
#include "profile.h"

namespace nf {
namespace {

constexpr int DS_BOX = 16 * 128;  // one 16-row x 64-column 128B-swizzled box

// NS = pages in flight per warp (the warp's ring depth)
template <int HD, int W, int NS>
constexpr int ds_smem() { return W * NS * (2 * 16 * HD * 2) + W * NS * 8 + 1024; }

NF_DEV uint32_t movm_trans(uint32_t a) {
  uint32_t d;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(d) : "r"(a));
  return d;
}

NF_DEV int ld_uniform(const int* p) {  // every lane loads the same word (one transaction)
  int v;
  asm volatile("ld.global.nc.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

template <int HD, int W, int NS, int CH = 2, int LA = 0>
// (registers: the warps of an SM sub-partition share its 16 K registers, ceil(W / 4) warps each)
__global__ void __maxnreg__((512 / ((W + 3) / 4) / 8 * 8) < 255 ? (512 / ((W + 3) / 4) / 8 * 8) : 255)
    decode_stream_kernel(const __grid_constant__ CUtensorMap pages, const AttnArgs a,
                         const DecodeItem* __restrict__ items, int n_items) {
  constexpr int KB = 16 * HD * 2;  // K (or V) bytes of one page of one KV head
  constexpr int SB = 2 * KB;       // stage: K then V
  constexpr int KS = HD / 16;      // k-steps of S^T = m-tiles of O^T
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring_p = smem + warp * NS * SB;
  const uint32_t ring = smem_u32(ring_p);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + W * NS * SB) + warp * NS;
  if (lane == 0) {
    if (warp == 0) tma_prefetch_desc(&pages);
    for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
    fence_barrier_init();
  }
  __syncwarp();

  // Items (sorted longest first on the host) in snake order, warp-major across CTAs --
  // the order build_dec_rows_kernel wrote this warp's row stream in.
  const int gw = warp * gridDim.x + blockIdx.x, TW = gridDim.x * W;
  auto item_of = [&](int round) { return round * TW + ((round & 1) ? TW - 1 - gw : gw); };
  const int R = a.qh / a.kh;
  const int r0 = a.dec_wstart[gw];
  const int n_pg = a.dec_wstart[gw + 1] - r0;
  const int* rows = a.dec_rows + r0;
  const uint64_t kv_policy = policy_evict_first();  // K/V pages are read exactly once: keep L2 for the GEMMs

  auto issue = [&](uint32_t j, int row) {  // page j of the stream -> slot j % NS
    if (lane == 0) {
      const uint32_t s = j % NS;
      fence_proxy_async();  // WAR: this warp's ldmatrix reads of the slot before the async-proxy refill
      mbar_arrive_expect_tx(&bars[s], SB);
      tma_load_4d_hint(ring_p + s * SB, &pages, &bars[s], 0, row, 0, 0, kv_policy);
    }
  };
#pragma unroll
  for (int j = 0; j < NS; ++j)
    if (j < n_pg) issue((uint32_t)j, ld_uniform(rows + j));
  int nrow = NS < n_pg ? ld_uniform(rows + NS) : 0;  // row of the next page to issue (loaded one page early)
  // ldmatrix lane offsets inside a stage (128B swizzle: 16-byte chunk c of row r at r*128 + ((c ^ (r&7)) << 4));
  // for k-step ks the chunk is 2*(ks&3) + hi in box ks>>2, so four offsets serve all k-steps
  const int x7 = lane & 7;
  uint32_t offK[4], offV[4];
  {
    const int keyK = x7 + (((lane >> 3) & 1) << 3), hiK = lane >> 4;
    const int keyV = x7 + ((lane >> 4) << 3), hiV = (lane >> 3) & 1;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      offK[i] = keyK * 128 + (((2 * i + hiK) ^ x7) << 4);
      offV[i] = KB + keyV * 128 + (((2 * i + hiV) ^ x7) << 4);
    }
  }
  const uint32_t ones[4] = {0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u};  // bf16 1.0 pairs
  const float sl2 = a.scale_log2, inv_sl2 = 1.f / a.scale_log2;
  const int g = lane >> 2;           // key row (C fragments) / query head column (B fragments)
  const int hc = 2 * (lane & 3);     // first of the two head columns of this lane's C fragments
  const int kk = 2 * (lane & 3);     // first key of this lane's V^T A-fragment registers 0/1 (+8: 2/3)
  uint32_t qb[KS][2];                // the item's query rows as B fragments

  // One page of the stream: wait for its slot, S^T = K.Q^T in CH independent MMA chains,
  // V^T fragments into registers, then refill the slot with the page NS ahead.
  auto load_page = [&](uint32_t jj, float (&sc)[4], uint32_t (&vf)[KS][4]) __attribute__((always_inline)) {
    const uint32_t s = jj % NS;
    mbar_wait(&bars[s], (jj / NS) & 1);
    const uint32_t base = ring + s * SB;
    float sa[CH][4];
#pragma unroll
    for (int c = 0; c < CH; ++c) sa[c][0] = sa[c][1] = sa[c][2] = sa[c][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      uint32_t kf[4];
      ldmatrix_x4(kf, base + offK[ks & 3] + (ks >> 2) * DS_BOX);
      mma_bf16_16816(sa[ks % CH], kf, qb[ks]);
    }
#pragma unroll
    for (int mt = 0; mt < KS; ++mt) ldmatrix_x4_trans(vf[mt], base + offV[mt & 3] + (mt >> 2) * DS_BOX);
    __syncwarp();
    if ((int)jj + NS < n_pg) {  // refill the slot with the page NS ahead
      issue(jj + NS, nrow);
      if ((int)jj + NS + 1 < n_pg) nrow = ld_uniform(rows + jj + NS + 1);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if constexpr (CH == 4) sc[e] = (sa[0][e] + sa[1][e]) + (sa[2][e] + sa[3][e]);
      else sc[e] = sa[0][e] + sa[1][e];
    }
  };
  // LA 2 halves of load_page: S^T of page jj (slot waited, K fragments, CH chains) ...
  auto s_only = [&](uint32_t jj, float (&sc)[4]) __attribute__((always_inline)) {
    const uint32_t s = jj % NS;
    mbar_wait(&bars[s], (jj / NS) & 1);
    const uint32_t base = ring + s * SB;
    float sa[CH][4];
#pragma unroll
    for (int c = 0; c < CH; ++c) sa[c][0] = sa[c][1] = sa[c][2] = sa[c][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      uint32_t kf[4];
      ldmatrix_x4(kf, base + offK[ks & 3] + (ks >> 2) * DS_BOX);
      mma_bf16_16816(sa[ks % CH], kf, qb[ks]);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if constexpr (CH == 4) sc[e] = (sa[0][e] + sa[1][e]) + (sa[2][e] + sa[3][e]);
      else sc[e] = sa[0][e] + sa[1][e];
    }
  };
  // ... and its V^T fragments, then the slot's refill with the page NS ahead
  auto v_only = [&](uint32_t jj, uint32_t (&vf)[KS][4]) __attribute__((always_inline)) {
    const uint32_t base = ring + (jj % NS) * SB;
#pragma unroll
    for (int mt = 0; mt < KS; ++mt) ldmatrix_x4_trans(vf[mt], base + offV[mt & 3] + (mt >> 2) * DS_BOX);
    __syncwarp();
    if ((int)jj + NS < n_pg) {
      issue(jj + NS, nrow);
      if ((int)jj + NS + 1 < n_pg) nrow = ld_uniform(rows + jj + NS + 1);
    }
  };
  // Softmax of one page's scores and its P.V contribution (page p of an item with np pages).
  auto consume = [&](int p, int np, int kv_len, float (&sc)[4], uint32_t (&vf)[KS][4], float& m0, float& m1,
                     float& thr0, float& thr1, float (&oacc)[KS][4], float (&lacc)[4]) __attribute__((always_inline)) {
    if (p == np - 1) {  // keys past kv_len exist only on the item's last page
      const int valid = kv_len - p * 16;
      if (g >= valid) sc[0] = sc[1] = -INFINITY;
      if (g + 8 >= valid) sc[2] = sc[3] = -INFINITY;
      // V rows past kv_len may hold anything (NaN in unused pool slots): zero them so P=0 rows add 0
      const uint32_t mlo = (kk < valid ? 0x0000FFFFu : 0u) | (kk + 1 < valid ? 0xFFFF0000u : 0u);
      const uint32_t mhi = (kk + 8 < valid ? 0x0000FFFFu : 0u) | (kk + 9 < valid ? 0xFFFF0000u : 0u);
#pragma unroll
      for (int mt = 0; mt < KS; ++mt) {
        vf[mt][0] &= mlo;
        vf[mt][1] &= mlo;
        vf[mt][2] &= mhi;
        vf[mt][3] &= mhi;
      }
    }
    // Online softmax with a lazily updated running max (attention.cu): probabilities are
    // taken against a stale max as long as no raw score exceeds thr = (m + 8) / scale;
    // the cross-lane max and the rescale of O and l run only when the max really moves.
    if (__any_sync(0xffffffffu, fmaxf(sc[0], sc[2]) > thr0 || fmaxf(sc[1], sc[3]) > thr1)) {
      float r0m = fmaxf(sc[0], sc[2]), r1m = fmaxf(sc[1], sc[3]);
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        r0m = fmaxf(r0m, __shfl_xor_sync(0xffffffffu, r0m, o));
        r1m = fmaxf(r1m, __shfl_xor_sync(0xffffffffu, r1m, o));
      }
      const float mn0 = fmaxf(m0, r0m * sl2), mn1 = fmaxf(m1, r1m * sl2);
      const float al0 = exp2f(m0 - mn0), al1 = exp2f(m1 - mn1);
      m0 = mn0;
      m1 = mn1;
      thr0 = (mn0 + 8.f) * inv_sl2;
      thr1 = (mn1 + 8.f) * inv_sl2;
      lacc[0] *= al0; lacc[2] *= al0;
      lacc[1] *= al1; lacc[3] *= al1;
#pragma unroll
      for (int mt = 0; mt < KS; ++mt) {
        oacc[mt][0] *= al0; oacc[mt][1] *= al1;
        oacc[mt][2] *= al0; oacc[mt][3] *= al1;
      }
    }
    const float p0 = ex2_approx(fmaf(sc[0], sl2, -m0)), p1 = ex2_approx(fmaf(sc[1], sl2, -m1));
    const float p2 = ex2_approx(fmaf(sc[2], sl2, -m0)), p3 = ex2_approx(fmaf(sc[3], sl2, -m1));
    const uint32_t pb[2] = {movm_trans(pack_bf16x2(p0, p1)), movm_trans(pack_bf16x2(p2, p3))};
    mma_bf16_16816(lacc, ones, pb);  // l_h = sum_k P^T[k][h] (every row of the ones tile)
#pragma unroll
    for (int mt = 0; mt < KS; ++mt) mma_bf16_16816(oacc[mt], vf[mt], pb);
  };

  uint32_t j = 0;  // pages of the stream consumed
  for (int round = 0, item = gw; item < n_items; item = item_of(++round)) {
    const DecodeItem it = items[item];
    {  // next item's query rows into L1 while this item streams
      const int nx = item_of(round + 1);
      if (nx < n_items && lane < R) {
        const DecodeItem n2 = items[nx];
        asm volatile("prefetch.global.L1 [%0];" ::"l"(a.q + ((int64_t)n2.t * a.qh + (int64_t)n2.kvh * R + lane) * HD));
      }
    }
    const __nv_bfloat16* qbase = a.q + ((int64_t)it.t * a.qh + (int64_t)it.kvh * R) * HD;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int kc = ks * 16 + hc;
      qb[ks][0] = g < R ? *reinterpret_cast<const uint32_t*>(qbase + g * HD + kc) : 0u;
      qb[ks][1] = g < R ? *reinterpret_cast<const uint32_t*>(qbase + g * HD + kc + 8) : 0u;
    }
    float m0 = -INFINITY, m1 = -INFINITY;      // running max (log2 units) of head columns hc, hc+1
    float thr0 = -INFINITY, thr1 = -INFINITY;  // raw-score thresholds (m + 8) / scale of the lazy max
    float oacc[KS][4], lacc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int d = 0; d < KS; ++d) oacc[d][0] = oacc[d][1] = oacc[d][2] = oacc[d][3] = 0.f;

    const int np = (it.kv_len + 15) >> 4;
    if constexpr (LA == 2) {
      // S^T look-ahead: page p+1's K fragments and S^T MMAs are issued before page p's softmax
      // and P.V (independent chains in one warp's instruction stream); page p+1's V fragments
      // come in after page p's P.V, reusing page p's registers (one V set: 3 warps per SM
      // sub-partition still fit)
      float sc[4];
      uint32_t vf[KS][4];
      load_page(j, sc, vf);
      for (int p = 0; p < np; ++p, ++j) {
        float sn[4];
        const bool more = p + 1 < np;
        if (more) s_only(j + 1, sn);
        consume(p, np, it.kv_len, sc, vf, m0, m1, thr0, thr1, oacc, lacc);
        if (more) {
          v_only(j + 1, vf);
#pragma unroll
          for (int e = 0; e < 4; ++e) sc[e] = sn[e];
        }
      }
    } else if constexpr (LA == 0) {
      for (int p = 0; p < np; ++p, ++j) {
        float sc[4];
        uint32_t vf[KS][4];
        load_page(j, sc, vf);
        consume(p, np, it.kv_len, sc, vf, m0, m1, thr0, thr1, oacc, lacc);
      }
    } else {
      // look-ahead: page p+1's S^T chain is issued before page p's softmax and P.V, so the
      // two dependent chains of consecutive pages overlap (ping-pong register sets A / B)
      float scA[4], scB[4];
      uint32_t vA[KS][4], vB[KS][4];
      load_page(j, scA, vA);
      for (int p = 0;;) {
        if (p + 1 < np) load_page(j + 1, scB, vB);
        consume(p, np, it.kv_len, scA, vA, m0, m1, thr0, thr1, oacc, lacc);
        ++p, ++j;
        if (p >= np) break;
        if (p + 1 < np) load_page(j + 1, scA, vA);
        consume(p, np, it.kv_len, scB, vB, m0, m1, thr0, thr1, oacc, lacc);
        ++p, ++j;
        if (p >= np) break;
      }
    }
    const float i0 = 1.f / lacc[0], i1 = 1.f / lacc[1];
    __nv_bfloat16* obase = a.o + (int64_t)it.t * a.qh * HD + (int64_t)it.kvh * R * HD;
#pragma unroll
    for (int mt = 0; mt < KS; ++mt) {
      const int d0 = mt * 16 + g;
      if (hc < R) {
        obase[hc * HD + d0] = __float2bfloat16_rn(oacc[mt][0] * i0);
        obase[hc * HD + d0 + 8] = __float2bfloat16_rn(oacc[mt][2] * i0);
      }
      if (hc + 1 < R) {
        obase[(hc + 1) * HD + d0] = __float2bfloat16_rn(oacc[mt][1] * i1);
        obase[(hc + 1) * HD + d0 + 8] = __float2bfloat16_rn(oacc[mt][3] * i1);
      }
    }
  }
}

template <int HD, int W, int NS, int CH = 2, int LA = 0>
cudaError_t launch_stream_hdw(const CUtensorMap& pm, const AttnArgs& a, const DecodeItem* items, int n_items,
                              int grid, cudaStream_t st) {
  static_assert(ds_smem<HD, W, NS>() <= 232448, "shared memory");
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(decode_stream_kernel<HD, W, NS, CH, LA>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, ds_smem<HD, W, NS>());
    if (e != cudaSuccess) return e;
    attr = true;
  }
  decode_stream_kernel<HD, W, NS, CH, LA><<<grid, W * 32, ds_smem<HD, W, NS>(), st>>>(pm, a, items, n_items);
  count_launch();
  return cudaGetLastError();
}

// (dev) NF_DEC_STREAM_VAR: 1 = four S^T chains, 2 = page look-ahead (two V register sets), 3 = both,
// 4 / 5 = S^T look-ahead with one V register set (two / four chains) (A/B runs)
int decode_stream_var() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("NF_DEC_STREAM_VAR");
    v = e ? atoi(e) : 0;
    if (v < 0 || v > 5) v = 0;
  }
  return v;
}

}  // namespace

// Consumer warps per CTA at head_dim 128 and their ring depth (8 KB pages): 12 x 2 by
// default; NF_DEC_STREAM_WARPS (A/B runs) = 13 / 14 / 11 / 10 (x 2 pages), 9 / 8 (x 3), 7 / 6 (x 4).
int decode_stream_warps() {
  static int w = -1;
  if (w < 0) {
    const char* e = getenv("NF_DEC_STREAM_WARPS");
    w = e ? atoi(e) : 12;
    if (w != 13 && w != 14 && w != 11 && w != 10 && w != 9 && w != 8 && w != 7 && w != 6) w = 12;
  }
  return w;
}

bool decode_stream_supported(const AttnArgs& a) {
  return (a.hd == 128 || a.hd == 64) && a.page_size == 16 && a.kh > 0 && a.qh % a.kh == 0 && a.qh / a.kh <= 8;
}

cudaError_t launch_decode_attention_stream(const CUtensorMap& page_map, const AttnArgs& a, const DecodeItem* items,
                                           int n_items, int sm_budget, cudaStream_t st) {
  if (n_items <= 0) return cudaSuccess;
  if (!a.dec_rows || !a.dec_wstart || !decode_stream_supported(a)) return cudaErrorInvalidValue;
  // (an L2 prefetch of pages ahead of the ring, TMA or LSU, measured slower in every
  // configuration: profiles/r2f_decode_stream_l2_prefetch_ab.log, r2f_tma_probe_lsu.log)
  const AttnArgs& a2 = a;
  const int W = decode_stream_warps();
  const int grid = decode_grid(n_items, sm_budget, W);
  if (a.hd == 128) {
    const int v = decode_stream_var();
    if (v >= 4) {  // S^T look-ahead (4: two chains, 5: four chains)
      if (W == 12) return v == 4 ? launch_stream_hdw<128, 12, 2, 2, 2>(page_map, a2, items, n_items, grid, st)
                                 : launch_stream_hdw<128, 12, 2, 4, 2>(page_map, a2, items, n_items, grid, st);
      if (W == 8) return v == 4 ? launch_stream_hdw<128, 8, 3, 2, 2>(page_map, a2, items, n_items, grid, st)
                                : launch_stream_hdw<128, 8, 3, 4, 2>(page_map, a2, items, n_items, grid, st);
      return cudaErrorInvalidValue;
    }
    switch (W * 4 + v) {
      case 12 * 4 + 1: return launch_stream_hdw<128, 12, 2, 4, 0>(page_map, a2, items, n_items, grid, st);
      case 12 * 4 + 2: return launch_stream_hdw<128, 12, 2, 2, 1>(page_map, a2, items, n_items, grid, st);
      case 12 * 4 + 3: return launch_stream_hdw<128, 12, 2, 4, 1>(page_map, a2, items, n_items, grid, st);
      case 8 * 4 + 2: return launch_stream_hdw<128, 8, 3, 2, 1>(page_map, a2, items, n_items, grid, st);
      case 8 * 4 + 3: return launch_stream_hdw<128, 8, 3, 4, 1>(page_map, a2, items, n_items, grid, st);
      case 8 * 4 + 1: return launch_stream_hdw<128, 8, 3, 4, 0>(page_map, a2, items, n_items, grid, st);
      case 11 * 4: return launch_stream_hdw<128, 11, 2>(page_map, a2, items, n_items, grid, st);
      case 10 * 4: return launch_stream_hdw<128, 10, 2>(page_map, a2, items, n_items, grid, st);
      case 13 * 4: return launch_stream_hdw<128, 13, 2>(page_map, a2, items, n_items, grid, st);
      case 14 * 4: return launch_stream_hdw<128, 14, 2>(page_map, a2, items, n_items, grid, st);
      case 9 * 4: return launch_stream_hdw<128, 9, 3>(page_map, a2, items, n_items, grid, st);
      case 8 * 4: return launch_stream_hdw<128, 8, 3>(page_map, a2, items, n_items, grid, st);
      case 7 * 4: return launch_stream_hdw<128, 7, 4>(page_map, a2, items, n_items, grid, st);
      case 6 * 4: return launch_stream_hdw<128, 6, 4>(page_map, a2, items, n_items, grid, st);
      case 12 * 4: return launch_stream_hdw<128, 12, 2>(page_map, a2, items, n_items, grid, st);
      default: return cudaErrorInvalidValue;  // (dev) warps / variant combination not instantiated
    }
  }
  return launch_stream_hdw<64, 12, 4>(page_map, a2, items, n_items, grid, st);
}

// One kernel of this translation unit (preload_all_kernels: its module is loaded eagerly).
const void* kernel_anchor_decode_stream() { return reinterpret_cast<const void*>(decode_stream_kernel<128, 12, 2>); }

}  // namespace nf
