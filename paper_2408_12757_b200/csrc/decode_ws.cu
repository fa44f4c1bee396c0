// Warp-specialised paged GQA decode attention for sm_100a.
//
// Same math and smem layout as decode_attn_kernel (attention.cu: transposed
// formulation S^T = K Q^T on mma.sync m16n8k16, the GQA group's R <= 8 query heads
// as the MMA N columns, P^T by movmatrix, O^T += V^T P^T), but the TMA page loads
// of all consumer warps are issued by one producer warp: lane i of the producer
// drives consumer warp i's 2-slot ring (its item cursor, page-id prefetch and the
// 4-D page box), polling the ring's "empty" barriers.  A consumer warp's per-page
// work is then wait -> fragment pulls -> release -> math, with none of the
// loader bookkeeping (item switches, page-id windows, shuffles) on its critical
// chain: ncu showed ~220 issued instructions per 16-key page in the fused design,
// half of them loader overhead, with the SM issue-active 51 % and "wait" stalls
// dominating (profiles/r2_ncu_decode.md).
#include <algorithm>

#include "attention.cuh"
#include "common.cuh"
#include "profile.h"

namespace nf {
namespace {

constexpr int WS_BOX = 16 * 128;  // 16 rows x 64 bf16

NF_DEV uint32_t ws_swz(int row, int chunk) { return row * 128 + (((chunk & 7) ^ (row & 7)) << 4); }
NF_DEV uint32_t ws_ldg_u32(const __nv_bfloat16* p) { return *reinterpret_cast<const uint32_t*>(p); }
NF_DEV uint32_t ws_movm(uint32_t a) {
  uint32_t d;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(d) : "r"(a));
  return d;
}
NF_DEV bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

template <int HD, int CW>
constexpr int ws_smem() {
  return CW * 2 * (2 * 16 * HD * 2) + CW * 2 * 2 * 8 + 1024;
}

template <int HD, int CW>
__global__ void __launch_bounds__((CW + 1) * 32, 1)
    decode_ws_kernel(const __grid_constant__ CUtensorMap pages, const AttnArgs a,
                     const DecodeItem* __restrict__ items, int n_items) {
  constexpr int NBOX = HD / 64;
  constexpr int PAGE_BYTES = 16 * HD * 2;
  constexpr int STAGE_BYTES = 2 * PAGE_BYTES;
  constexpr int NS = 2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + CW * NS * STAGE_BYTES);  // [CW][NS]
  uint64_t* empty = full + CW * NS;                                          // [CW][NS]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&pages);
    for (int i = 0; i < CW * NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  // items sorted longest-first (host); consumer warp gw takes them in snake order,
  // warp-major across CTAs (LPT-like makespan; same order as decode_attn_kernel)
  const int TW = gridDim.x * CW;
  auto item_of = [&](int gw, int round) { return round * TW + ((round & 1) ? TW - 1 - gw : gw); };
  const int kh = a.kh, R = a.qh / a.kh;

  if (warp == CW) {
    // ---------------------------------------------------------------- producer warp
    const uint64_t pol = policy_evict_first();  // K/V pages are read once: keep L2 for the GEMMs
    const int gw = lane * gridDim.x + blockIdx.x;
    int round = 0, item = lane < CW ? item_of(gw, 0) : n_items;
    int np = 0, ps = 0, kvh = 0, p = 0;
    int pid0 = 0, pid1 = 0;                   // page ids of pages p, p + 1 of the current item
    DecodeItem nh{0, 0, 0, 0};                // header of the next item (prefetched)
    int nid0 = 0, nid1 = 0;                   // its first two page ids (prefetched near the end)
    bool nxt_ids = false;
    if (item < n_items) {
      const DecodeItem it = items[item];
      np = (it.kv_len + 15) >> 4;
      ps = it.page_start;
      kvh = it.kvh;
      pid0 = a.page_ids[ps];
      pid1 = np > 1 ? a.page_ids[ps + 1] : 0;
      const int ni = item_of(gw, 1);
      if (ni < n_items) nh = items[ni];
    }
    bool active = item < n_items;
    uint32_t issued = 0;
    while (__any_sync(0xffffffffu, active)) {
      bool progressed = false;
      if (active) {
        const int s = issued % NS;
        const uint32_t ph = (issued / NS) & 1;
        uint64_t* fb = &full[lane * NS + s];
        if (mbar_test(&empty[lane * NS + s], ph ^ 1)) {
          mbar_arrive_expect_tx(fb, STAGE_BYTES);
          tma_load_4d_hint(smem + (lane * NS + s) * STAGE_BYTES, &pages, fb, 0, ((pid0 * 2) * kh + kvh) * 16, 0, 0, pol);
          ++issued;
          ++p;
          progressed = true;
          pid0 = pid1;
          if (p + 1 < np) pid1 = a.page_ids[ps + p + 1];
          if (!nxt_ids && p + 2 >= np) {  // first page ids of the next item, two pages ahead
            const int nnp = (nh.kv_len + 15) >> 4;
            if (nnp > 0) {
              nid0 = a.page_ids[nh.page_start];
              nid1 = nnp > 1 ? a.page_ids[nh.page_start + 1] : 0;
            }
            nxt_ids = true;
          }
          if (p == np) {
            item = item_of(gw, ++round);
            if (item < n_items) {
              np = (nh.kv_len + 15) >> 4;
              ps = nh.page_start;
              kvh = nh.kvh;
              pid0 = nid0;
              pid1 = nid1;
              p = 0;
              nxt_ids = false;
              const int ni = item_of(gw, round + 1);
              if (ni < n_items) nh = items[ni];
              else nh = DecodeItem{0, 0, 0, 0};
            } else {
              active = false;
            }
          }
        }
      }
      if (!__any_sync(0xffffffffu, progressed)) __nanosleep(32);
    }
    return;
  }

  // ------------------------------------------------------------------ consumer warps
  const int gw = warp * gridDim.x + blockIdx.x;
  uint8_t* ring = smem + warp * NS * STAGE_BYTES;
  const float inv_scale = 1.f / a.scale_log2;
  const int hq = lane >> 2;       // query head of this lane's B-fragment column
  const int hc = 2 * (lane & 3);  // first of the two head columns this lane holds in C fragments
  uint32_t consumed = 0;
  for (int round = 0, item = item_of(gw, 0); item < n_items; item = item_of(gw, ++round)) {
    const DecodeItem it = items[item];
    const int kv_len = it.kv_len;
    const __nv_bfloat16* qbase = a.q + ((int64_t)it.t * a.qh + (int64_t)it.kvh * R) * HD;
    uint32_t qb[HD / 16][2];
#pragma unroll
    for (int ks = 0; ks < HD / 16; ++ks) {
      const int kc = ks * 16 + 2 * (lane & 3);
      qb[ks][0] = hq < R ? ws_ldg_u32(qbase + hq * HD + kc) : 0u;
      qb[ks][1] = hq < R ? ws_ldg_u32(qbase + hq * HD + kc + 8) : 0u;
    }
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
    float thr0 = -INFINITY, thr1 = -INFINITY;
    float oacc[HD / 16][4];
#pragma unroll
    for (int d = 0; d < HD / 16; ++d) oacc[d][0] = oacc[d][1] = oacc[d][2] = oacc[d][3] = 0.f;
    const int np = (kv_len + 15) >> 4;
    for (int p = 0; p < np; ++p) {
      const int s = consumed & 1;
      mbar_wait(&full[warp * NS + s], (consumed >> 1) & 1);
      uint8_t* kb = ring + s * STAGE_BYTES;
      uint8_t* vb = kb + PAGE_BYTES;
      if (p == np - 1 && kv_len - p * 16 < 16) {  // zero V rows of slots past kv_len
        const int valid = kv_len - p * 16;
        for (int i = lane; i < (16 - valid) * NBOX * 8; i += 32) {
          const int row = valid + i / (NBOX * 8), rem = i % (NBOX * 8);
          *reinterpret_cast<uint4*>(vb + (rem >> 3) * WS_BOX + row * 128 + (rem & 7) * 16) = make_uint4(0, 0, 0, 0);
        }
        __syncwarp();
      }
      float sacc[4][4];
      {
        uint32_t kf[HD / 16][4];
        const int key = (lane & 7) + (((lane >> 3) & 1) << 3);
        const int hi = lane >> 4;
#pragma unroll
        for (int ks = 0; ks < HD / 16; ++ks) {
          const int ch = ks * 2 + hi;
          ldmatrix_x4(kf[ks], smem_u32(kb) + (ch >> 3) * WS_BOX + ws_swz(key, ch));
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) sacc[c][0] = sacc[c][1] = sacc[c][2] = sacc[c][3] = 0.f;
#pragma unroll
        for (int ks = 0; ks < HD / 16; ++ks) mma_bf16_16816(sacc[ks & 3], kf[ks], qb[ks]);
      }
      uint32_t vf[HD / 16][4];
      {
        const int key = (lane & 7) + ((lane >> 4) << 3);
        const int hi = (lane >> 3) & 1;
#pragma unroll
        for (int mt = 0; mt < HD / 16; ++mt) {
          const int ch = mt * 2 + hi;
          ldmatrix_x4_trans(vf[mt], smem_u32(vb) + (ch >> 3) * WS_BOX + ws_swz(key, ch));
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[warp * NS + s]);  // the page is in registers: slot back to the producer
      ++consumed;
      float sc[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) sc[e] = (sacc[0][e] + sacc[1][e]) + (sacc[2][e] + sacc[3][e]);
      if (p == np - 1) {  // keys past kv_len only exist in the last page
        const int k0 = p * 16 + hq, k1 = k0 + 8;
        if (k0 >= kv_len) sc[0] = sc[1] = -INFINITY;
        if (k1 >= kv_len) sc[2] = sc[3] = -INFINITY;
      }
      // lazily updated running max (reading A-18; see decode_attn_kernel)
      if (__any_sync(0xffffffffu, fmaxf(sc[0], sc[2]) > thr0 || fmaxf(sc[1], sc[3]) > thr1)) {
        float r0 = fmaxf(sc[0], sc[2]), r1 = fmaxf(sc[1], sc[3]);
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
          r0 = fmaxf(r0, __shfl_xor_sync(0xffffffffu, r0, o));
          r1 = fmaxf(r1, __shfl_xor_sync(0xffffffffu, r1, o));
        }
        const float mn0 = fmaxf(m0, r0 * a.scale_log2), mn1 = fmaxf(m1, r1 * a.scale_log2);
        const float al0 = exp2f(m0 - mn0), al1 = exp2f(m1 - mn1);
        m0 = mn0;
        m1 = mn1;
        thr0 = (mn0 + 8.f) * inv_scale;
        thr1 = (mn1 + 8.f) * inv_scale;
        l0 *= al0;
        l1 *= al1;
#pragma unroll
        for (int mt = 0; mt < HD / 16; ++mt) {
          oacc[mt][0] *= al0; oacc[mt][1] *= al1;
          oacc[mt][2] *= al0; oacc[mt][3] *= al1;
        }
      }
      const float p0 = ex2_approx(fmaf(sc[0], a.scale_log2, -m0)), p1 = ex2_approx(fmaf(sc[1], a.scale_log2, -m1));
      const float p2 = ex2_approx(fmaf(sc[2], a.scale_log2, -m0)), p3 = ex2_approx(fmaf(sc[3], a.scale_log2, -m1));
      l0 += p0 + p2;
      l1 += p1 + p3;
      const uint32_t pb[2] = {ws_movm(pack_bf16x2(p0, p1)), ws_movm(pack_bf16x2(p2, p3))};
#pragma unroll
      for (int mt = 0; mt < HD / 16; ++mt) mma_bf16_16816(oacc[mt], vf[mt], pb);
    }
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      l0 += __shfl_xor_sync(0xffffffffu, l0, o);
      l1 += __shfl_xor_sync(0xffffffffu, l1, o);
    }
    const float i0 = 1.f / l0, i1 = 1.f / l1;
    __nv_bfloat16* obase = a.o + (int64_t)it.t * a.qh * HD + (int64_t)it.kvh * R * HD;
#pragma unroll
    for (int mt = 0; mt < HD / 16; ++mt) {
      const int d0 = mt * 16 + hq;
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

template <int HD, int CW>
cudaError_t launch_ws(const CUtensorMap& pm, const AttnArgs& a, const DecodeItem* items, int n_items, int sm_budget,
                      cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e =
        cudaFuncSetAttribute(decode_ws_kernel<HD, CW>, cudaFuncAttributeMaxDynamicSharedMemorySize, ws_smem<HD, CW>());
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int grid = std::min((n_items + CW - 1) / CW, std::max(sm_budget, 1));
  decode_ws_kernel<HD, CW><<<grid, (CW + 1) * 32, ws_smem<HD, CW>(), st>>>(pm, a, items, n_items);
  count_launch();
  return cudaGetLastError();
}

}  // namespace

// Warp-specialised decode (NF_DECODE_IMPL=ws): head_dim 128 with 12 consumer warps, 64 with 12.
cudaError_t launch_decode_attention_ws(const CUtensorMap& page_map, const AttnArgs& a, const DecodeItem* items,
                                       int n_items, int sm_budget, cudaStream_t st) {
  if (n_items <= 0) return cudaSuccess;
  static int env_w = -1;
  if (env_w < 0) {
    const char* e = getenv("NF_DEC_WS_WARPS");
    env_w = e ? atoi(e) : 12;
  }
  if (a.hd == 128) {
    if (env_w == 13) return launch_ws<128, 13>(page_map, a, items, n_items, sm_budget, st);
    if (env_w == 11) return launch_ws<128, 11>(page_map, a, items, n_items, sm_budget, st);
    if (env_w == 10) return launch_ws<128, 10>(page_map, a, items, n_items, sm_budget, st);
    return launch_ws<128, 12>(page_map, a, items, n_items, sm_budget, st);
  }
  if (a.hd == 64) return launch_ws<64, 12>(page_map, a, items, n_items, sm_budget, st);
  return cudaErrorInvalidValue;
}

// One kernel of this translation unit (preload_all_kernels: its module is loaded eagerly).
const void* kernel_anchor_decode_ws() { return reinterpret_cast<const void*>(decode_ws_kernel<128, 12>); }

}  // namespace nf
