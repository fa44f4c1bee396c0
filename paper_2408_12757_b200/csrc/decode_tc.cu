// tcgen05 paged GQA decode attention for sm_100a (head_dim 128, GQA group <= 8).
//
// PAPER.md:161 / :626 (decode attention, "memory-bound"); SURVEY.md §2C C2.
// Transposed formulation so that the long dimension (keys) is the MMA M:
//   S^T [128 keys x 16 heads] = K [128 keys x 128 dims] . Q^T       (tcgen05, f32 in TMEM)
//   O^T [128 dims x 16 heads] = V^T [128 dims x 128 keys] . P^T     (V read MN-major)
// The GQA group's R <= 8 query heads (padded to N = 16) share every K/V byte.
// One block = 128 keys = 8 pages.  K and V pages arrive by TMA (128B-swizzled
// 16-row boxes) laid out so that the block is directly a K-major operand (K)
// and an MN-major operand (V); no register staging of K/V at all.
//
// Warp roles (256 threads, 1 CTA per SM, persistent over (token, kv-head) items):
//   warp 0      : TMA producer (page ids prefetched per block by the whole warp)
//   warp 1 lane0: tcgen05.mma issuer; S of block j+1 is issued before PV of block j
//   warp 2      : TMEM allocator (64 columns: 2 S buffers + 2 O buffers)
//   warp 3      : Q loader (global -> swizzled smem B operand, double-buffered per item)
//   warps 4..7  : softmax (thread i <-> key i for S, dim i for O), online rescaling
#include <algorithm>

#include "attention.cuh"
#include "common.cuh"
#include "profile.h"

namespace nf {
namespace {

constexpr int TC_THREADS = 256;
constexpr int TC_BK = 128;                    // keys per block
constexpr int TC_PAGES = TC_BK / 16;          // pages per block
constexpr int TC_BOX = 16 * 128;              // one TMA box: 16 rows x 128 B
constexpr int TC_HALF = TC_PAGES * TC_BOX;    // 64-dim column of a K (or V) block: 16 KB
constexpr int TC_KV = 2 * TC_HALF;            // K (or V) block: 32 KB
constexpr int TC_STAGE = 2 * TC_KV;           // K + V block: 64 KB
constexpr int TC_OPB = 2 * 16 * 128;          // 16-row x 128-elem K-major SW128 operand (2 atoms): 4 KB
constexpr int TC_NS = 3;
constexpr int TC_NH = 16;                     // MMA N
constexpr int TC_RMAX = 8;                    // GQA group supported

constexpr int tc_smem() { return TC_NS * TC_STAGE + 2 * TC_OPB + 2 * TC_OPB + 2048 + 1024; }

NF_DEV uint64_t sdesc(uint32_t addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}

NF_DEV void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

NF_DEV float warp_max(float v) {
  float r;
  asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
  return r;
}

NF_DEV void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__global__ void __launch_bounds__(TC_THREADS, 1)
    decode_tc_kernel(const __grid_constant__ CUtensorMap pool, const AttnArgs a, const DecodeItem* __restrict__ items,
                     int n_items) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* kv = smem;                                   // [NS][K 32 KB | V 32 KB]
  uint8_t* qs = kv + TC_NS * TC_STAGE;                  // [2][4 KB]
  uint8_t* ps = qs + 2 * TC_OPB;                        // [2][4 KB]
  uint64_t* bar = reinterpret_cast<uint64_t*>(ps + 2 * TC_OPB);
  uint64_t* kv_full = bar;
  uint64_t* kv_empty = bar + TC_NS;
  uint64_t* q_full = bar + 2 * TC_NS;
  uint64_t* q_empty = q_full + 2;
  uint64_t* s_full = q_full + 4;
  uint64_t* s_free = q_full + 6;
  uint64_t* p_full = q_full + 8;
  uint64_t* p_free = q_full + 10;
  uint64_t* o_full = q_full + 12;
  uint64_t* o_free = q_full + 14;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_full + 16);
  float* red = reinterpret_cast<float*>(tmem_slot + 4);  // [2 parity][4 warps][8 heads] block maxima, then [4][8] sums

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kh = a.kh, R = a.qh / a.kh;
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&pool);
    for (int s = 0; s < TC_NS; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 4);
      mbar_init(&p_full[i], 4);
      mbar_init(&p_free[i], 1);
      mbar_init(&o_full[i], 1);
      mbar_init(&o_free[i], 4);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 64);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer (whole warp)
    const uint64_t pol = policy_evict_first();
    uint32_t blk = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const DecodeItem it = items[item];
      const int np = (it.kv_len + 15) >> 4;
      const int nb = (it.kv_len + TC_BK - 1) / TC_BK;
      for (int j = 0; j < nb; ++j, ++blk) {
        const int s = blk % TC_NS;
        const int npg = min(TC_PAGES, np - j * TC_PAGES);
        const int pid = lane < npg ? a.page_ids[it.page_start + j * TC_PAGES + lane] : 0;
        mbar_wait(&kv_empty[s], ((blk / TC_NS) & 1) ^ 1);
        if (lane == 0) mbar_arrive_expect_tx(&kv_full[s], npg * 4 * TC_BOX);
        __syncwarp();
        if (lane < npg) {
          const int rowK = (int)(((int64_t)pid * 2 * kh + it.kvh) * 16);
          const int rowV = rowK + kh * 16;
          uint8_t* kb = kv + s * TC_STAGE + lane * TC_BOX;
          tma_load_2d_hint(kb, &pool, &kv_full[s], 0, rowK, pol);
          tma_load_2d_hint(kb + TC_HALF, &pool, &kv_full[s], 64, rowK, pol);
          tma_load_2d_hint(kb + TC_KV, &pool, &kv_full[s], 0, rowV, pol);
          tma_load_2d_hint(kb + TC_KV + TC_HALF, &pool, &kv_full[s], 64, rowV, pol);
        }
        __syncwarp();
      }
    }
  } else if (warp == 3) {
    // ---------------------------------------------------------------- Q loader (whole warp)
    uint32_t qi = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++qi) {
      const DecodeItem it = items[item];
      const int qb = qi & 1;
      mbar_wait(&q_empty[qb], ((qi >> 1) & 1) ^ 1);
      uint8_t* qd = qs + qb * TC_OPB;
      const __nv_bfloat16* src = a.q + ((int64_t)it.t * a.qh + (int64_t)it.kvh * R) * 128;
      for (int e = lane; e < TC_NH * 16; e += 32) {  // 16 rows x 16 chunks of 16 B
        const int h = e >> 4, c = e & 15;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (h < R) v = *reinterpret_cast<const uint4*>(src + h * 128 + c * 8);
        *reinterpret_cast<uint4*>(qd + (c >> 3) * 2048 + h * 128 + (((c & 7) ^ (h & 7)) << 4)) = v;
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&q_full[qb]);
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------------------------------------------------------- MMA issuer
      constexpr uint32_t idS = idesc_bf16_f32(128, TC_NH);
      constexpr uint32_t idPV = idesc_bf16_f32(128, TC_NH) | (1u << 15);  // A (V^T) MN-major
      uint32_t blk = 0, qi = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++qi) {
        const DecodeItem it = items[item];
        const int nb = (it.kv_len + TC_BK - 1) / TC_BK;
        const int qb = qi & 1;
        mbar_wait(&q_full[qb], (qi >> 1) & 1);
        const uint32_t qaddr = smem_u32(qs + qb * TC_OPB);
        auto issue_S = [&](uint32_t b) {
          const int s = b % TC_NS, sb = b & 1;
          mbar_wait(&kv_full[s], (b / TC_NS) & 1);
          mbar_wait(&s_free[sb], ((b >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t kaddr = smem_u32(kv + s * TC_STAGE);
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            const uint64_t ad = sdesc(kaddr + (ks >> 2) * TC_HALF + (ks & 3) * 32, 16, 1024);
            const uint64_t bd = sdesc(qaddr + (ks >> 2) * 2048 + (ks & 3) * 32, 16, 1024);
            umma_bf16(tmem + sb * TC_NH, ad, bd, idS, ks > 0);
          }
          umma_commit(&s_full[sb]);
        };
        auto issue_PV = [&](uint32_t b) {
          const int s = b % TC_NS, pb = b & 1;
          mbar_wait(&p_full[pb], (b >> 1) & 1);
          mbar_wait(&o_free[pb], ((b >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t vaddr = smem_u32(kv + s * TC_STAGE + TC_KV);
          const uint32_t paddr = smem_u32(ps + pb * TC_OPB);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint64_t ad = sdesc(vaddr + kk * 2048, TC_HALF, 1024);   // 16 keys = 2 groups of 8 rows
            const uint64_t bd = sdesc(paddr + (kk >> 2) * 2048 + (kk & 3) * 32, 16, 1024);
            umma_bf16(tmem + 32 + pb * TC_NH, ad, bd, idPV, kk > 0);
          }
          umma_commit(&kv_empty[s]);
          umma_commit(&o_full[pb]);
          umma_commit(&p_free[pb]);
        };
        for (int j = 0; j < nb; ++j) {
          issue_S(blk + j);
          if (j == nb - 1) umma_commit(&q_empty[qb]);
          if (j > 0) issue_PV(blk + j - 1);
        }
        issue_PV(blk + nb - 1);
        blk += nb;
      }
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------------- softmax / output
    const int i = threadIdx.x - 128;       // key (S) or dim (O) of this thread
    const int w = warp - 4;
    const uint32_t lane_off = (uint32_t)(w * 32) << 16;
    uint32_t blk = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const DecodeItem it = items[item];
      const int nb = (it.kv_len + TC_BK - 1) / TC_BK;
      float m[TC_RMAX], l[TC_RMAX], o[TC_RMAX], al_prev[TC_RMAX];
#pragma unroll
      for (int h = 0; h < TC_RMAX; ++h) { m[h] = -INFINITY; l[h] = 0.f; o[h] = 0.f; al_prev[h] = 1.f; }
      auto accumulate_o = [&](uint32_t b, const float (&al)[TC_RMAX]) {
        const int ob = b & 1;
        mbar_wait(&o_full[ob], (b >> 1) & 1);
        tc_fence_after();
        uint32_t r[16];
        tmem_ld16(tmem + 32 + ob * TC_NH + lane_off, r);
        tmem_ld_wait();
#pragma unroll
        for (int h = 0; h < TC_RMAX; ++h) o[h] = fmaf(o[h], al[h], __uint_as_float(r[h]));
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&o_free[ob]);
      };
      for (int j = 0; j < nb; ++j) {
        const uint32_t b = blk + j;
        const int sb = b & 1;
        mbar_wait(&s_full[sb], (b >> 1) & 1);
        tc_fence_after();
        uint32_t r[16];
        tmem_ld16(tmem + sb * TC_NH + lane_off, r);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_free[sb]);
        const int valid = min(TC_BK, it.kv_len - j * TC_BK);
        float x[TC_RMAX];
#pragma unroll
        for (int h = 0; h < TC_RMAX; ++h) x[h] = i < valid ? __uint_as_float(r[h]) * a.scale_log2 : -INFINITY;
        // block max per head: warp redux, then across the 4 softmax warps
        float* rb = red + (b & 1) * 32;
#pragma unroll
        for (int h = 0; h < TC_RMAX; ++h) {
          const float wm = warp_max(x[h]);
          if (lane == h) rb[w * 8 + h] = wm;
        }
        named_bar(1, 128);
        float al[TC_RMAX], p[TC_RMAX];
#pragma unroll
        for (int h = 0; h < TC_RMAX; ++h) {
          const float mb = fmaxf(fmaxf(rb[h], rb[8 + h]), fmaxf(rb[16 + h], rb[24 + h]));
          const float mn = fmaxf(m[h], mb);
          al[h] = exp2f(m[h] - mn);
          p[h] = exp2f(x[h] - mn);
          l[h] = fmaf(l[h], al[h], p[h]);
          m[h] = mn;
        }
        const int s = b % TC_NS, pb = b & 1;
        if (i >= valid) {  // zero this key's V row (slots past kv_len may hold anything, 0*NaN = NaN)
          uint8_t* vrow = kv + s * TC_STAGE + TC_KV + (i >> 4) * TC_BOX + (i & 15) * 128;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            *reinterpret_cast<uint4*>(vrow + c * 16) = make_uint4(0, 0, 0, 0);
            *reinterpret_cast<uint4*>(vrow + TC_HALF + c * 16) = make_uint4(0, 0, 0, 0);
          }
        }
        mbar_wait(&p_free[pb], ((b >> 1) & 1) ^ 1);
        uint8_t* pd = ps + pb * TC_OPB + (i >> 6) * 2048;
        const int kc = (i & 63) >> 3, ke = (i & 7) * 2;
#pragma unroll
        for (int h = 0; h < TC_NH; ++h) {
          const float v = h < R && h < TC_RMAX ? p[h < TC_RMAX ? h : 0] : 0.f;
          *reinterpret_cast<__nv_bfloat16*>(pd + h * 128 + ((kc ^ (h & 7)) << 4) + ke) = __float2bfloat16_rn(v);
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[pb]);
        if (j > 0) accumulate_o(b - 1, al_prev);
#pragma unroll
        for (int h = 0; h < TC_RMAX; ++h) al_prev[h] = al[h];
      }
      accumulate_o(blk + nb - 1, al_prev);
      blk += nb;
      // total l per head across the 128 threads
      float* rs = red + 64;
#pragma unroll
      for (int h = 0; h < TC_RMAX; ++h) {
        float v = l[h];
#pragma unroll
        for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if (lane == h) rs[w * 8 + h] = v;
      }
      named_bar(1, 128);
      __nv_bfloat16* obase = a.o + ((int64_t)it.t * a.qh + (int64_t)it.kvh * R) * 128;
#pragma unroll
      for (int h = 0; h < TC_RMAX; ++h) {
        if (h < R) {
          const float L = rs[h] + rs[8 + h] + rs[16 + h] + rs[24 + h];
          obase[h * 128 + i] = __float2bfloat16_rn(o[h] / L);
        }
      }
      named_bar(1, 128);  // rs reused by the next item
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 64);
  }
}

}  // namespace

cudaError_t launch_decode_attention_tc(const CUtensorMap& m, const AttnArgs& a, const DecodeItem* items, int n_items,
                                       int sm_budget, cudaStream_t st) {
  if (n_items <= 0) return cudaSuccess;
  if (a.hd != 128 || a.qh / a.kh > TC_RMAX) return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(decode_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tc_smem());
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int grid = std::min(n_items, std::max(sm_budget, 1));
  decode_tc_kernel<<<grid, TC_THREADS, tc_smem(), st>>>(m, a, items, n_items);
  count_launch();
  return cudaGetLastError();
}

// One kernel of this translation unit (preload_all_kernels: its module is loaded eagerly).
const void* kernel_anchor_decode_tc() { return reinterpret_cast<const void*>(decode_tc_kernel); }

}  // namespace nf
