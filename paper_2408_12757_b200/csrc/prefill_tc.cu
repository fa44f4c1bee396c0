// tcgen05 causal paged prefill attention for sm_100a (head_dim 128).
//
// PAPER.md:161 (attention of a prefill chunk over its cached prefix + itself),
// :437 (prefill attention is compute-bound; the paper saw launch overhead
// dominate), SURVEY.md §8a a5.  One work item = 128 query rows of one request
// chunk and one query head; keys are streamed in 128-key blocks (8 pages):
//   S  [128 q x 128 keys] = Q . K^T            (tcgen05, f32 in TMEM, 2 buffers)
//   O  [128 q x 128 dims] += P . V             (P bf16 written by the softmax warps to TMEM,
//                                               V read MN-major straight from its pages)
// Causal mask key <= pos(row); blocks past the tile's last position are never loaded.
//
// Warp roles (256 threads, 1 CTA per SM, persistent over items, longest first):
//   warp 0      : K producer (TMA, 3-stage ring freed when S is done; lane p loads page p)
//   warp 1 lane0: tcgen05.mma issuer; S of block j+1 is issued before PV of block j;
//                 PV reads P from tensor memory (TS form), V from smem (MN-major)
//   warp 2      : TMEM allocator (512 columns: S0 | S1 | O | P), then V producer (2-stage ring)
//   warp 3      : Q loader (TMA, 3-D map over q [T, qh, hd] -> K-major SW128 operand, 2 buffers)
//   warps 4..11 : softmax, two warps per TMEM lane quarter: row i = 32*(warp%4) + lane,
//                 each warp of the pair owns 64 of the 128 keys / O columns; the pair
//                 combines row maxima through smem, everything else is thread-local.
//                 The running max is updated lazily (only when a row max grows by
//                 > 2^8), so the O row rescale through TMEM (ld, scale, st) is rare.
#include <algorithm>

#include "attention.cuh"
#include "common.cuh"
#include "profile.h"

namespace nf {
namespace {

constexpr int PT_THREADS = 384;             // 4 role warps + 8 softmax warps (2 per TMEM lane quarter)
constexpr int PT_BK = 128;                  // keys per block
constexpr int PT_PAGES = PT_BK / 16;        // pages per block
constexpr int PT_BOX = 16 * 128;            // one TMA box: 16 rows x 128 B (64 bf16)
constexpr int PT_HALF = 128 * 128;          // 128 rows x 64 cols (one 128B-swizzled column half): 16 KB
constexpr int PT_OPND = 2 * PT_HALF;        // 128 x 128 bf16 operand: 32 KB
constexpr int PT_KS = 3, PT_VS = 2;         // K / V block stages (separate rings: K frees after S, V after PV)
constexpr int PT_COL_S = 0, PT_COL_O = 256, PT_COL_P = 384;  // TMEM: S0 | S1 | O | P (bf16 pairs, 64 cols)

// operands (1024-aligned dynamic smem, checked at run time) + barriers + the pair exchange buffer
constexpr int pt_smem() { return (PT_KS + PT_VS + 2) * PT_OPND + 512 + 2 * 2 * 128 * 4; }

NF_DEV uint64_t sdesc(uint32_t addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}

NF_DEV void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
NF_DEV void named_bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
NF_DEV void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// D[tmem] (+)= A[tmem] * B[smem]: A (P, bf16 pairs) read from tensor memory
NF_DEV void umma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

struct ItemGeom {
  int nb;       // key blocks
  int kv_need;  // keys any row of the tile can see: pos0 + n
};
NF_DEV ItemGeom geom(const PrefillItem& it) {
  ItemGeom g;
  g.kv_need = it.pos0 + it.n;
  g.nb = (g.kv_need + PT_BK - 1) / PT_BK;
  return g;
}

// Items are sorted longest first (host); CTA b takes them in snake order (round k:
// k*G + b, or k*G + G-1-b for odd k) so the per-CTA block counts even out.
NF_DEV int item_at(int round) {
  return round * gridDim.x + ((round & 1) ? gridDim.x - 1 - blockIdx.x : blockIdx.x);
}

__global__ void __launch_bounds__(PT_THREADS, 1)
    prefill_tc_kernel(const __grid_constant__ CUtensorMap pool, const __grid_constant__ CUtensorMap qmap,
                      const AttnArgs a, const PrefillItem* __restrict__ items, int n_items) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if (threadIdx.x == 0 && (smem_u32(smem) & 1023) != 0) __trap();  // SW128 operands need 1024-B alignment
  uint8_t* ks = smem;                       // [KS][K block 32 KB]
  uint8_t* vs = ks + PT_KS * PT_OPND;       // [VS][V block 32 KB]
  uint8_t* qs = vs + PT_VS * PT_OPND;       // [2][Q tile 32 KB]
  uint64_t* bar = reinterpret_cast<uint64_t*>(qs + 2 * PT_OPND);
  uint64_t* k_full = bar;                   // [KS]
  uint64_t* k_empty = k_full + PT_KS;       // [KS]
  uint64_t* v_full = k_empty + PT_KS;       // [VS]
  uint64_t* v_empty = v_full + PT_VS;       // [VS]
  uint64_t* q_full = v_empty + PT_VS;       // [2]
  uint64_t* q_empty = q_full + 2;           // [2]
  uint64_t* s_full = q_full + 4;            // [2]
  uint64_t* s_free = q_full + 6;            // [2]
  uint64_t* p_full = q_full + 8;
  uint64_t* p_free = q_full + 9;
  uint64_t* o_full = q_full + 10;
  uint64_t* o_free = q_full + 11;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_full + 12);
  float* xchg = reinterpret_cast<float*>(q_full + 32);  // [2 block parities][2 halves][128 rows]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kh = a.kh, R = a.qh / a.kh;
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&pool);
    tma_prefetch_desc(&qmap);
    for (int s = 0; s < PT_KS; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < PT_VS; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 8);
    }
    mbar_init(p_full, 8);
    mbar_init(p_free, 1);
    mbar_init(o_full, 1);
    mbar_init(o_free, 8);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 || warp == 2) {
    // ---------------------------------------------------------------- TMA producers (whole warps):
    // warp 0 streams K blocks, warp 2 V blocks; lane p loads page p of a block (two 64-column boxes)
    const bool isK = warp == 0;
    const int NS = isK ? PT_KS : PT_VS;
    uint8_t* ring = isK ? ks : vs;
    uint64_t* full = isK ? k_full : v_full;
    uint64_t* empty = isK ? k_empty : v_empty;
    const uint64_t pol = policy_evict_last();  // a block is re-read by the other R-1 query heads / later tiles
    uint32_t blk = 0;
    for (int round = 0, item = item_at(0); item < n_items; item = item_at(++round)) {
      const PrefillItem it = items[item];
      const ItemGeom g = geom(it);
      const int np = (g.kv_need + 15) >> 4;
      const int row0 = (it.h / R) * 16 + (isK ? 0 : kh * 16);
      for (int j = 0; j < g.nb; ++j, ++blk) {
        const int s = blk % NS;
        const int npg = min(PT_PAGES, np - j * PT_PAGES);
        const int pid = lane < npg ? a.page_ids[it.page_start + j * PT_PAGES + lane] : 0;
        mbar_wait(&empty[s], ((blk / NS) & 1) ^ 1);
        if (lane == 0) mbar_arrive_expect_tx(&full[s], npg * 2 * PT_BOX);
        __syncwarp();
        if (lane < npg) {
          const int row = (int)((int64_t)pid * 2 * kh * 16 + row0);
          uint8_t* dst = ring + s * PT_OPND + lane * PT_BOX;
          tma_load_2d_hint(dst, &pool, &full[s], 0, row, pol);
          tma_load_2d_hint(dst + PT_HALF, &pool, &full[s], 64, row, pol);
        }
        __syncwarp();
      }
    }
  } else if (warp == 3) {
    // ---------------------------------------------------------------- Q loader (TMA: 128 token rows of
    // head h, two 64-column boxes; rows past T are zero-filled, rows of other requests are masked)
    if (lane == 0) {
      uint32_t qi = 0;
      for (int round = 0, item = item_at(0); item < n_items; item = item_at(++round), ++qi) {
        const PrefillItem it = items[item];
        const int qb = qi & 1;
        mbar_wait(&q_empty[qb], ((qi >> 1) & 1) ^ 1);
        uint8_t* qd = qs + qb * PT_OPND;
        mbar_arrive_expect_tx(&q_full[qb], PT_OPND);
        tma_load_3d(qd, &qmap, &q_full[qb], 0, it.h, it.t0);
        tma_load_3d(qd + PT_HALF, &qmap, &q_full[qb], 64, it.h, it.t0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------------------------------------------------------- MMA issuer
      constexpr uint32_t idS = idesc_bf16_f32(128, 128);
      constexpr uint32_t idPV = idesc_bf16_f32(128, 128) | (1u << 16);  // B (V) MN-major
      uint32_t blk = 0, qi = 0;
      for (int round = 0, item = item_at(0); item < n_items; item = item_at(++round), ++qi) {
        const PrefillItem it = items[item];
        const ItemGeom g = geom(it);
        const int qb = qi & 1;
        mbar_wait(&q_full[qb], (qi >> 1) & 1);
        const uint32_t qaddr = smem_u32(qs + qb * PT_OPND);
        auto issue_S = [&](uint32_t b) {
          const int s = b % PT_KS, sb = b & 1;
          mbar_wait(&k_full[s], (b / PT_KS) & 1);
          mbar_wait(&s_free[sb], ((b >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t kaddr = smem_u32(ks + s * PT_OPND);
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint32_t off = (k >> 2) * PT_HALF + (k & 3) * 32;
            umma_bf16(tmem + PT_COL_S + sb * 128, sdesc(qaddr + off, 16, 1024), sdesc(kaddr + off, 16, 1024), idS,
                      k > 0);
          }
          umma_commit(&k_empty[s]);
          umma_commit(&s_full[sb]);
        };
        auto issue_PV = [&](uint32_t b, bool first) {
          const int s = b % PT_VS;
          mbar_wait(&v_full[s], (b / PT_VS) & 1);
          mbar_wait(p_full, b & 1);
          if (first) mbar_wait(o_free, (qi & 1) ^ 1);
          tc_fence_after();
          const uint32_t vaddr = smem_u32(vs + s * PT_OPND);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint64_t bd = sdesc(vaddr + kk * 2048, PT_HALF, 1024);  // 16 keys = 2 groups of 8 rows
            umma_bf16_ts(tmem + PT_COL_O, tmem + PT_COL_P + kk * 8, bd, idPV, (first && kk == 0) ? 0u : 1u);
          }
          umma_commit(&v_empty[s]);
          umma_commit(p_free);
        };
        for (int j = 0; j < g.nb; ++j) {
          issue_S(blk + j);
          if (j == g.nb - 1) umma_commit(&q_empty[qb]);
          if (j > 0) issue_PV(blk + j - 1, j == 1);
        }
        issue_PV(blk + g.nb - 1, g.nb == 1);
        umma_commit(o_full);
        blk += g.nb;
      }
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------------- softmax / output
    // Two warps per TMEM lane quarter: row i = 32*(warp%4) + lane; half hf owns keys / O columns
    // [64 hf, 64 hf + 64).  The pair combines its row maxima through shared memory (one 64-thread
    // named barrier per block); row sums stay per half until the output.
    const int qd = warp & 3, hf = (warp - 4) >> 2;
    const int i = qd * 32 + lane;
    const uint32_t lane_off = (uint32_t)(qd * 32) << 16;
    const int bar_id = 1 + qd;
    uint32_t blk = 0, qi = 0;
    for (int round = 0, item = item_at(0); item < n_items; item = item_at(++round), ++qi) {
      const PrefillItem it = items[item];
      const ItemGeom g = geom(it);
      const bool row_ok = i < it.n;
      const int pos = it.pos0 + i;  // keys 0..pos visible to this row
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j < g.nb; ++j) {
        const uint32_t b = blk + j;
        const int sb = b & 1;
        mbar_wait(&s_full[sb], (b >> 1) & 1);
        tc_fence_after();
        uint32_t x[64];  // raw S bits of this row's 64 keys
        {
          uint32_t r0[32], r1[32];
          tmem_ld32(tmem + PT_COL_S + sb * 128 + hf * 64 + lane_off, r0);
          tmem_ld32(tmem + PT_COL_S + sb * 128 + hf * 64 + 32 + lane_off, r1);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            x[e] = r0[e];
            x[32 + e] = r1[e];
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_free[sb]);
        const int k0 = j * PT_BK + hf * 64;
        const int lim = row_ok ? pos - k0 : -1;  // visible keys of this half block: e <= lim
        const bool full = lim >= 63;
        float mx8[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) mx8[u] = -INFINITY;
        if (full) {
#pragma unroll
          for (int e = 0; e < 64; ++e) mx8[e & 7] = fmaxf(mx8[e & 7], __uint_as_float(x[e]));
        } else {
#pragma unroll
          for (int e = 0; e < 64; ++e)
            if (e <= lim) mx8[e & 7] = fmaxf(mx8[e & 7], __uint_as_float(x[e]));
        }
        float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                         fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
        float* xb = xchg + (b & 1) * 256;
        xb[hf * 128 + i] = mx;
        named_bar_sync(bar_id, 64);
        mx = fmaxf(mx, xb[(hf ^ 1) * 128 + i]) * a.scale_log2;  // identical in both halves
        const bool need = mx > m + 8.f;
        float al = 1.f;
        if (need) {
          al = exp2f(m - mx);  // 0 on the first visible block (m = -inf)
          m = mx;
          l *= al;
        }
        const float mref = m == -INFINITY ? 0.f : m;
        // p = 2^(s*scale - m): one FFMA + one MUFU.EX2 per key, masked keys 0
        float rs8[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) rs8[u] = 0.f;
        uint32_t pk[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          float p0 = ex2_approx(fmaf(__uint_as_float(x[2 * e]), a.scale_log2, -mref));
          float p1 = ex2_approx(fmaf(__uint_as_float(x[2 * e + 1]), a.scale_log2, -mref));
          if (!full) {
            p0 = 2 * e <= lim ? p0 : 0.f;
            p1 = 2 * e + 1 <= lim ? p1 : 0.f;
          }
          rs8[e & 7] += p0 + p1;
          pk[e] = pack_bf16x2(p0, p1);
        }
        l += ((rs8[0] + rs8[1]) + (rs8[2] + rs8[3])) + ((rs8[4] + rs8[5]) + (rs8[6] + rs8[7]));
        // V rows of keys no row of this tile sees: zero (slots past the context may hold NaN);
        // this half zeroes its 64 columns of key row i
        if (j * PT_BK + PT_BK > g.kv_need) {
          const int sv = b % PT_VS;
          mbar_wait(&v_full[sv], (b / PT_VS) & 1);
          if (j * PT_BK + i >= g.kv_need) {
            uint8_t* vrow = vs + sv * PT_OPND + hf * PT_HALF + i * 128;
#pragma unroll
            for (int c = 0; c < 8; ++c) *reinterpret_cast<uint4*>(vrow + c * 16) = make_uint4(0, 0, 0, 0);
          }
          fence_proxy_async();
        }
        // PV of the previous block has finished: the P columns and O are ours
        mbar_wait(p_free, (b & 1) ^ 1);
        tc_fence_after();
        if (__any_sync(0xffffffffu, need) && j > 0) {  // warp-collective TMEM access; al = 1 for other rows
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            uint32_t r[32];
            tmem_ld32(tmem + PT_COL_O + hf * 64 + c * 32 + lane_off, r);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * al);
            tmem_st32(tmem + PT_COL_O + hf * 64 + c * 32 + lane_off, r);
          }
        }
        tmem_st32(tmem + PT_COL_P + hf * 32 + lane_off, pk);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full);
      }
      blk += g.nb;
      // output: O / (l_half0 + l_half1), each half writes its 64 columns.  The sums go
      // through the exchange slot of the parity after the last block's (its reads are done)
      float* xl = xchg + (blk & 1) * 256;
      xl[hf * 128 + i] = l;
      named_bar_sync(bar_id, 64);
      const float L = l + xl[(hf ^ 1) * 128 + i];
      mbar_wait(o_full, qi & 1);
      tc_fence_after();
      const float inv = row_ok ? 1.f / L : 0.f;
      __nv_bfloat16* orow = a.o + ((int64_t)(it.t0 + (row_ok ? i : 0)) * a.qh + it.h) * 128 + hf * 64;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t r[32];
        tmem_ld32(tmem + PT_COL_O + hf * 64 + c * 32 + lane_off, r);
        tmem_ld_wait();
        if (row_ok) {
          uint4* d = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            d[q] = make_uint4(pack_bf16x2(__uint_as_float(r[8 * q]) * inv, __uint_as_float(r[8 * q + 1]) * inv),
                              pack_bf16x2(__uint_as_float(r[8 * q + 2]) * inv, __uint_as_float(r[8 * q + 3]) * inv),
                              pack_bf16x2(__uint_as_float(r[8 * q + 4]) * inv, __uint_as_float(r[8 * q + 5]) * inv),
                              pack_bf16x2(__uint_as_float(r[8 * q + 6]) * inv, __uint_as_float(r[8 * q + 7]) * inv));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(o_free);
      named_bar_sync(bar_id, 64);  // xl is rewritten by the next item
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace

cudaError_t launch_prefill_attention_tc(const CUtensorMap& m, const AttnArgs& a, const PrefillItem* items, int n_items,
                                        int sm_budget, cudaStream_t st) {
  if (n_items <= 0) return cudaSuccess;
  if (a.hd != 128) return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(prefill_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, pt_smem());
    if (e != cudaSuccess) return e;
    attr = true;
  }
  CUtensorMap qm;
  cudaError_t e = make_q_tmap(&qm, a.q, a.n_rows, a.qh, 128);
  if (e != cudaSuccess) return e;
  const int grid = std::min(n_items, std::max(sm_budget, 1));
  prefill_tc_kernel<<<grid, PT_THREADS, pt_smem(), st>>>(m, qm, a, items, n_items);
  count_launch();
  return cudaGetLastError();
}

// One kernel of this translation unit (preload_all_kernels: its module is loaded eagerly).
const void* kernel_anchor_prefill_tc() { return reinterpret_cast<const void*>(prefill_tc_kernel); }

}  // namespace nf
