// Paged GQA attention for sm_100a.
//
// KV pool layout [n_pages][2][kv_heads][16][head_dim] bf16: the
// K (or V) block of one page and one KV head is 16 contiguous rows, fetched by
// TMA as 128B-swizzled boxes of 16 rows x 64 columns into shared memory, so
// the mma.sync fragment loads (ldmatrix) are bank-conflict free.
//
// Decode: one warp per (decode token, KV head) item; the R = qh/kh query heads
// of the group are the M rows of m16n8k16 tensor-core MMAs, so each K/V byte
// read from HBM is used R times on the tensor pipe (HBM-bound by design).
// Every warp runs its own NS-deep TMA ring that streams ahead across items.
// Prefill: FlashAttention-2 style, one CTA per (64-query tile, query head),
// double-buffered 64-key K/V tiles, causal mask j <= pos.
#include <algorithm>
#include <string>

#include "attention.cuh"
#include "common.cuh"
#include "profile.h"

namespace nf {

cudaError_t make_tmap_bf16(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld_elems,
                           uint32_t box_inner, uint32_t box_outer);

cudaError_t make_pool_tmap(CUtensorMap* m, const void* pool, int64_t n_pages, int kh, int hd, int page_size) {
  return make_tmap_bf16(m, pool, hd, (uint64_t)n_pages * 2 * kh * page_size, hd, 64, page_size);
}

namespace {

constexpr int BOX_BYTES = 16 * 128;  // 16 rows x 64 bf16

NF_DEV uint32_t swz(int row, int chunk) { return row * 128 + (((chunk & 7) ^ (row & 7)) << 4); }

NF_DEV uint32_t ldg_u32(const __nv_bfloat16* p) { return *reinterpret_cast<const uint32_t*>(p); }

template <int HD, int DEC_WARPS>
constexpr int dec_stages() {
  // per-page compute (~1.3 us) exceeds HBM latency (~0.9 us, tools/tma_probe.py), so two stages per
  // warp suffice and the smem goes to more warps (more pages in flight per SM)
  return HD == 128 ? (DEC_WARPS >= 12 ? 2 : DEC_WARPS == 8 ? 3 : DEC_WARPS == 6 ? 4 : 2)
                   : (DEC_WARPS >= 12 ? 4 : DEC_WARPS == 8 ? 6 : DEC_WARPS == 6 ? 8 : 4);
}

template <int HD, int DEC_WARPS>
constexpr int dec_smem() {
  return DEC_WARPS * dec_stages<HD, DEC_WARPS>() * (2 * 16 * HD * 2) + DEC_WARPS * dec_stages<HD, DEC_WARPS>() * 8 + 1024;
}

// ---------------------------------------------------------------------------- decode
// Transposed formulation: S^T[16 keys x 8 heads] = K[16 x hd] . Q^T[hd x 8]
// (m16n8k16: the page's 16 keys are the M rows, the GQA group's R <= 8 query
// heads the N columns), then O^T[hd x 8] += V^T[hd x 16] . P^T[16 x 8] with P^T
// turned into a B fragment in registers by movmatrix.  16 MMAs per 16-key page.
NF_DEV uint32_t movmatrix_trans(uint32_t a) {
  uint32_t d;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(d) : "r"(a));
  return d;
}

// ROWS: the loader streams precomputed TMA rows (a.dec_rows / a.dec_wstart: the warp's
// pages in consumption order across its items) instead of walking item headers and
// page-id windows -- the loader bookkeeping was ~1/4 of the issued instructions per page
// (profiles/r2_ncu_decode.md).
template <int HD, int DEC_WARPS, bool ROWS = false>
__global__ void __launch_bounds__(DEC_WARPS * 32)
    decode_attn_kernel(const __grid_constant__ CUtensorMap pool, const __grid_constant__ CUtensorMap pages,
                       const AttnArgs a,
                       const DecodeItem* __restrict__ items, int n_items) {
  constexpr int NBOX = HD / 64;
  constexpr int PAGE_BYTES = 16 * HD * 2;
  constexpr int STAGE_BYTES = 2 * PAGE_BYTES;
  constexpr int NS = dec_stages<HD, DEC_WARPS>();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = smem + warp * NS * STAGE_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + DEC_WARPS * NS * STAGE_BYTES) + warp * NS;
  if (lane == 0) {
    if (warp == 0) tma_prefetch_desc(&pages);
    for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
    fence_barrier_init();
  }
  __syncwarp();

  // Items are sorted longest-first (host); warps take them in snake order
  // (round k: k*TW + gw, or k*TW + TW-1-gw for odd k) and warp-major across
  // CTAs, so every SM gets a mix of lengths and the second round's short items
  // go to the warps whose first item was shortest (LPT-like makespan).
  const int gw = warp * gridDim.x + blockIdx.x, TW = gridDim.x * DEC_WARPS;
  auto item_of = [&](int round) { return round * TW + ((round & 1) ? TW - 1 - gw : gw); };
  const int kh = a.kh, R = a.qh / a.kh;

  // Look-ahead loader cursor (warp-uniform) with a 32-entry window of page ids
  // (one per lane).  Metadata is software-pipelined across item switches so no
  // load is consumed right after it is issued: at a switch the next item's
  // header (loaded one switch earlier) becomes current, the item after it gets
  // its first page-id window, and the header two items ahead is requested;
  // within an item the following 32-page window is loaded 32 pages ahead.
  struct Hdr { int np, ps, kvh; };
  auto header = [&](int item) {
    Hdr h{0, 0, 0};
    if (item < n_items) {
      const DecodeItem it = items[item];
      h.np = (it.kv_len + 15) >> 4;
      h.ps = it.page_start;
      h.kvh = it.kvh;
    }
    return h;
  };
  auto window = [&](const Hdr& h, int first) {
    return first + lane < h.np ? a.page_ids[h.ps + first + lane] : 0;
  };
  int l_round = 0, l_item = gw, l_page = 0;
  Hdr cur{0, 0, 0}, nxt{0, 0, 0}, nn{0, 0, 0};
  int pid_win = 0, pid_nwin = 0, n_win = 0;
  // ROWS loader state: position in the warp's row stream and two 32-row windows
  int r_pos = 0, r_len = 0, r_base = 0, r_win = 0, r_nwin = 0;
  if constexpr (ROWS) {
    r_base = a.dec_wstart[gw];
    r_len = a.dec_wstart[gw + 1] - r_base;
    r_win = lane < r_len ? a.dec_rows[r_base + lane] : 0;
    r_nwin = 32 + lane < r_len ? a.dec_rows[r_base + 32 + lane] : 0;
  } else {
    cur = header(l_item);
    nxt = header(item_of(1));
    nn = header(item_of(2));
    pid_win = window(cur, 0);
    pid_nwin = window(cur, 32);
    n_win = window(nxt, 0);
  }
  uint32_t issued = 0, consumed = 0;
  const uint64_t kv_policy = policy_evict_first();  // K/V pages are read exactly once: keep L2 for the GEMMs
  auto issue_one = [&]() {
    if constexpr (ROWS) {
      if (r_pos >= r_len) return;
      const int s = issued % NS;
      const int rowK = __shfl_sync(0xffffffffu, r_win, r_pos & 31);
      if (lane == 0) {
        fence_proxy_async();  // WAR: this warp's ldmatrix reads of the slot before the async-proxy refill
        mbar_arrive_expect_tx(&bars[s], STAGE_BYTES);
        tma_load_4d_hint(ring + s * STAGE_BYTES, &pages, &bars[s], 0, rowK, 0, 0, kv_policy);
      }
      ++issued;
      if ((++r_pos & 31) == 0) {
        r_win = r_nwin;
        r_nwin = r_pos + 32 + lane < r_len ? a.dec_rows[r_base + r_pos + 32 + lane] : 0;
      }
      return;
    }
    if (l_item >= n_items) return;
    const int s = issued % NS;
    const int64_t page = __shfl_sync(0xffffffffu, pid_win, l_page & 31);
    if (lane == 0) {
      uint8_t* dst = ring + s * STAGE_BYTES;
      const int rowK = (int)(((page * 2 + 0) * kh + cur.kvh) * 16);
      fence_proxy_async();  // WAR: this warp's ldmatrix reads of the slot before the async-proxy refill
      mbar_arrive_expect_tx(&bars[s], STAGE_BYTES);
      tma_load_4d_hint(dst, &pages, &bars[s], 0, rowK, 0, 0, kv_policy);  // K and V of the page: one 4-D box
    }
    ++issued;
    if (++l_page == cur.np) {
      l_item = item_of(++l_round);
      l_page = 0;
      cur = nxt;
      pid_win = n_win;
      pid_nwin = window(cur, 32);
      nxt = nn;
      n_win = window(nxt, 0);
      nn = header(item_of(l_round + 2));
    } else if ((l_page & 31) == 0) {
      pid_win = pid_nwin;
      pid_nwin = window(cur, l_page + 32);
    }
  };
  for (int i = 0; i < NS; ++i) issue_one();

  const float inv_scale = 1.f / a.scale_log2;
  const int hq = lane >> 2;            // query head of this lane's B-fragment column (n = lane/4)
  const int hc = 2 * (lane & 3);       // first of the two head columns this lane holds in C fragments
  for (int round = 0, item = gw; item < n_items; item = item_of(++round)) {
    const DecodeItem it = items[item];
    const int kv_len = it.kv_len;
    const __nv_bfloat16* qbase = a.q + ((int64_t)it.t * a.qh + (int64_t)it.kvh * R) * HD;
    uint32_t qb[HD / 16][2];
#pragma unroll
    for (int ks = 0; ks < HD / 16; ++ks) {
      const int kc = ks * 16 + 2 * (lane & 3);
      qb[ks][0] = hq < R ? ldg_u32(qbase + hq * HD + kc) : 0u;
      qb[ks][1] = hq < R ? ldg_u32(qbase + hq * HD + kc + 8) : 0u;
    }
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
    float thr0 = -INFINITY, thr1 = -INFINITY;  // raw-score thresholds (m + 8) / scale of the lazy max
    float oacc[HD / 16][4];
#pragma unroll
    for (int d = 0; d < HD / 16; ++d) oacc[d][0] = oacc[d][1] = oacc[d][2] = oacc[d][3] = 0.f;

    const int np = (kv_len + 15) >> 4;
    for (int p = 0; p < np; ++p) {
      const int s = consumed % NS;
      mbar_wait(&bars[s], (consumed / NS) & 1);
      uint8_t* kb = ring + s * STAGE_BYTES;
      uint8_t* vb = kb + PAGE_BYTES;
      const int valid = min(16, kv_len - p * 16);
      if (valid < 16) {  // zero V rows of slots past kv_len (pool may hold anything there)
        for (int i = lane; i < (16 - valid) * NBOX * 8; i += 32) {
          const int row = valid + i / (NBOX * 8), rem = i % (NBOX * 8);
          *reinterpret_cast<uint4*>(vb + (rem >> 3) * BOX_BYTES + row * 128 + (rem & 7) * 16) = make_uint4(0, 0, 0, 0);
        }
        __syncwarp();
      }
      // Pull the whole page into registers (K fragments for S^T, transposed V
      // fragments for O^T) and hand the slot back to the TMA ring before any
      // math: a slot is then busy for the load latency only, not latency +
      // compute, so the same shared memory keeps more bytes in flight.
      // K fragments -> S^T = K Q^T (four independent accumulation chains over the
      // head dim, raw scores), then V fragments; the slot goes back to the TMA ring
      // as soon as both are in registers (kf and vf are never live together).
      float sacc[4][4];
      {
        uint32_t kf[HD / 16][4];
        const int key = (lane & 7) + (((lane >> 3) & 1) << 3);
        const int hi = lane >> 4;
#pragma unroll
        for (int ks = 0; ks < HD / 16; ++ks) {
          const int ch = ks * 2 + hi;
          ldmatrix_x4(kf[ks], smem_u32(kb) + (ch >> 3) * BOX_BYTES + swz(key, ch));
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
          ldmatrix_x4_trans(vf[mt], smem_u32(vb) + (ch >> 3) * BOX_BYTES + swz(key, ch));
        }
      }
      __syncwarp();
      ++consumed;
      issue_one();
      float sc[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) sc[e] = (sacc[0][e] + sacc[1][e]) + (sacc[2][e] + sacc[3][e]);
      if (p == np - 1) {  // keys past kv_len only exist in the last page
        const int k0 = p * 16 + hq, k1 = k0 + 8;
        if (k0 >= kv_len) sc[0] = sc[1] = -INFINITY;
        if (k1 >= kv_len) sc[2] = sc[3] = -INFINITY;
      }
      // Online softmax with a lazily updated running max m (per head column, in
      // log2 units): probabilities are taken against a stale max as long as no
      // raw score exceeds thr = (m + 8) / scale, so the cross-lane max reduction
      // and the O/l rescale run only when the max really moves (first page, rare
      // later); p <= 256 is exact enough in bf16 (relative rounding) and the
      // final 1/l normalisation makes the result independent of m.
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
      const uint32_t pb[2] = {movmatrix_trans(pack_bf16x2(p0, p1)), movmatrix_trans(pack_bf16x2(p2, p3))};
      // O^T += V^T P^T
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

// ---------------------------------------------------------------------------- prefill
constexpr int PF_THREADS = 128;
constexpr int PF_KT = 64;  // keys per tile (4 pages)

template <int HD>
constexpr int pf_smem() { return 2 * 2 * 4 * 16 * HD * 2 + 64 + 1024; }

template <int HD>
__global__ void __launch_bounds__(PF_THREADS)
    prefill_attn_kernel(const __grid_constant__ CUtensorMap pool, const AttnArgs a,
                        const PrefillItem* __restrict__ items, int n_items) {
  constexpr int NBOX = HD / 64;
  constexpr int BLK = 16 * HD * 2;        // one page block (K or V)
  constexpr int TILE = 4 * BLK;           // 64 keys of K (or V)
  constexpr int STAGE = 2 * TILE;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * STAGE);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  if (tid == 0) {
    tma_prefetch_desc(&pool);
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_barrier_init();
  }
  __syncthreads();
  const int kh = a.kh, R = a.qh / a.kh;
  uint32_t tiles_done = 0;  // running count of consumed tiles (phase tracking)

  for (int idx = blockIdx.x; idx < n_items; idx += gridDim.x) {
    const PrefillItem it = items[idx];
    const int g = it.h / R;
    const int n_pages = (it.kv_total + 15) >> 4;
    const int last_pos = it.pos0 + it.n - 1;
    const int n_kt = last_pos / PF_KT + 1;

    auto issue = [&](int kt, int s) {  // thread 0 only
      int np = min(4, n_pages - kt * 4);
      fence_proxy_async();
      mbar_arrive_expect_tx(&bars[s], np * 2 * BLK);
      uint8_t* dst = smem + s * STAGE;
      for (int i = 0; i < np; ++i) {
        const int64_t page = a.page_ids[it.page_start + kt * 4 + i];
        const int rowK = (int)(((page * 2 + 0) * kh + g) * 16);
        const int rowV = rowK + kh * 16;
        for (int b = 0; b < NBOX; ++b) {
          tma_load_2d(dst + i * BLK + b * BOX_BYTES, &pool, &bars[s], b * 64, rowK);
          tma_load_2d(dst + TILE + i * BLK + b * BOX_BYTES, &pool, &bars[s], b * 64, rowV);
        }
      }
    };
    if (tid == 0) {
      issue(0, tiles_done & 1);
      if (n_kt > 1) issue(1, (tiles_done + 1) & 1);
    }

    // Q fragments of this warp's 16 rows
    const int r0 = warp * 16 + (lane >> 2), r1 = r0 + 8;
    const int p0 = it.pos0 + min(r0, it.n - 1), p1 = it.pos0 + min(r1, it.n - 1);
    const __nv_bfloat16* q0 = a.q + ((int64_t)(it.t0 + min(r0, it.n - 1)) * a.qh + it.h) * HD;
    const __nv_bfloat16* q1 = a.q + ((int64_t)(it.t0 + min(r1, it.n - 1)) * a.qh + it.h) * HD;
    uint32_t qf[HD / 16][4];
#pragma unroll
    for (int ks = 0; ks < HD / 16; ++ks) {
      const int kc = ks * 16 + 2 * (lane & 3);
      qf[ks][0] = ldg_u32(q0 + kc);
      qf[ks][1] = ldg_u32(q1 + kc);
      qf[ks][2] = ldg_u32(q0 + kc + 8);
      qf[ks][3] = ldg_u32(q1 + kc + 8);
    }
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
    float oacc[HD / 8][4];
#pragma unroll
    for (int d = 0; d < HD / 8; ++d) oacc[d][0] = oacc[d][1] = oacc[d][2] = oacc[d][3] = 0.f;

    for (int kt = 0; kt < n_kt; ++kt) {
      const int s = tiles_done & 1;
      mbar_wait(&bars[s], (tiles_done >> 1) & 1);
      uint8_t* kb = smem + s * STAGE;
      uint8_t* vb = kb + TILE;
      const int valid = min(PF_KT, it.kv_total - kt * PF_KT);
      if (valid < PF_KT) {  // zero V rows past kv_total (incl. pages not loaded)
        for (int i = tid; i < (PF_KT - valid) * NBOX * 8; i += PF_THREADS) {
          const int key = valid + i / (NBOX * 8), rem = i % (NBOX * 8);
          *reinterpret_cast<uint4*>(vb + (key >> 4) * BLK + (rem >> 3) * BOX_BYTES + (key & 15) * 128 + (rem & 7) * 16) =
              make_uint4(0, 0, 0, 0);
        }
        __syncthreads();
      }
      const int kbase = kt * PF_KT;
      const bool active = kbase <= it.pos0 + min(warp * 16 + 15, it.n - 1);  // warp has visible keys
      if (active) {
        float sacc[8][4];
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) sacc[nt][0] = sacc[nt][1] = sacc[nt][2] = sacc[nt][3] = 0.f;
        const int hi = (lane >> 3) & 1;
#pragma unroll
        for (int n2 = 0; n2 < 4; ++n2) {
          const int key = n2 * 16 + (lane & 7) + ((lane >> 4) << 3);
          const uint32_t base = smem_u32(kb) + (key >> 4) * BLK;
#pragma unroll
          for (int ks = 0; ks < HD / 16; ++ks) {
            const int ch = ks * 2 + hi;
            uint32_t kf[4];
            ldmatrix_x4(kf, base + (ch >> 3) * BOX_BYTES + swz(key & 15, ch));
            const uint32_t b0[2] = {kf[0], kf[1]}, b1[2] = {kf[2], kf[3]};
            mma_bf16_16816(sacc[2 * n2], qf[ks], b0);
            mma_bf16_16816(sacc[2 * n2 + 1], qf[ks], b1);
          }
        }
        float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
        for (int nt = 0; nt < 8; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int key = kbase + nt * 8 + 2 * (lane & 3) + (e & 1);
            const int pr = e < 2 ? p0 : p1;
            const float v = key <= pr ? sacc[nt][e] * a.scale_log2 : -INFINITY;
            sacc[nt][e] = v;
            if (e < 2) mx0 = fmaxf(mx0, v); else mx1 = fmaxf(mx1, v);
          }
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
        const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
        const float al0 = exp2f(m0 - mn0), al1 = exp2f(m1 - mn1);
        m0 = mn0;
        m1 = mn1;
        float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
          sacc[nt][0] = exp2f(sacc[nt][0] - mn0);
          sacc[nt][1] = exp2f(sacc[nt][1] - mn0);
          sacc[nt][2] = exp2f(sacc[nt][2] - mn1);
          sacc[nt][3] = exp2f(sacc[nt][3] - mn1);
          rs0 += sacc[nt][0] + sacc[nt][1];
          rs1 += sacc[nt][2] + sacc[nt][3];
        }
        l0 = l0 * al0 + rs0;
        l1 = l1 * al1 + rs1;
#pragma unroll
        for (int d = 0; d < HD / 8; ++d) {
          oacc[d][0] *= al0; oacc[d][1] *= al0;
          oacc[d][2] *= al1; oacc[d][3] *= al1;
        }
        const int vk = (lane & 7) + (((lane >> 3) & 1) << 3);
        const int vhi = lane >> 4;
#pragma unroll
        for (int kc = 0; kc < 4; ++kc) {
          const uint32_t pf[4] = {pack_bf16x2(sacc[2 * kc][0], sacc[2 * kc][1]),
                                  pack_bf16x2(sacc[2 * kc][2], sacc[2 * kc][3]),
                                  pack_bf16x2(sacc[2 * kc + 1][0], sacc[2 * kc + 1][1]),
                                  pack_bf16x2(sacc[2 * kc + 1][2], sacc[2 * kc + 1][3])};
          const int key = kc * 16 + vk;
          const uint32_t base = smem_u32(vb) + (key >> 4) * BLK;
#pragma unroll
          for (int dp = 0; dp < HD / 16; ++dp) {
            const int ch = dp * 2 + vhi;
            uint32_t vf[4];
            ldmatrix_x4_trans(vf, base + (ch >> 3) * BOX_BYTES + swz(key & 15, ch));
            const uint32_t b0[2] = {vf[0], vf[1]}, b1[2] = {vf[2], vf[3]};
            mma_bf16_16816(oacc[2 * dp], pf, b0);
            mma_bf16_16816(oacc[2 * dp + 1], pf, b1);
          }
        }
      }
      __syncthreads();
      ++tiles_done;
      if (tid == 0 && kt + 2 < n_kt) issue(kt + 2, s);
    }
    l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
    l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
    const float i0 = 1.f / l0, i1 = 1.f / l1;
#pragma unroll
    for (int d = 0; d < HD / 8; ++d) {
      const int col = d * 8 + 2 * (lane & 3);
      if (r0 < it.n)
        *reinterpret_cast<uint32_t*>(a.o + ((int64_t)(it.t0 + r0) * a.qh + it.h) * HD + col) =
            pack_bf16x2(oacc[d][0] * i0, oacc[d][1] * i0);
      if (r1 < it.n)
        *reinterpret_cast<uint32_t*>(a.o + ((int64_t)(it.t0 + r1) * a.qh + it.h) * HD + col) =
            pack_bf16x2(oacc[d][2] * i1, oacc[d][3] * i1);
    }
  }
}

// Row streams for one decode launch: block-parallel.  Every block computes the page totals
// of all consumer warps (their items in the kernel's snake order) and the exclusive scan
// (block 0 writes wstart); then each warp of the grid writes one consumer warp's rows
// (lanes over pages).
__global__ void build_dec_rows_kernel(const DecodeItem* __restrict__ items, int n_items, int grid, int warps,
                                      const int* __restrict__ page_ids, int kh, int* __restrict__ rows,
                                      int* __restrict__ wstart) {
  __shared__ int tot[2048 + 1];
  __shared__ int wsum[8];
  const int TW = grid * warps;
  auto item_of = [&](int gw, int round) { return round * TW + ((round & 1) ? TW - 1 - gw : gw); };
  // per-warp page totals, then a block-wide exclusive scan (blockDim 256, 8 consecutive warps per thread)
  const int per = (TW + 255) / 256, g0 = threadIdx.x * per;
  int run = 0;
  for (int k = 0; k < per; ++k) {
    const int gw = g0 + k;
    int t = 0;
    if (gw < TW)
      for (int round = 0, it = item_of(gw, 0); it < n_items; it = item_of(gw, ++round)) t += (items[it].kv_len + 15) >> 4;
    if (gw < TW) tot[gw] = t;
    run += t;
  }
  int incl = run;  // inclusive scan of the per-thread sums: warp shuffles, then the 8 warp totals
  const int ln = threadIdx.x & 31, wp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (ln >= o) incl += v;
  }
  if (ln == 31) wsum[wp] = incl;
  __syncthreads();
  int base = 0;
  for (int w2 = 0; w2 < wp; ++w2) base += wsum[w2];
  int acc = base + incl - run;  // exclusive prefix of this thread's first warp
  for (int k = 0; k < per; ++k) {
    const int gw = g0 + k;
    if (gw < TW) {
      const int v = tot[gw];
      tot[gw] = acc;
      acc += v;
    }
  }
  if (threadIdx.x == 255) tot[TW] = acc;
  __syncthreads();
  if (blockIdx.x == 0)
    for (int gw = threadIdx.x; gw <= TW; gw += blockDim.x) wstart[gw] = tot[gw];
  const int lane = threadIdx.x & 31;
  for (int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); gw < TW; gw += gridDim.x * (blockDim.x >> 5)) {
    int o = tot[gw];
    for (int round = 0, it = item_of(gw, 0); it < n_items; it = item_of(gw, ++round)) {
      const DecodeItem d = items[it];
      const int np = (d.kv_len + 15) >> 4;
      for (int p = lane; p < np; p += 32) rows[o + p] = ((page_ids[d.page_start + p] * 2) * kh + d.kvh) * 16;
      o += np;
    }
  }
}

template <int HD, int W>
cudaError_t launch_decode_hdw(const CUtensorMap& m, const CUtensorMap& pm, const AttnArgs& a, const DecodeItem* items, int n_items,
                              int sm_budget, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(decode_attn_kernel<HD, W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         dec_smem<HD, W>());
    if (e != cudaSuccess) return e;
    attr = true;
  }
  // one CTA per SM of the budget (8-warp CTAs fill an SM's smem; 4-warp CTAs leave room for a GEMM CTA)
  int grid = decode_grid(n_items, sm_budget, W);
  if (a.dec_rows) {
    static bool attr_r = false;
    if (!attr_r) {
      cudaError_t e = cudaFuncSetAttribute(decode_attn_kernel<HD, W, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           dec_smem<HD, W>());
      if (e != cudaSuccess) return e;
      attr_r = true;
    }
    decode_attn_kernel<HD, W, true><<<grid, W * 32, dec_smem<HD, W>(), st>>>(m, pm, a, items, n_items);
  } else {
    decode_attn_kernel<HD, W><<<grid, W * 32, dec_smem<HD, W>(), st>>>(m, pm, a, items, n_items);
  }
  count_launch();
  return cudaGetLastError();
}

template <int HD>
cudaError_t launch_decode_hd(const CUtensorMap& m, const CUtensorMap& pm, const AttnArgs& a, const DecodeItem* items, int n_items,
                             int sm_budget, cudaStream_t st) {
  const int w = decode_warps(HD, a.dec_warps);
  if (w == 4) return launch_decode_hdw<HD, 4>(m, pm, a, items, n_items, sm_budget, st);
  if (w == 6) return launch_decode_hdw<HD, 6>(m, pm, a, items, n_items, sm_budget, st);
  if (w == 12) return launch_decode_hdw<HD, 12>(m, pm, a, items, n_items, sm_budget, st);
  if (w == 14) return launch_decode_hdw<HD, 14>(m, pm, a, items, n_items, sm_budget, st);
  return launch_decode_hdw<HD, 8>(m, pm, a, items, n_items, sm_budget, st);
}

template <int HD>
cudaError_t launch_prefill_hd(const CUtensorMap& m, const AttnArgs& a, const PrefillItem* items, int n_items,
                              int sm_budget, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(prefill_attn_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         pf_smem<HD>());
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int per_sm = std::max(1, (227 * 1024) / pf_smem<HD>());
  int grid = std::min(n_items, std::max(sm_budget, 1) * per_sm);
  prefill_attn_kernel<HD><<<grid, PF_THREADS, pf_smem<HD>(), st>>>(m, a, items, n_items);
  count_launch();
  return cudaGetLastError();
}

}  // namespace

int decode_warps(int hd, int dec_warps_arg) {
  static int env_w = -1;
  if (env_w < 0) {
    const char* e = getenv("NF_DEC_WARPS");
    env_w = e ? atoi(e) : 0;
  }
  const int w = dec_warps_arg == 4 ? 4 : (env_w ? env_w : (hd == 128 ? 12 : 8));
  return (w == 4 || w == 6 || w == 8 || w == 12 || w == 14) ? w : 8;
}

int decode_grid(int n_items, int sm_budget, int warps) {
  return std::min((n_items + warps - 1) / warps, std::max(sm_budget, 1));
}

cudaError_t launch_build_dec_rows(const DecodeItem* items, int n_items, int grid, int warps, const int* page_ids, int kh,
                                  int* rows, int* wstart, cudaStream_t st) {
  if (n_items <= 0) return cudaSuccess;
  if (grid * warps > 2048) return cudaErrorInvalidValue;
  build_dec_rows_kernel<<<std::max(1, std::min(148, grid * warps / 8)), 256, 0, st>>>(items, n_items, grid, warps, page_ids, kh,
                                                                          rows, wstart);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_decode_attention(const CUtensorMap& m, const CUtensorMap& pm, const AttnArgs& a0, const DecodeItem* items, int n_items,
                                    int sm_budget, cudaStream_t st) {
  if (n_items <= 0) return cudaSuccess;
  // L2 prefetch distance (pages ahead of the TMA ring within an item; NF_DEC_PF, 0 = off)
  static int pf_env = -1;
  if (pf_env < 0) {
    const char* e = getenv("NF_DEC_PF");
    pf_env = e ? atoi(e) : 0;
  }
  AttnArgs a = a0;
  a.pf_dist = std::min(std::max(pf_env, 0), 31);
  if (a.hd == 128) return launch_decode_hd<128>(m, pm, a, items, n_items, sm_budget, st);
  if (a.hd == 64) return launch_decode_hd<64>(m, pm, a, items, n_items, sm_budget, st);
  return cudaErrorInvalidValue;
}

int prefill_rows(int head_dim) {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("NF_PREFILL_IMPL");
    env = (e && std::string(e) == "mma") ? 1 : 0;
  }
  return (head_dim == 128 && env == 0) ? 128 : 64;
}

cudaError_t launch_prefill_attention(const CUtensorMap& m, const AttnArgs& a, const PrefillItem* items,
                                     int n_items, int sm_budget, cudaStream_t st) {
  if (n_items <= 0) return cudaSuccess;
  if (a.hd == 128 && prefill_rows(128) == 128) return launch_prefill_attention_tc(m, a, items, n_items, sm_budget, st);
  if (a.hd == 128) return launch_prefill_hd<128>(m, a, items, n_items, sm_budget, st);
  if (a.hd == 64) return launch_prefill_hd<64>(m, a, items, n_items, sm_budget, st);
  return cudaErrorInvalidValue;
}

// One kernel of this translation unit (preload_all_kernels: its module is loaded eagerly).
const void* kernel_anchor_attention() { return reinterpret_cast<const void*>(build_dec_rows_kernel); }

}  // namespace nf
