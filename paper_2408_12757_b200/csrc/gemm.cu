// Persistent, warp-specialised tcgen05 GEMM for sm_100a with the decoder
// layer's fused epilogues.
//
//   warp 0 lane 0 : TMA producer (A and B 128B-swizzled K-major tiles, 4-stage ring)
//   warp 1 lane 0 : tcgen05.mma issuer (M=128, N=256, K=16 per instruction, f32 in TMEM)
//   warp 2        : TMEM allocator (2 accumulator stages x 256 columns = 512 columns)
//   warps 4..7    : epilogue (tcgen05.ld: one thread per accumulator row)
//
// The grid is min(#tiles, SM budget): one CTA per SM (smem-bound), so the SM
// budget of the nano-batch plan ("limits the execution units
// usage of each kernel") is exactly the number of SMs the GEMM occupies.
#include <cudaTypedefs.h>

#include <mutex>

#include "common.cuh"
#include "profile.h"
#include "gemm.cuh"

namespace nf {

namespace {

constexpr int A_STAGE_ELEMS = GEMM_BM * GEMM_BK;

#ifdef NF_GEMM_TS
// (dev build, -DNF_GEMM_TS) phase timestamps of CTA 0 of the last GEMM launch (tools/gemm_phases.py)
__device__ unsigned long long g_gemm_ts[8];
NF_DEV void gemm_ts(int i) {
  if (blockIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_gemm_ts[i] = t;
  }
}
#else
NF_DEV void gemm_ts(int) {}
#endif

NF_DEV void store32_bf16(__nv_bfloat16* dst, const float (&v)[32]) {
  uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint4 u;
    u.x = pack_bf16x2(v[q * 8 + 0], v[q * 8 + 1]);
    u.y = pack_bf16x2(v[q * 8 + 2], v[q * 8 + 3]);
    u.z = pack_bf16x2(v[q * 8 + 4], v[q * 8 + 5]);
    u.w = pack_bf16x2(v[q * 8 + 6], v[q * 8 + 7]);
    d[q] = u;
  }
}

// 1-D bulk copy global -> shared memory, completing on an mbarrier (transaction bytes)
NF_DEV void bulk_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

NF_DEV int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
NF_DEV void named_bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
// Programmatic dependent launch: wait for the preceding kernel of the stream (its
// memory is visible afterwards); let the next kernel of the stream start launching.
// Both are no-ops when the launch carries no programmatic-serialization attribute.
NF_DEV void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
NF_DEV void griddep_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }


// 1/rms of one row from its sum-of-squares partials part[p * stride], p < np, with 4
// independent accumulators in a fixed order (kept out of line: inlined into the GEMM
// epilogue it pushed the kernel into a local-memory stack frame).
// EPI_PEER (peer.cuh): base such that base + col addresses row `trow` of output block
// (bm, n0 / 256) in its owner's staging slot [this rank][owned block][128][256].
__device__ __forceinline__ __nv_bfloat16* peer_row(const GemmArgs& a, int bm, int n0, int trow) {
  const int blk = bm + (n0 / 256) * a.peer_mb;
  const int owner = blk % a.peer_n, lb = blk / a.peer_n;
  __nv_bfloat16* row = reinterpret_cast<__nv_bfloat16*>(a.peer_bases[owner] + a.peer_site_off + a.peer_stage_off) +
                       (((int64_t)a.peer_rank * a.peer_maxown + lb) * 128 + trow) * 256;
  return row - (n0 & ~255);
}
// EPI_RESID in a PEER instance (args.peer_mode 1, the O column-parallel projection): row r
// of this rank's slice in rank q's all-gather region [peer_n][M][N] (a site's result region).
__device__ __forceinline__ __nv_bfloat16* peer_ag_row(const GemmArgs& a, int q, int r) {
  return reinterpret_cast<__nv_bfloat16*>(a.peer_bases[q] + a.peer_site_off + a.peer_result_off) +
         ((int64_t)a.peer_rank * a.M + r) * a.N;
}
// ... then every rank's `done` counter of the site grows by this unit's 64-column chunks.
__device__ __forceinline__ void peer_ag_signal(const GemmArgs& a, int bm, int n0, int bn) {
  if (bm >= a.peer_mb || n0 >= a.N) return;
  const uint32_t chunks = (uint32_t)(min(bn, a.N - n0) / 64);
  for (int q = 0; q < a.peer_n; ++q) {
    uint32_t* done = reinterpret_cast<uint32_t*>(a.peer_bases[(a.peer_rank + 1 + q) % a.peer_n] + a.peer_site_off +
                                                 a.peer_flags_off);
    asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(done), "r"(chunks) : "memory");
  }
}
// EPI_PEER: after every epilogue thread's stores are fenced (system scope) and the 128
// threads met, add BN/64 to the owner's flag of (block, this rank) with release semantics.
__device__ __forceinline__ void peer_signal(const GemmArgs& a, int bm, int n0, int bn) {
  if (bm >= a.peer_mb || n0 >= a.N) return;
  const int blk = bm + (n0 / 256) * a.peer_mb;
  const int owner = blk % a.peer_n, lb = blk / a.peer_n;
  uint32_t* flag = reinterpret_cast<uint32_t*>(a.peer_bases[owner] + a.peer_site_off + a.peer_flags_off + 256) +
                   lb * a.peer_n + a.peer_rank;
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(flag), "r"((uint32_t)(bn / 64)) : "memory");
}

__device__ __noinline__ float rms_row_scale(const float* part, int64_t stride, int np, float inv_d, float eps) {
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
  int p = 0;
  for (; p + 4 <= np; p += 4) {
    a0 += part[(p + 0) * stride];
    a1 += part[(p + 1) * stride];
    a2 += part[(p + 2) * stride];
    a3 += part[(p + 3) * stride];
  }
  for (; p < np; ++p) a0 += part[p * stride];
  return rsqrtf(((a0 + a1) + (a2 + a3)) * inv_d + eps);
}

// sin/cos of a large fp32 angle: Cody-Waite reduction to [-pi, pi] then SFU.
NF_DEV void sincos_reduced(float a, float* s, float* c) {
  const float k = rintf(a * 0.15915494309189535f);
  float r = fmaf(-k, 6.28318548202514648f, a);
  r = fmaf(-k, -1.7484556e-07f, r);
  __sincosf(r, s, c);
}

// CG = 2: CTA-pair (cta_group::2) variant.  A cluster of two CTAs on one TPC computes
// a 256 x BN tile: each CTA loads its 128 rows of A and half (BN/2 rows) of the B
// tile, the even CTA issues tcgen05.mma.cta_group::2 (M = 256) over both CTAs' smem,
// and each CTA's TMEM receives its own 128 x BN accumulator.  Per CTA the smem stage
// is 32 KB instead of 48 KB, so the ring is 6 deep, and each B byte is fetched
// once per pair.  Data-parallel or split-K tail schedule (split-K=2 is CG = 1 only);
// split-K partial slots and arrival flags are per CTA of the pair.
//
// SR (smem residual, EPI_RESID with short K): the epilogue stages the tile's residual
// in shared memory by TMA (issued before the accumulator is ready), adds the
// accumulator in place and TMA-stores each finished 64-column box, so the epilogue
// no longer waits on per-thread global loads and scattered row stores (short-K GEMMs,
// e.g. the 70B TP8 rank's O projection with K = 1024, were epilogue-bound).
// PEER: EPI_PEER instances (peer.cuh) -- the plain instances carry no peer code.
template <int GEMM_STAGES, int BN, int CG, bool SR = false, bool PEER = false>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_tcgen05_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        const __grid_constant__ CUtensorMap tmR, const __grid_constant__ CUtensorMap tmO,
                        const __grid_constant__ GemmArgs args) {
  constexpr int B_ROWS = BN / CG;  // B tile rows held by this CTA
  constexpr int B_STAGE_ELEMS = B_ROWS * GEMM_BK;
  constexpr uint32_t STAGE_BYTES = (A_STAGE_ELEMS + B_STAGE_ELEMS) * 2;  // per CTA
  constexpr int TM = GEMM_BM * CG;                                         // tile rows
  constexpr uint32_t TMEM_COLS = 2 * BN;  // two accumulator stages
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __nv_bfloat16* sA = reinterpret_cast<__nv_bfloat16*>(smem);
  __nv_bfloat16* sB = sA + GEMM_STAGES * A_STAGE_ELEMS;
  uint8_t* sR = reinterpret_cast<uint8_t*>(sB + GEMM_STAGES * B_STAGE_ELEMS);  // SR: [BN/64][128 rows][128 B]
  constexpr uint32_t SR_BYTES = SR ? (uint32_t)BN * GEMM_BM * 2 : 0u;
  uint64_t* full = reinterpret_cast<uint64_t*>(sR + SR_BYTES);
  uint64_t* empty = full + GEMM_STAGES;
  uint64_t* tfull = empty + GEMM_STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* rbar = tempty + 2;  // SR: residual tile landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rbar + 2);
  float* inv_freq = reinterpret_cast<float*>(tmem_slot + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef NF_GEMM_TS
  if (threadIdx.x == 0 && blockIdx.x == 0) g_gemm_ts[6] = g_gemm_ts[5];  // previous launch's CTA-0 exit
#endif
  if (threadIdx.x == 0) gemm_ts(0);  // kernel entry
  const int M = args.M, N = args.N, K = args.K;
  uint32_t rank = 0;  // CTA rank in the pair
  if constexpr (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int wid = blockIdx.x / CG;  // tile worker: a CTA (CG 1) or a CTA pair (CG 2)
  const bool grouped = args.grp_off != nullptr;
  if (grouped) griddep_wait();  // the tile list is the previous kernel's output
  // grouped: the row count in use is device data (written by the routing kernels)
  const int tiles_m = grouped ? min(args.grp_off[args.n_groups], M) / TM : (M + TM - 1) / TM;
  const int tiles_n = (N + BN - 1) / BN;
  // group of an m-tile (grouped mode): the last g with grp_off[g] <= row
  auto group_of = [&](int mb) {
    int g = 0;
    if (grouped)
      while (g + 1 < args.n_groups && args.grp_off[g + 1] <= mb * TM) ++g;
    return g;
  };
  const int tiles = tiles_m * tiles_n;
  const int num_kb = (K + GEMM_BK - 1) / GEMM_BK;
  // Split-K tail schedule (args.tail_split = s > 1): the full waves of tiles run
  // data-parallel in lockstep (CTA b: tiles b, b+G, ...), then each of the
  // remaining `rem` tiles is split into s equal K ranges run at the same time by
  // CTAs u = s*i .. s*i+s-1 (u < rem*s <= G).  Split j > 0 leaves an fp32 partial
  // in slot u; split 0 (the owner) adds them in split order and runs the fused
  // epilogue.  A partial last wave then costs 1/s of a tile round instead of a
  // whole one, and concurrent splits stay aligned in K (L2 reuse is kept).
  const int G = gridDim.x / CG;
  // split-K=2 schedule (args.split == 2): units (tile, K-half) in tile-major
  // order, so both halves of a tile run at the same time on adjacent CTAs (L2
  // reuse of the weight tile across m-tiles is kept); half 1 leaves an fp32
  // partial in the tile's slot, half 0 adds it in its epilogue.
  const bool split2 = CG == 1 && args.split == 2 && args.sk_part != nullptr;
  const int ts = (!split2 && args.sk_part != nullptr) ? max(1, args.tail_split) : 1;
  // Stream-K (args.stream_k, sub-wave GEMMs): CTA c runs k-blocks [c U / G, (c+1) U / G)
  // of the tile-major (tile, k-block) space, U = tiles * num_kb, so every SM of the
  // budget works even when there are fewer tiles than SMs.  A CTA's first segment
  // may start inside a tile (a contributor: fp32 partial to its slot); the CTA
  // holding a tile's k-block 0 owns it and adds the later CTAs' partials in CTA order.
  // Mode 2 (grouped GEMMs, whose tile count is device data): full waves run
  // data-parallel and the remaining tiles [sk_t0, tiles) run stream-K, decided here
  // from the device tile count when each CTA gets >= 16 of their k-blocks.
  const int sk_mode = (!split2 && args.sk_part != nullptr) ? args.stream_k : 0;  // CG 2: G = pairs, slots per CTA
  bool sk = sk_mode == 1;
  int sk_t0 = 0;
  if (sk_mode == 2) {
    const int rem = tiles % G;
    if (rem > 0 && (int64_t)rem * num_kb >= 16LL * G) {
      sk = true;
      sk_t0 = tiles - rem;
    }
  }
  const int64_t U_sk = (int64_t)(tiles - sk_t0) * num_kb;
  auto sk_cta_of = [&](int64_t u) { return (int)(((u + 1) * G - 1) / U_sk); };  // CTA covering unit u
  const int tiles_dp = split2 ? 0 : (ts > 1 ? (tiles / G) * G : tiles);
  const int tail_units = ts > 1 ? (tiles - tiles_dp) * ts : 0;
  const int kb_half = num_kb / 2;
  // (the tile loop and its three bodies are always inlined: a body the compiler keeps out of
  // line gets its captures through a local-memory closure -- a 328-400 byte stack frame that
  // cost the sub-wave / short-K GEMMs 15-28 %, profiles/r2i_gemm_r1_vs_now.log)
  // fn(tile, kb0, kb1, last): `last` = no further segment follows on this CTA (its smem stages
  // are idle once this segment's accumulator is complete)
  auto for_each_seg = [&](auto&& fn) __attribute__((always_inline)) {
    if (sk) {
      const int64_t a = (int64_t)wid * U_sk / G, b = (int64_t)(wid + 1) * U_sk / G;
      for (int t = wid; t < sk_t0; t += G) fn(t, 0, num_kb, t + G >= sk_t0 && a >= b);
      for (int64_t u = a; u < b;) {
        const int t = (int)(u / num_kb);
        const int k0 = (int)(u - (int64_t)t * num_kb);
        const int k1 = (int)min((int64_t)num_kb, b - (int64_t)t * num_kb);
        fn(sk_t0 + t, k0, k1, (int64_t)t * num_kb + k1 >= b);
        u = (int64_t)t * num_kb + k1;
      }
      return;
    }
    if (split2) {
      for (int u = wid; u < 2 * tiles; u += G) {
        if (u & 1) fn(u >> 1, kb_half, num_kb, u + G >= 2 * tiles);
        else fn(u >> 1, 0, kb_half, u + G >= 2 * tiles);
      }
      return;
    }
    for (int t = wid; t < tiles_dp; t += G) fn(t, 0, num_kb, t + G >= tiles_dp && wid >= tail_units);
    if (wid < tail_units) {
      const int j = wid % ts;
      fn(tiles_dp + wid / ts, j * num_kb / ts, (j + 1) * num_kb / ts, true);
    }
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < GEMM_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4 * CG);  // epilogue warps of both CTAs drain into the even CTA's barrier
    }
    if constexpr (SR) mbar_init(rbar, 1);
    mbar_init(rbar + 1, 1);  // smem-staged stream-K fix-up
    fence_barrier_init();
  }
  if constexpr (CG == 2) cluster_sync();  // peer barriers initialised before any remote arrive / TMA
  if (warp == 2) {
    if constexpr (CG == 2) tmem_alloc_cg2(tmem_slot, TMEM_COLS);
    else tmem_alloc(tmem_slot, TMEM_COLS);
  }
  if (args.epi == EPI_QKV && warp >= 4) {
    const int i = threadIdx.x - 128;
    if (i < args.hd / 2) inv_freq[i] = (float)exp2(-(2.0 * i / args.hd) * (double)args.log2_theta);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) gemm_ts(1);  // prologue done (barriers, TMEM allocated)
  // everything above (barriers, TMEM, descriptor prefetch) overlaps the previous kernel's
  // tail under PDL; every global read of its outputs and every global write is below
  griddep_wait();

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer
      int stage = 0;
      uint32_t phase = 0;
      const uint64_t a_policy = policy_evict_last();  // activations are re-read by every n-tile
      const uint64_t b_policy = policy_evict_normal();
      for_each_seg([&](int tile, int kb0, int kb1, bool) __attribute__((always_inline)) {
        const int mb = tile % tiles_m, nb = tile / tiles_m;
        const int b_row0 = grouped ? group_of(mb) * N : 0;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if constexpr (CG == 2) {
            // both CTAs' loads complete on the even CTA's full barrier, armed once for both
            const uint32_t fb = mapa_shared(smem_u32(&full[stage]), 0);
            if (rank == 0) mbar_arrive_expect_tx(&full[stage], STAGE_BYTES * CG);
            tma_load_2d_cg2(sA + stage * A_STAGE_ELEMS, &tmA, fb, kb * GEMM_BK, mb * TM + (int)rank * GEMM_BM,
                            a_policy);
            tma_load_2d_cg2(sB + stage * B_STAGE_ELEMS, &tmB, fb, kb * GEMM_BK, nb * BN + (int)rank * B_ROWS,
                            b_policy);
          } else {
            mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
            if (args.a_slots > 1)  // slot layout: k-block kb lies in slot kb*BK / a_slot_w
              tma_load_3d(sA + stage * A_STAGE_ELEMS, &tmA, &full[stage], (kb * GEMM_BK) % args.a_slot_w, mb * GEMM_BM,
                          (kb * GEMM_BK) / args.a_slot_w);
            else
              tma_load_2d_hint(sA + stage * A_STAGE_ELEMS, &tmA, &full[stage], kb * GEMM_BK, mb * GEMM_BM, a_policy);
            tma_load_2d(sB + stage * B_STAGE_ELEMS, &tmB, &full[stage], kb * GEMM_BK, nb * BN + b_row0);
          }
          if (++stage == GEMM_STAGES) { stage = 0; phase ^= 1; }
        }
      });
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ------------------------------------------------------------ MMA issuer (even CTA of a pair)
      constexpr uint32_t idesc = idesc_bf16_f32(TM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int as = 0;
      uint32_t aphase = 0;
      bool first_full = true;
      for_each_seg([&](int tile, int kb0, int kb1, bool) __attribute__((always_inline)) {
        mbar_wait(&tempty[as], aphase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + as * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          if (first_full) {
            gemm_ts(2);  // first A/B stage landed
            first_full = false;
          }
          tc_fence_after();
          const uint64_t ad = sdesc_sw128(sA + stage * A_STAGE_ELEMS);
          const uint64_t bd = sdesc_sw128(sB + stage * B_STAGE_ELEMS);
#pragma unroll
          for (int k = 0; k < GEMM_BK / 16; ++k) {
            if constexpr (CG == 2) umma_bf16_cg2(d, ad + 2 * k, bd + 2 * k, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
            else umma_bf16(d, ad + 2 * k, bd + 2 * k, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          }
          if constexpr (CG == 2) umma_commit_cg2_mc(&empty[stage]);  // frees the stage in both CTAs
          else umma_commit(&empty[stage]);
          if (++stage == GEMM_STAGES) { stage = 0; phase ^= 1; }
        }
        if constexpr (CG == 2) umma_commit_cg2_mc(&tfull[as]);
        else umma_commit(&tfull[as]);
        as ^= 1;
        if (as == 0) aphase ^= 1;
      });
      gemm_ts(3);                   // last MMA issued
      griddep_launch_dependents();  // all MMAs issued: the next kernel may start its prologue
    }
  } else if (warp >= 4) {
    // -------------------------------------------------------------- epilogue
    const int ew = warp - 4;
    int as = 0;
    uint32_t aphase = 0, rphase = 0, fphase = 0;
    // smem-staged fix-up (NF_GEMM_SKSMEM=0 disables it for A/B): the stage ring holds one partial
    const bool sk_smem_ok = args.sk_smem && (uint32_t)GEMM_STAGES * STAGE_BYTES >= (uint32_t)(GEMM_BM * BN * 4);
    const int trow = ew * 32 + lane;  // row within the tile
    const bool leader = ew == 0 && lane == 0;
    if constexpr (SR) {
      if (leader) tma_prefetch_desc(&tmR);
    }
    for_each_seg([&](int tile, int kb0, int kb1, bool last) __attribute__((always_inline)) {
      const int mb = tile % tiles_m, nb = tile / tiles_m;
      const int r = mb * TM + (int)rank * GEMM_BM + trow;
      const bool valid = grouped ? r < args.grp_end[group_of(mb)] : r < M;
      if constexpr (SR) {
        // the residual tile -> smem while the mainloop runs (after the previous tile's
        // stores have read the buffer); rows >= M / cols >= N are zero-filled and clipped
        if (leader && kb0 == 0 && args.epi == EPI_RESID) {
          bulk_wait_read0();
          mbar_arrive_expect_tx(rbar, SR_BYTES);
#pragma unroll
          for (int b = 0; b < BN / 64; ++b)
            tma_load_2d(sR + b * GEMM_BM * 128, &tmR, rbar, nb * BN + b * 64, mb * TM + (int)rank * GEMM_BM);
        }
      } else if (args.epi == EPI_RESID && valid && kb0 == 0) {
        // residual row segment -> L2 while the tile's mainloop still runs (short-K
        // GEMMs are otherwise epilogue-bound on these dependent global loads)
        const char* rp = reinterpret_cast<const char*>(args.resid + (int64_t)r * args.ldr + nb * BN);
#pragma unroll
        for (int q = 0; q < BN * 2 / 128; ++q)
          if (nb * BN + q * 64 < N) asm volatile("prefetch.global.L2 [%0];" ::"l"(rp + q * 128));
      }
      // the row's scale (folded RMSNorm 1/rms from the previous kernel's D/128 sum-of-squares
      // partials, 4 independent accumulators in a fixed order so every n-tile of a row gets the
      // identical scale) while the tile's mainloop still runs: its dependent loads are off the
      // epilogue's critical path (split-K contributors store raw partials and need none)
      float s = 1.f;
      if (kb0 == 0 && valid) {
        if (args.norm_part != nullptr)
          s = rms_row_scale(args.norm_part + r, args.norm_stride, args.norm_nparts, args.inv_d, args.eps);
        if (args.row_scale != nullptr) s *= args.row_scale[r];
      }
      mbar_wait(&tfull[as], aphase);
      tc_fence_after();
      bool fix_smem = false;
      const uint32_t taddr = tmem_base + as * BN + ((uint32_t)(ew * 32) << 16);
      if (kb0 > 0) {
        // split-K contributor: raw fp32 partial tile to its slot, then signal the
        // tile's owner.  Slot layout float4[BN/4][128 rows]: a warp's 32 rows write
        // (and the owner later reads) 512 contiguous bytes per instruction.
        const size_t slot_idx = split2 ? (size_t)tile : (size_t)(wid * CG + (int)rank);  // per CTA of a pair
        float4* slot = reinterpret_cast<float4*>(args.sk_part + slot_idx * GEMM_BM * GEMM_SK_LD) + trow;
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t rr[32];
          tmem_ld32(taddr + c * 32, rr);
          tmem_ld_wait();
#pragma unroll
          for (int q = 0; q < 8; ++q)
            slot[(c * 8 + q) * GEMM_BM] = make_float4(__uint_as_float(rr[4 * q]), __uint_as_float(rr[4 * q + 1]),
                                                      __uint_as_float(rr[4 * q + 2]), __uint_as_float(rr[4 * q + 3]));
        }
        __threadfence();
        tc_fence_before();
        named_bar_sync(1, 128);
        if (trow == 0) atomicAdd(args.sk_flag + tile * CG + (int)rank, 1);
        __syncwarp();
        if (lane == 0) {
          if constexpr (CG == 2) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[as]), 0));
          else mbar_arrive(&tempty[as]);
        }
        as ^= 1;
        if (as == 0) aphase ^= 1;
        return;
      }
      // owner: this CTA holds the tile's first K range; the other splits were run
      // concurrently by the next CTAs (tail split) or the adjacent unit (split-K=2)
      int c_first = wid + 1, n_contrib = 0;
      if (kb1 < num_kb) {
        if (split2) {
          c_first = tile;  // the tile's own partial slot
          n_contrib = 1;
        } else {
          n_contrib = sk ? sk_cta_of((int64_t)(tile - sk_t0) * num_kb + num_kb - 1) - wid : ts - 1;
        }
        // the CTA's last segment: its stage buffers are idle once the accumulator is complete, so
        // the first contributor's fp32 partial (128 x BN) comes in by one bulk copy and the fix-up
        // reads it from shared memory (a chain of dependent L2 round trips otherwise)
        fix_smem = last && sk_smem_ok;
        if (trow == 0) {
          while (ld_acquire_gpu(args.sk_flag + tile * CG + (int)rank) < n_contrib) __nanosleep(32);
          args.sk_flag[tile * CG + (int)rank] = 0;  // self-reset for the next launch
          if (fix_smem) {
            const size_t cs = split2 ? (size_t)c_first : (size_t)(c_first * CG + (int)rank);
            asm volatile("fence.proxy.async.global;" ::: "memory");  // generic-proxy partial stores -> bulk copy
            mbar_arrive_expect_tx(rbar + 1, (uint32_t)(GEMM_BM * BN * 4));
            bulk_load_1d(smem, args.sk_part + cs * GEMM_BM * GEMM_SK_LD, (uint32_t)(GEMM_BM * BN * 4), rbar + 1);
          }
        }
        named_bar_sync(1, 128);
        (void)ld_acquire_gpu(args.sk_flag + tile * CG + (int)rank);
        if (fix_smem) {
          mbar_wait(rbar + 1, fphase);
          fphase ^= 1;
        }
      }
      // accumulator + contributors' partials (fixed CTA order), times the row scale
      auto ldacc = [&](int col, float sc, float (&v)[32]) __attribute__((always_inline)) {
        uint32_t rr[32];
        tmem_ld32(taddr + col, rr);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(rr[j]);
        int c = c_first;
        if (fix_smem) {  // first contributor from shared memory (same float4[BN/4][128] layout)
          const uint32_t sp = smem_u32(smem) + (uint32_t)(((col / 4) * GEMM_BM + trow) * 16);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            float f0, f1, f2, f3;
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(f0), "=f"(f1), "=f"(f2), "=f"(f3)
                         : "r"(sp + q * GEMM_BM * 16));
            v[4 * q] += f0; v[4 * q + 1] += f1; v[4 * q + 2] += f2; v[4 * q + 3] += f3;
          }
          ++c;
        }
        for (; c < c_first + n_contrib; ++c) {
          const size_t cs = split2 ? (size_t)c : (size_t)(c * CG + (int)rank);
          const float4* src = reinterpret_cast<const float4*>(args.sk_part + cs * GEMM_BM * GEMM_SK_LD) + trow +
                              (col / 4) * GEMM_BM;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 f = src[q * GEMM_BM];
            v[4 * q] += f.x; v[4 * q + 1] += f.y; v[4 * q + 2] += f.z; v[4 * q + 3] += f.w;
          }
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] *= sc;
      };
      const int n0 = nb * BN;
      float v[32];
      switch (args.epi) {
        case EPI_STORE:
        case EPI_PEER:
        case EPI_F32: {
          if constexpr (SR) {
            if (args.epi == EPI_STORE) {
              // bf16 tile staged in smem (after the previous tile's stores have read it),
              // each finished 64-column box TMA-stored
              if (leader) bulk_wait_read0();
              named_bar_sync(2, 128);
              const uint32_t row_base = smem_u32(sR) + trow * 128;
#pragma unroll 1
              for (int c = 0; c < BN / 32; ++c) {
                ldacc(c * 32, s, v);
                const uint32_t box = row_base + (c >> 1) * GEMM_BM * 128;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  const uint32_t addr = box + ((((c & 1) * 4 + q) ^ (trow & 7)) << 4);
                  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr),
                               "r"(pack_bf16x2(v[q * 8 + 0], v[q * 8 + 1])), "r"(pack_bf16x2(v[q * 8 + 2], v[q * 8 + 3])),
                               "r"(pack_bf16x2(v[q * 8 + 4], v[q * 8 + 5])), "r"(pack_bf16x2(v[q * 8 + 6], v[q * 8 + 7]))
                               : "memory");
                }
                if (c & 1) {
                  fence_proxy_async();
                  named_bar_sync(2, 128);
                  if (leader) {
                    tma_store_2d(&tmO, sR + (c >> 1) * GEMM_BM * 128, n0 + (c >> 1) * 64,
                                 mb * TM + (int)rank * GEMM_BM);
                    bulk_commit();
                  }
                }
              }
              break;
            }
          }
          // EPI_PEER: the same bf16 stores, into the block owner's staging row (peer_row: the
          // tile's columns all lie in one 256-column block) -- out of line, like the signal
          // below, so the epilogue keeps its registers (inlined, they pushed the kernel into
          // a local-memory stack frame)
          __nv_bfloat16* obase;
          if constexpr (PEER) obase = peer_row(args, mb * CG + (int)rank, n0, trow);
          else obase = args.out + (int64_t)r * args.ldo;
#pragma unroll 1
          for (int c = 0; c < BN / 32; ++c) {
            ldacc(c * 32, s, v);
            const int col = n0 + c * 32;
            if (valid && col < N) {
              if (args.epi != EPI_F32) {
                store32_bf16(obase + col, v);
              } else {
                float4* d = reinterpret_cast<float4*>(args.outf + (int64_t)r * args.ldo + col);
#pragma unroll
                for (int q = 0; q < 8; ++q) d[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
              }
            }
          }
          if constexpr (PEER) {
            asm volatile("fence.acq_rel.sys;" ::: "memory");  // this thread's peer stores before the flag
            named_bar_sync(1, 128);
            if (trow == 0) peer_signal(args, mb * CG + (int)rank, n0, BN);
          }
          break;
        }
        case EPI_RESID: {
          if constexpr (SR) {
            mbar_wait(rbar, rphase);
            rphase ^= 1;
            float sq = 0.f;
            const uint32_t row_base = smem_u32(sR) + trow * 128;
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {
              ldacc(c * 32, s, v);
              const uint32_t box = row_base + (c >> 1) * GEMM_BM * 128;
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const uint32_t addr = box + ((((c & 1) * 4 + q) ^ (trow & 7)) << 4);
                uint32_t w0, w1, w2, w3;
                asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3)
                             : "r"(addr));
                const uint32_t w[4] = {w0, w1, w2, w3};
                uint32_t o[4];
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                  const float2 f = unpack_bf16x2(w[h]);
                  const float x0 = round_bf16(f.x + v[q * 8 + 2 * h]), x1 = round_bf16(f.y + v[q * 8 + 2 * h + 1]);
                  sq = fmaf(x0, x0, sq);
                  sq = fmaf(x1, x1, sq);
                  o[h] = pack_bf16x2(x0, x1);
                }
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(o[0]), "r"(o[1]), "r"(o[2]),
                             "r"(o[3])
                             : "memory");
              }
              if ((c & 3) == 3) {
                if (args.sq_out != nullptr && valid && n0 + c * 32 < N)
                  args.sq_out[(int64_t)((n0 >> 7) + (c >> 2)) * args.sq_stride + r] = sq;
                sq = 0.f;
              }
              if (c & 1) {  // a 64-column box is complete: store it
                fence_proxy_async();
                named_bar_sync(2, 128);
                if (leader) {
                  tma_store_2d(&tmO, sR + (c >> 1) * GEMM_BM * 128, n0 + (c >> 1) * 64, mb * TM + (int)rank * GEMM_BM);
                  bulk_commit();
                }
              }
            }
            break;
          }
          // sum-of-squares partials in 128-column units (independent of the tile width)
          float sq = 0.f;
          // residual loads run one 32-column chunk ahead of their use
          uint4 rnext[4];
          auto ld_resid = [&](int c) {
            if (valid && n0 + c * 32 < N) {
              const uint4* src = reinterpret_cast<const uint4*>(args.resid + (int64_t)r * args.ldr + n0 + c * 32);
#pragma unroll
              for (int q = 0; q < 4; ++q) rnext[q] = src[q];
            }
          };
          ld_resid(0);
#pragma unroll 1
          for (int c = 0; c < BN / 32; ++c) {
            uint4 rcur[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) rcur[q] = rnext[q];
            if (c + 1 < BN / 32) ld_resid(c + 1);
            ldacc(c * 32, s, v);
            const int col = n0 + c * 32;
            if (valid && col < N) {
              float rr[32];
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const float2 a = unpack_bf16x2(rcur[q].x), b = unpack_bf16x2(rcur[q].y);
                const float2 c2 = unpack_bf16x2(rcur[q].z), d = unpack_bf16x2(rcur[q].w);
                rr[q * 8 + 0] = a.x; rr[q * 8 + 1] = a.y; rr[q * 8 + 2] = b.x; rr[q * 8 + 3] = b.y;
                rr[q * 8 + 4] = c2.x; rr[q * 8 + 5] = c2.y; rr[q * 8 + 6] = d.x; rr[q * 8 + 7] = d.y;
              }
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                v[j] = round_bf16(rr[j] + v[j]);
                sq = fmaf(v[j], v[j], sq);
              }
              if constexpr (PEER) {  // all-gather fused into the epilogue: the row segment to every rank
                for (int q = 0; q < args.peer_n; ++q) store32_bf16(peer_ag_row(args, (args.peer_rank + 1 + q) % args.peer_n, r) + col, v);
              } else {
                store32_bf16(args.out + (int64_t)r * args.ldo + col, v);
              }
            }
            if ((c & 3) == 3) {
              if (args.sq_out != nullptr && valid) args.sq_out[(int64_t)((n0 >> 7) + (c >> 2)) * args.sq_stride + r] = sq;
              sq = 0.f;
            }
          }
          if constexpr (PEER) {
            asm volatile("fence.acq_rel.sys;" ::: "memory");  // this thread's peer stores before the counters
            named_bar_sync(1, 128);
            if (trow == 0) peer_ag_signal(args, mb * CG + (int)rank, n0, BN);
          }
          break;
        }
        case EPI_SILU: {
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            float u[32];
            ldacc(c * 32, s, v);
            ldacc(128 + c * 32, s, u);
            const int col = nb * 128 + c * 32;
            if (valid && col < args.n_valid) {
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                const float g = v[j];
                v[j] = g / (1.f + __expf(-g)) * u[j];
              }
              store32_bf16(args.out + (int64_t)r * args.ldo + col, v);
            }
          }
          break;
        }
        case EPI_QKV: {
          const int hd = args.hd, qh = args.qh, kh = args.kh;
          const int hpt = BN / hd;
          const int pos = valid ? args.tok_pos[r] : 0;
          const int slot = valid ? args.tok_slot[r] : 0;
          const int64_t page = slot / args.page_size, off = slot % args.page_size;
#pragma unroll 1
          for (int hh = 0; hh < hpt; ++hh) {
            const int gh = nb * hpt + hh;
            if (gh >= qh + 2 * kh) break;
            __nv_bfloat16* dst;
            if (gh < qh) {
              dst = args.q_out + (int64_t)r * qh * hd + (int64_t)gh * hd;
            } else {
              const int kv = gh < qh + kh ? 0 : 1;
              const int kvh = gh - qh - kv * kh;
              dst = args.kv_pool + (((page * 2 + kv) * kh + kvh) * args.page_size + off) * hd;
            }
            if (gh >= qh + kh) {  // V: no rotation
#pragma unroll 1
              for (int c = 0; c < hd / 32; ++c) {
                ldacc(hh * hd + c * 32, s, v);
                if (valid) store32_bf16(dst + c * 32, v);
              }
            } else {  // Q or K: rotate-half RoPE at pos (reading A-4)
#pragma unroll 1
              for (int c = 0; c < hd / 64; ++c) {
                float x2[32];
                ldacc(hh * hd + c * 32, s, v);
                ldacc(hh * hd + hd / 2 + c * 32, s, x2);
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                  float sn, cs;
                  sincos_reduced((float)pos * inv_freq[c * 32 + j], &sn, &cs);
                  const float a = v[j], b = x2[j];
                  v[j] = a * cs - b * sn;
                  x2[j] = b * cs + a * sn;
                }
                if (valid) {
                  store32_bf16(dst + c * 32, v);
                  store32_bf16(dst + hd / 2 + c * 32, x2);
                }
              }
            }
          }
          break;
        }
        case EPI_ARGMAX: {
          float best = -INFINITY;
          int bi = 0x7fffffff;
#pragma unroll 1
          for (int c = 0; c < BN / 32; ++c) {
            ldacc(c * 32, 1.f, v);
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int col = n0 + c * 32 + j;
              if (col < N && v[j] > best) { best = v[j]; bi = col; }
            }
          }
          if (valid) {
            args.am_val[(int64_t)nb * args.am_stride + r] = best;
            args.am_idx[(int64_t)nb * args.am_stride + r] = bi;
          }
          break;
        }
        default:
          break;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 2) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[as]), 0));
        else mbar_arrive(&tempty[as]);
      }
      as ^= 1;
      if (as == 0) aphase ^= 1;
    });
  }
  if (warp == 4 && lane == 0) gemm_ts(4);  // epilogue done
  if constexpr (SR) {
    if (warp == 4 && lane == 0) bulk_wait0();  // the last tile's stores are complete
  }
  __syncthreads();
  if constexpr (CG == 2) cluster_sync();  // the peer's remote arrives / MMA writes are done before teardown
  if (warp == 2) {
    tc_fence_after();
    if constexpr (CG == 2) tmem_dealloc_cg2(tmem_base, TMEM_COLS);
    else tmem_dealloc(tmem_base, TMEM_COLS);
    if (lane == 0) gemm_ts(5);  // teardown done
  }
}

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_once;
bool g_attr_set[12] = {};

cudaError_t get_encode() {
  std::call_once(g_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode ? cudaSuccess : cudaErrorNotSupported;
}

}  // namespace

// 2D bf16 tensor map [outer rows, inner cols] with 128B swizzle.
cudaError_t make_tmap_bf16(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld_elems,
                           uint32_t box_inner, uint32_t box_outer) {
  cudaError_t e = get_encode();
  if (e != cudaSuccess) return e;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld_elems * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// Slot-layout A (GemmArgs::a_slots): dims (slot width, rows, slots), box (box_inner, box_rows, 1)
cudaError_t make_tmap_slots_bf16(CUtensorMap* m, const void* ptr, uint64_t slot_w, uint64_t rows, uint64_t slots,
                                 uint32_t box_inner, uint32_t box_rows) {
  cudaError_t e = get_encode();
  if (e != cudaSuccess) return e;
  cuuint64_t dims[3] = {slot_w, rows, slots};
  cuuint64_t strides[2] = {slot_w * 2, rows * slot_w * 2};
  cuuint32_t box[3] = {box_inner, box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// Paged-KV page map: dims (64 cols, rows, half, kv) so one box {64, 16, hd/64, 2} = one page's
// K and V block of one KV head (hd*16*2*2 bytes) lands as [kv][half][16 rows][128 B], 128B-swizzled.
cudaError_t make_page_tmap(CUtensorMap* m, const void* pool, int64_t n_pages, int kh, int hd, int page_size) {
  cudaError_t e = get_encode();
  if (e != cudaSuccess) return e;
  const uint64_t rows = (uint64_t)n_pages * 2 * kh * page_size;
  cuuint64_t dims[4] = {64, rows, (cuuint64_t)(hd / 64), 2};
  cuuint64_t strides[3] = {(cuuint64_t)hd * 2, 128, (cuuint64_t)kh * page_size * hd * 2};
  cuuint32_t box[4] = {64, (cuuint32_t)page_size, (cuuint32_t)(hd / 64), 2};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(pool), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t make_q_tmap(CUtensorMap* m, const void* q, int64_t T, int qh, int hd) {
  cudaError_t e = get_encode();
  if (e != cudaSuccess) return e;
  cuuint64_t dims[3] = {(cuuint64_t)hd, (cuuint64_t)qh, (cuuint64_t)T};
  cuuint64_t strides[2] = {(cuuint64_t)hd * 2, (cuuint64_t)qh * hd * 2};
  cuuint32_t box[3] = {64, 1, 128};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(q), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t launch_gemm(const __nv_bfloat16* A, int64_t lda, const __nv_bfloat16* B, int64_t ldb,
                        const GemmArgs& args, int sm_budget, cudaStream_t stream) {
  if (args.M <= 0) return cudaSuccess;
  // Tile width: 128x256.  A 128x128 variant (6-stage ring, NF_GEMM_BN=128)
  // halves wave quantisation for nano-batch-sized GEMMs but measured slower:
  // with a 1-CTA N=128 MMA the A+B smem reads reach the smem bandwidth.
  // SiLU / argmax epilogues need the 256-wide tile layout.
  static int bn_env = -1, stages_env = -1, cg2_env = -1;
  if (bn_env < 0) {
    const char* e = getenv("NF_GEMM_BN");
    bn_env = e ? atoi(e) : 0;
    e = getenv("NF_GEMM_STAGES");  // (dev) NF_GEMM_STAGES=3 forces the shallow ring, for interference A/B
    stages_env = e ? atoi(e) : 0;
    e = getenv("NF_GEMM_CG2");     // CTA-pair kernel (default on; 0 = single-CTA tiles only)
    cg2_env = e ? atoi(e) : 1;
  }
  const bool need256 = args.epi == EPI_SILU || args.epi == EPI_ARGMAX;  // tile-layout-dependent epilogues
  const int bn = (bn_env == 128 && !need256) ? 128 : 256;
  const bool coloc = args.stages == 3 || stages_env == 3;
  const int tiles = ((args.M + GEMM_BM - 1) / GEMM_BM) * ((args.N + bn - 1) / bn);
  int grid = tiles < sm_budget ? tiles : sm_budget;
  GemmArgs a2 = args;
  // Schedule choice by tile-rounds (cost in units of one 128-row tile's mainloop per CTA):
  //   data-parallel        ceil(tiles / SB)
  //   CTA pairs            ceil(pair_tiles / (SB/2)) for 256-row pair tiles (6-stage ring, B shared)
  //   split-K tail (s)     floor(tiles / SB) + 1/s for the partial last wave, s = min(4, SB / rem)
  //                        splits of >= 32 k-blocks each (also covers sub-wave GEMMs; 16 measured
  //                        slower for K = 4096 under overlap: the fp32 fix-up outweighs the gain)
  //   split-K=2            ceil(2 tiles / SB) / 2, for K >= 8192 (a half tile must outweigh
  //                        writing + reading its 128 KB fp32 partial; measured on O vs Down)
  // Ties prefer CTA pairs (long-K, wide-N GEMMs only), then the simpler schedule.  NF_STREAMK=0 / NF_SPLITK=0 / NF_GEMM_CG2=0
  // disable a schedule (A/B runs).
  const int num_kb = (args.K + GEMM_BK - 1) / GEMM_BK;
  static int split_env = -1, tail_env = -1;
  if (split_env < 0) {
    const char* e = getenv("NF_SPLITK");
    split_env = e ? atoi(e) : 1;
    e = getenv("NF_STREAMK");
    tail_env = e ? atoi(e) : 1;
  }
  const int SB = std::max(1, sm_budget);
  // (dev) NF_GEMM_FORCE=k: schedule k wins whenever it is feasible (A/B of schedules)
  static int force_env = -2;
  if (force_env == -2) {
    const char* e = getenv("NF_GEMM_FORCE");
    force_env = e ? atoi(e) : -1;
  }
  auto bias = [&](int k) { return force_env == k ? -1000.0 : 0.0; };
  double best = (double)((tiles + SB - 1) / SB) + bias(0);
  int choice = 0, best_s = 1;
  const bool grouped = args.grp_off != nullptr;
  // (grouped: device-sized tile list, data-parallel or device-decided stream-K tail only)
  if (!grouped && tail_env && args.sk_part != nullptr && args.sk_slots >= SB) {
    const int rem = tiles % SB;
    if (rem > 0) {
      int s = std::min(4, SB / rem);
      while (s > 1 && num_kb / s < 32) --s;
      const double c = tiles / SB + 1.0 / s + bias(1);
      if (s > 1 && c < best - 1e-9) { best = c; choice = 1; best_s = s; }
    }
  }
  const int g2 = std::min(SB, 2 * tiles);
  const double rounds2 = ((2 * tiles + g2 - 1) / g2) / 2.0 + bias(2);
  if (!grouped && split_env && args.sk_part != nullptr && args.sk_slots >= tiles && num_kb >= 128 && rounds2 < best - 1e-9 &&
      args.epi != EPI_SILU && args.epi != EPI_ARGMAX) {
    best = rounds2;
    choice = 2;
  }
  const bool aslots = args.a_slots > 1;  // slot-layout A: single-CTA schedules only
  if (aslots && (args.a_slot_w % GEMM_BK != 0 || (int64_t)args.a_slots * args.a_slot_w != args.K || grouped))
    return cudaErrorInvalidValue;
  const int pairs = SB / 2;
  const int pair_tiles = ((args.M + 2 * GEMM_BM - 1) / (2 * GEMM_BM)) * ((args.N + bn - 1) / bn);
  int pair_s = 1;
  if (!grouped && !aslots && cg2_env && bn == 256 && !coloc && pairs >= 1) {
    // on a tie the pair kernel measured faster only with a long mainloop and many n-tiles
    // (>= 32 k-blocks, N >= 2048; tools/gemm_micro.py): short-K pairs couple the two CTAs'
    // epilogues through the shared accumulator barrier
    // (dev) NF_GEMM_PAIR_MINN raises the N threshold of the tie rule (A/B of single-CTA tiles on
    // the narrow-N GEMMs: O, Down, KQV)
    static int pair_min_n = -1;
    if (pair_min_n < 0) {
      const char* e2 = getenv("NF_GEMM_PAIR_MINN");
      pair_min_n = e2 ? atoi(e2) : 2048;
    }
    const bool tie_ok = num_kb >= 32 && args.N >= pair_min_n;
    double c = (double)((pair_tiles + pairs - 1) / pairs) + bias(3);
    // pairs with a split-K tail (same rule as single CTAs, pair tiles over pairs)
    const int rem = pair_tiles % pairs;
    if (tail_env && rem > 0 && args.sk_part != nullptr && args.sk_slots >= SB && pair_tiles > pairs / 4) {
      int s = std::min(4, pairs / rem);
      while (s > 1 && num_kb / s < 32) --s;
      const double ct = pair_tiles / pairs + 1.0 / s;
      if (s > 1 && ct < c - 1e-9) {
        c = ct;
        pair_s = s;
      }
    }
    if (c < best - 1e-9 || (tie_ok && c <= best + 1e-9)) {
      best = c;
      choice = 3;
    }
  }
  // stream-K for sub-wave GEMMs (fewer tiles than SMs): the work spreads over G CTAs
  // with >= 16 k-blocks each; cost = work per CTA in tile rounds + a fix-up allowance
  // Only when A and B fit in L2 together (<= 64 MB): stream-K staggers the CTAs in K,
  // so the weight k-blocks are no longer read in lockstep by the m-tiles (Down of the
  // 8B nano-batch, 117 MB of weights, measured 1.6x slower); and only with a clear
  // margin, since every split tile pays an fp32 partial round trip and a second epilogue
  // (the 8B nano-batch O projection, 0.86 of a wave, measured 1.3x slower).
  int sk_grid = 0;
  const double l2_mb = ((double)args.N * args.K + (double)args.M * args.K) * 2.0 / 1048576.0;
  if (!grouped && tail_env && args.sk_part != nullptr && args.sk_slots >= SB && tiles < SB && !coloc && l2_mb <= 64.0) {
    const int64_t U = (int64_t)tiles * num_kb;
    const int G = (int)std::min<int64_t>(SB, std::max<int64_t>(tiles, U / 16));
    const double c = (double)U / ((double)G * num_kb) + 0.3 + bias(4);
    if (G > tiles && c < best - 1e-9) {
      best = c;
      choice = 4;
      sk_grid = G;
    }
  }
  // CTA pairs + stream-K (sub-wave in pair tiles): each CTA fetches half the B bytes per
  // k-block
  int skp_grid = 0;
  if (!grouped && !aslots && cg2_env && bn == 256 && tail_env && args.sk_part != nullptr && args.sk_slots >= SB &&
      pair_tiles < pairs && !coloc && l2_mb <= 64.0) {
    const int64_t U = (int64_t)pair_tiles * num_kb;
    const int G = (int)std::min<int64_t>(pairs, std::max<int64_t>(pair_tiles, U / 16));
    const double c = (double)U / ((double)G * num_kb) + 0.3 + bias(5);
    // measured no faster than single-CTA stream-K on the 70B-rank KQV (r1c_gemm_micro_streamk_pairs.log:
    // 900 vs 912 TF/s at M 2048, 626 vs 672 at M 1024): taken only when clearly better
    if (G > pair_tiles && c < best - 0.05) {
      best = c;
      choice = 5;
      skp_grid = G;
    }
  }
  static int sks_env = -1;
  if (sks_env < 0) {
    // (dev) NF_GEMM_SKSMEM=1: the owner of a split tile stages its first contributor's partial in the
    // idle stage ring (one bulk copy) instead of reading it chunk by chunk from L2.  Off by default:
    // shape-dependent, +13 % on the 70B-rank O_col, -7 % on the 70B-rank Up/Gate at M 1024
    // (profiles/r2l_sksmem_*.log)
    const char* e2 = getenv("NF_GEMM_SKSMEM");
    sks_env = e2 ? atoi(e2) : 0;
  }
  a2.sk_smem = sks_env;
  a2.stream_k = (choice == 4 || choice == 5) ? 1 : 0;
  if (grouped && tail_env && args.sk_part != nullptr && args.sk_slots >= SB && !coloc) a2.stream_k = 2;
  a2.split = choice == 2 ? 2 : 1;
  a2.tail_split = choice == 1 ? best_s : (choice == 3 ? pair_s : 1);
  if (choice == 1) grid = SB;
  if (choice == 4) grid = sk_grid;
  if (choice == 2) grid = g2;
  if ((choice == 0 && a2.stream_k != 2) || (choice == 3 && pair_s == 1)) a2.sk_part = nullptr;
  if (grid < 1) grid = 1;
  CUtensorMap ta, tb;
  cudaError_t e = aslots ? make_tmap_slots_bf16(&ta, A, args.a_slot_w, args.M, args.a_slots, GEMM_BK, GEMM_BM)
                         : make_tmap_bf16(&ta, A, args.K, args.M, lda, GEMM_BK, GEMM_BM);
  if (e != cudaSuccess) return e;
  const bool pair_kernel = choice == 3 || choice == 5;
  e = make_tmap_bf16(&tb, B, args.K, (uint64_t)args.N * (grouped ? args.n_groups : 1), ldb, GEMM_BK,
                     pair_kernel ? bn / 2 : bn);
  if (e != cudaSuccess) return e;
  // smem ring: 4 x 48 KB (BN 256), 6 x 32 KB (BN 128 or CTA pairs); co-located plans use 3 / 4 stages.
  // Short-K residual / plain-store GEMMs (EPI_RESID / EPI_STORE bf16, K <= 2048: the 3-stage ring
  // costs 8-34 % on long mainloops, tools/gemm_micro.py r2f) stage the output tile
  // (and the residual) in smem and TMA-store it (SR): 3 x 48 KB (or pairs 4 x 32 KB) + 64 KB.
  // NF_GEMM_SR=0 disables it, NF_GEMM_SR_MAXKB caps its K (A/B runs).
  static int sr_env = -1;
  if (sr_env < 0) {
    const char* e2 = getenv("NF_GEMM_SR");
    sr_env = e2 ? atoi(e2) : 1;
  }
  static int sr_kb_env = -1;
  if (sr_kb_env < 0) {
    const char* e2 = getenv("NF_GEMM_SR_MAXKB");
    sr_kb_env = e2 ? atoi(e2) : 32;
  }
  const bool peer = args.epi == EPI_PEER || args.peer_mode == 1;  // fused reduce-scatter / all-gather epilogues
  const bool sr = sr_env && (args.epi == EPI_RESID || (args.epi == EPI_STORE && args.outf == nullptr)) && bn == 256 &&
                  !grouped && !coloc && num_kb <= sr_kb_env && !peer;
  int stages, cg = 1;
  void (*kern)(CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, GemmArgs);
  int attr_idx;
  if (pair_kernel) {
    stages = sr ? 4 : 6;
    cg = 2;
    kern = sr ? gemm_tcgen05_kernel<4, 256, 2, true>
              : (peer ? gemm_tcgen05_kernel<6, 256, 2, false, true> : gemm_tcgen05_kernel<6, 256, 2>);
    attr_idx = sr ? 6 : (peer ? 7 : 4);
  } else if (bn == 256) {
    stages = sr ? 3 : (coloc ? 3 : 4);
    if (peer)
      kern = coloc ? gemm_tcgen05_kernel<3, 256, 1, false, true> : gemm_tcgen05_kernel<4, 256, 1, false, true>;
    else
      kern = sr ? gemm_tcgen05_kernel<3, 256, 1, true>
                : (coloc ? gemm_tcgen05_kernel<3, 256, 1> : gemm_tcgen05_kernel<4, 256, 1>);
    attr_idx = sr ? 5 : (peer ? (coloc ? 8 : 9) : (coloc ? 1 : 0));
  } else {
    stages = coloc ? 4 : 6;
    if (peer)
      kern = coloc ? gemm_tcgen05_kernel<4, 128, 1, false, true> : gemm_tcgen05_kernel<6, 128, 1, false, true>;
    else
      kern = coloc ? gemm_tcgen05_kernel<4, 128, 1> : gemm_tcgen05_kernel<6, 128, 1>;
    attr_idx = peer ? (coloc ? 10 : 11) : (coloc ? 3 : 2);
  }
  const int smem = gemm_smem_bn(stages, bn / cg) + (sr ? bn * GEMM_BM * 2 : 0);
  CUtensorMap tr = ta, to = ta;
  if (sr) {
    if (args.epi == EPI_RESID) {
      e = make_tmap_bf16(&tr, args.resid, args.N, args.M, args.ldr, 64, GEMM_BM);
      if (e != cudaSuccess) return e;
    }
    e = make_tmap_bf16(&to, args.out, args.N, args.M, args.ldo, 64, GEMM_BM);
    if (e != cudaSuccess) return e;
  }
  if (!g_attr_set[attr_idx]) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    g_attr_set[attr_idx] = true;
  }
  // Programmatic dependent launch (opt-in, NF_PDL=1): the kernel's prologue overlaps the
  // tail of the previous kernel on the stream; it waits (griddepcontrol.wait) before
  // touching any global data.  Measured neutral on the bench steps (profiles/r1c_pdl_ab.log:
  // 8B and 70B-rank steps within run-to-run noise), so it is off by default.
  static int pdl_env = -1;
  if (pdl_env < 0) {
    const char* pe = getenv("NF_PDL");
    pdl_env = pe ? atoi(pe) : 0;
  }
  if (cg == 2) grid = 2 * (choice == 5 ? skp_grid : (pair_s > 1 ? pairs : std::min(pair_tiles, pairs)));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(GEMM_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (cg == 2) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 2;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl_env) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  e = cudaLaunchKernelEx(&cfg, kern, ta, tb, tr, to, a2);
  count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

#ifdef NF_GEMM_TS
extern "C" int nf_debug_gemm_ts(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_gemm_ts, sizeof(g_gemm_ts));
}
#endif

// One kernel of this translation unit (preload_all_kernels: its module is loaded eagerly).
const void* kernel_anchor_gemm() { return reinterpret_cast<const void*>(gemm_tcgen05_kernel<4, 256, 1>); }

}  // namespace nf
