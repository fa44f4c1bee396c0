// Diagnostic: per-SM HBM streaming ceiling with TMA (no compute).  Each CTA
// (one per SM) streams random 8 KB pages (the decode kernel's K+V page box)
// through an NS-deep smem ring and immediately re-issues.  Built by
// tools/tma_probe.py as a separate .so (not part of libnf).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// MODE 0: one 4-D tensor box (K and V of the page, 128B-swizzled); 1: two 1-D bulk copies of the
// contiguous 4 KB K and V blocks; 2: mode 0 plus an L2 prefetch (tensor) 4 pages ahead.
template <int NS, int WARPS, int MODE>
__global__ void __launch_bounds__(WARPS * 32, 1) probe_kernel(const __grid_constant__ CUtensorMap map,
                                                              const int* __restrict__ page_of, int n_pages_total,
                                                              int pages_per_warp, unsigned long long* sink,
                                                              const uint8_t* pool) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = smem + warp * NS * 8192;
  uint64_t* bars = (uint64_t*)(smem + WARPS * NS * 8192) + warp * NS;
  if (lane == 0) {
    for (int s = 0; s < NS; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  const int gw = blockIdx.x * WARPS + warp;
  auto issue = [&](int i) {
    const int s = i % NS;
    const int page = page_of[(gw * pages_per_warp + i) % n_pages_total];
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 8192;" ::"r"(su32(&bars[s])));
    if (MODE == 1) {
      const uint8_t* src = pool + (size_t)page * 8192;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 4096, [%2];" ::"r"(
                       su32(ring + s * 8192)), "l"(src), "r"(su32(&bars[s])) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 4096, [%2];" ::"r"(
                       su32(ring + s * 8192 + 4096)), "l"(src + 4096), "r"(su32(&bars[s])) : "memory");
    } else {
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
          "%5}], [%6];" ::"r"(su32(ring + s * 8192)),
          "l"((uint64_t)&map), "r"(0), "r"(page * 16), "r"(0), "r"(0), "r"(su32(&bars[s]))
          : "memory");
      if (MODE == 2) {
        const int pf = page_of[(gw * pages_per_warp + i + 4) % n_pages_total];
        asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];" ::"l"((uint64_t)&map),
                     "r"(0), "r"(pf * 16), "r"(0), "r"(0) : "memory");
      }
    }
  };
  // MODE 3/4: every lane prefetches its 256 B of the page PFD pages ahead into L2 (LSU, not TMA)
  constexpr int PFD = MODE == 4 ? 8 : 4;
  auto lsu_prefetch = [&](int i) {
    const int pf = page_of[(gw * pages_per_warp + i) % n_pages_total];
    const uint8_t* src = pool + (size_t)pf * 8192 + lane * 256;
    asm volatile("prefetch.global.L2 [%0];" ::"l"(src));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(src + 128));
  };
  if (MODE >= 3)
    for (int i = NS; i < NS + PFD; ++i) lsu_prefetch(i);
  if (lane == 0)
    for (int i = 0; i < NS && i < pages_per_warp; ++i) issue(i);
  unsigned long long acc = 0;
  for (int i = 0; i < pages_per_warp; ++i) {
    const int s = i % NS;
    const uint32_t par = (i / NS) & 1;
    asm volatile(
        "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 10000000;\n\t@!p bra "
        "W_%=;\n\t}" ::"r"(su32(&bars[s])),
        "r"(par)
        : "memory");
    acc += ring[s * 8192 + lane * 4];
    __syncwarp();
    if (MODE >= 3 && i + NS + PFD < pages_per_warp) lsu_prefetch(i + NS + PFD);
    if (lane == 0 && i + NS < pages_per_warp) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(i + NS);
    }
  }
  if (acc == 0x7fffffffffffULL) *sink = acc;
}

template <int NS, int W, int MODE>
void launch_probe(const CUtensorMap& m, const int* page_of, int n_pages_total, int grid, int ppw,
                  unsigned long long* sink, const uint8_t* pool) {
  const int smem = W * NS * 8192 + W * NS * 8 + 1024;
  cudaFuncSetAttribute(probe_kernel<NS, W, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe_kernel<NS, W, MODE><<<grid, W * 32, smem>>>(m, page_of, n_pages_total, ppw, sink, pool);
}

extern "C" int probe_run(void* pool, long long n_pages, const int* page_of, int n_pages_total, int grid, int warps,
                         int ns, int pages_per_warp, float* ms_out, int mode) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  }
  CUtensorMap m;
  // pool [n_pages][2][1][16][128] bf16 with one KV head: page = 64 rows of 128 cols (K and V of the head)
  cuuint64_t dims[4] = {64, (cuuint64_t)n_pages * 2 * 16, 2, 2};
  cuuint64_t strides[3] = {256, 128, 16 * 256};
  cuuint32_t box[4] = {64, 16, 2, 2};
  cuuint32_t es[4] = {1, 1, 1, 1};
  if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, pool, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
      CUDA_SUCCESS)
    return 1;
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  auto launch = [&]() {
    const uint8_t* pl = (const uint8_t*)pool;
#define P(NS_, W_)                                                                                     \
  if (ns == NS_ && warps == W_) {                                                                      \
    if (mode == 1) launch_probe<NS_, W_, 1>(m, page_of, n_pages_total, grid, pages_per_warp, sink, pl); \
    else if (mode == 2) launch_probe<NS_, W_, 2>(m, page_of, n_pages_total, grid, pages_per_warp, sink, pl); \
    else if (mode == 3) launch_probe<NS_, W_, 3>(m, page_of, n_pages_total, grid, pages_per_warp, sink, pl); \
    else if (mode == 4) launch_probe<NS_, W_, 4>(m, page_of, n_pages_total, grid, pages_per_warp, sink, pl); \
    else launch_probe<NS_, W_, 0>(m, page_of, n_pages_total, grid, pages_per_warp, sink, pl);          \
    return;                                                                                            \
  }
    P(1, 8) P(2, 8) P(3, 8) P(2, 12) P(2, 13) P(4, 6) P(6, 4) P(1, 24) P(2, 4)
#undef P
  };
  launch();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(ms_out, a, b);
  cudaFree(sink);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
