// Owner-side reduce + all-gather of a fused GEMM->AllReduce site (peer.cuh).
#include <cuda.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "peer.cuh"
#include "profile.h"

namespace nf {

PeerGeom peer_geom(int n, int rank, int max_rows, int cols) {
  PeerGeom g;
  g.n = n;
  g.rank = rank;
  g.max_rows = max_rows;
  g.cols = cols;
  const int mb = (max_rows + PEER_BM - 1) / PEER_BM, nb = cols / PEER_BN;
  g.maxb = mb * nb;
  g.maxown = (g.maxb + n - 1) / n;
  auto al = [](int64_t v) { return (v + 4095) / 4096 * 4096; };
  g.flags_off = 0;
  g.stage_off = al(256 + 4 * (int64_t)g.maxown * n);
  g.result_off = g.stage_off + al((int64_t)n * g.maxown * PEER_BM * PEER_BN * 2);
  g.site_bytes = g.result_off + al((int64_t)max_rows * cols * 2);
  g.total_bytes = PEER_CTL_BYTES + (int64_t)PEER_SITES * g.site_bytes;
  return g;
}

namespace {

NF_DEV uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
NF_DEV void red_release_sys_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
NF_DEV void fence_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
NF_DEV uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
NF_DEV uint4 ld_cg_u4(const void* p) {
  uint4 v;
  asm volatile("ld.global.cg.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

// Bounded wait for *p >= target (one thread).  On timeout: error word += 1, a diagnostic
// record {site, what (0 flag / 1 done), index, observed, target} in the header, returns false.
NF_DEV bool wait_geq(const uint32_t* p, uint32_t target, uint32_t* err, long long timeout_ns, int site, int what,
                     int index) {
  if (ld_acquire_sys(p) >= target) return true;
  const uint64_t t0 = globaltimer();
  uint32_t v;
  while ((v = ld_acquire_sys(p)) < target) {
    atomicMax(err + 8 + what, (uint32_t)((globaltimer() - t0) / 1000));  // longest wait so far (us), per kind
    __nanosleep(64);
    if ((long long)(globaltimer() - t0) > timeout_ns) {
      const uint32_t k = atomicAdd(err, 1u);
      if (k < 16) {
        uint32_t* rec = err + 16 + 8 * k;
        rec[0] = site; rec[1] = what; rec[2] = index; rec[3] = v; rec[4] = target;
      }
      return false;
    }
  }
  return true;
}

// 128 threads and <= 64 registers (8 K registers, no shared memory): a reduce CTA spinning on an
// SM leaves room for a whole GEMM CTA (256 threads x <= 224 registers = 57 K of the 64 K
// register file) -- the fused path only runs where the reduce cannot hold SMs a producer needs
// (fused_site_ok in api.cu), this keeps even a co-resident reduce harmless.
constexpr int PR_THREADS = 128;
constexpr int PR_U = 4;  // 16-byte chunks per thread per pass (memory-level parallelism)
__global__ void __launch_bounds__(PR_THREADS, 8) peer_reduce_kernel(uint8_t* const* __restrict__ bases, PeerGeom g, int site,
                                                          int M, long long timeout_ns) {
  const int P = g.n, me = g.rank;
  const int MB = (M + PEER_BM - 1) / PEER_BM, NB = g.cols / PEER_BN, nblk = MB * NB;
  uint8_t* mine = bases[me];
  uint32_t* err = reinterpret_cast<uint32_t*>(mine);
  uint8_t* s_mine = mine + g.site(site);
  uint32_t* done = reinterpret_cast<uint32_t*>(s_mine + g.flags_off);
  uint32_t* flags = reinterpret_cast<uint32_t*>(s_mine + g.flags_off + 256);
  const __nv_bfloat16* stage = reinterpret_cast<const __nv_bfloat16*>(s_mine + g.stage_off);
  const int n_own = (nblk - me + P - 1) / P;  // blocks me, me+P, ...
  for (int lb = blockIdx.x; lb < n_own; lb += gridDim.x) {
    const int blk = lb * P + me;
    const int bm = blk % MB, bn = blk / MB;
    const int rows = min(PEER_BM, M - bm * PEER_BM);
    if (threadIdx.x == 0) {
      for (int src = 0; src < P; ++src) {  // one flag per (owned block, source rank)
        wait_geq(&flags[lb * P + src], 4u, err, timeout_ns, site, 0, lb * 16 + src);
        flags[lb * P + src] = 0;  // cleared before this block's broadcast: no producer can add to it before then
      }
    }
    __syncthreads();
    // 128 rows x 32 chunks of 8 bf16: consecutive threads take consecutive 16 B of a row
    // 128 rows x 32 chunks of 8 bf16; each thread takes PR_U chunks per pass (consecutive threads
    // -> consecutive 16 B of a row), all PR_U loads of a source issued before their adds
    uint8_t* const* bp = bases;
    const int64_t rbase = g.site(site) + g.result_off;
    for (int i0 = threadIdx.x; i0 < PEER_BM * (PEER_BN / 8); i0 += PR_U * blockDim.x) {
      float acc[PR_U][8];
#pragma unroll
      for (int u = 0; u < PR_U; ++u)
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[u][e] = 0.f;
#pragma unroll 2
      for (int src = 0; src < P; ++src) {  // rank order: the emulated NF_AR_F32 arithmetic
        const __nv_bfloat16* sp = stage + ((int64_t)src * g.maxown + lb) * PEER_BM * PEER_BN;
        uint4 w[PR_U];
#pragma unroll
        for (int u = 0; u < PR_U; ++u) {
          const int i = i0 + u * blockDim.x, row = i >> 5, ch = i & 31;
          w[u] = row < rows ? ld_cg_u4(sp + row * PEER_BN + ch * 8) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < PR_U; ++u) {
          const uint32_t ww[4] = {w[u].x, w[u].y, w[u].z, w[u].w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float2 f = unpack_bf16x2(ww[k]);
            acc[u][2 * k] += f.x;
            acc[u][2 * k + 1] += f.y;
          }
        }
      }
#pragma unroll
      for (int u = 0; u < PR_U; ++u) {
        const int i = i0 + u * blockDim.x, row = i >> 5, ch = i & 31;
        if (row >= rows) continue;
        const uint4 o = make_uint4(pack_bf16x2(acc[u][0], acc[u][1]), pack_bf16x2(acc[u][2], acc[u][3]),
                                   pack_bf16x2(acc[u][4], acc[u][5]), pack_bf16x2(acc[u][6], acc[u][7]));
        const int64_t off = rbase + (((int64_t)(bm * PEER_BM + row)) * g.cols + bn * PEER_BN + ch * 8) * 2;
        for (int q = 0; q < P; ++q) {  // all-gather: start with the next rank so the links are spread
          const int p = (me + 1 + q) % P;
          *reinterpret_cast<uint4*>(bp[p] + off) = o;
        }
      }
    }
    fence_sys();
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int q = 0; q < P; ++q) {
        const int p = (me + 1 + q) % P;
        red_release_sys_add(reinterpret_cast<uint32_t*>(bases[p] + g.site(site) + g.flags_off), 1u);
      }
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    wait_geq(done, (uint32_t)nblk, err, timeout_ns, site, 1, 0);  // every owner's blocks have landed here
    *done = 0;
    fence_sys();
  }
}

// Consumer side of the fused all-gather (EPI_RESID peer_mode 1): wait until every rank's
// producer units have landed here (the site's `done` counter reaches `expected`), clear it.
__global__ void peer_wait_kernel(uint8_t* const* __restrict__ bases, PeerGeom g, int site, uint32_t expected,
                                 long long timeout_ns) {
  uint8_t* mine = bases[g.rank];
  uint32_t* done = reinterpret_cast<uint32_t*>(mine + g.site(site) + g.flags_off);
  wait_geq(done, expected, reinterpret_cast<uint32_t*>(mine), timeout_ns, site, 2, 0);
  *done = 0;
  fence_sys();
}

}  // namespace

cudaError_t launch_peer_wait(uint8_t* const* bases, const PeerGeom& g, int site, uint32_t expected, long long timeout_ns,
                             cudaStream_t st) {
  if (site < 0 || site >= PEER_SITES) return cudaErrorInvalidValue;
  peer_wait_kernel<<<1, 32, 0, st>>>(bases, g, site, expected, timeout_ns);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_peer_reduce(uint8_t* const* bases, const PeerGeom& g, int site, int M, int ctas,
                               long long timeout_ns, cudaStream_t st) {
  if (M <= 0) return cudaSuccess;
  if (M > g.max_rows || site < 0 || site >= PEER_SITES) return cudaErrorInvalidValue;
  const int MB = (M + PEER_BM - 1) / PEER_BM, NB = g.cols / PEER_BN;
  const int n_own = (MB * NB + g.n - 1) / g.n;
  const int grid = std::max(1, std::min(ctas, n_own));
  peer_reduce_kernel<<<grid, PR_THREADS, 0, st>>>(bases, g, site, M, timeout_ns);
  count_launch();
  return cudaGetLastError();
}

// Spin-waiting kernels (peer_reduce) must never wait on a kernel that is not loaded yet in
// the context it is launched in: under CUDA lazy loading the first launch of a function in a
// context can require that context to be idle, which a spinning kernel prevents (and every
// green context of a plan is a context of its own).  So every kernel of the library is
// loaded into the primary context when the fused path is switched on and into each green
// context when it is created (cuLibraryEnumerateKernels + cuKernelGetFunction + cuFuncLoad).
const void* kernel_anchor_gemm();
const void* kernel_anchor_moe();
const void* kernel_anchor_attention();
const void* kernel_anchor_misc();
const void* kernel_anchor_decode_tc();
const void* kernel_anchor_decode_ws();
const void* kernel_anchor_decode_stream();
const void* kernel_anchor_prefill_tc();
const void* kernel_anchor_peer();

namespace {
struct KernelSet {
  bool ok = false;
  std::vector<CUkernel> kernels;
  CUresult (*get_function)(CUfunction*, CUkernel) = nullptr;
  CUresult (*load)(CUfunction) = nullptr;
  CUresult (*push)(CUcontext) = nullptr;
  CUresult (*pop)(CUcontext*) = nullptr;
  CUresult (*current)(CUcontext*) = nullptr;
  CUresult (*from_green)(CUcontext*, CUgreenCtx) = nullptr;
};
const KernelSet& kernel_set() {
  static std::once_flag once;
  static KernelSet ks;
  std::call_once(once, [] {
    auto ep = [](const char* n, void** f) {
      cudaDriverEntryPointQueryResult q;
      return cudaGetDriverEntryPoint(n, f, cudaEnableDefault, &q) == cudaSuccess && *f != nullptr;
    };
    void *getlib = nullptr, *count = nullptr, *enumerate = nullptr, *gf = nullptr, *ld = nullptr, *pu = nullptr,
         *po = nullptr, *cur = nullptr, *fg = nullptr;
    if (!ep("cuKernelGetLibrary", &getlib) || !ep("cuLibraryGetKernelCount", &count) ||
        !ep("cuLibraryEnumerateKernels", &enumerate) || !ep("cuKernelGetFunction", &gf) || !ep("cuFuncLoad", &ld) ||
        !ep("cuCtxPushCurrent", &pu) || !ep("cuCtxPopCurrent", &po) || !ep("cuCtxGetCurrent", &cur) ||
        !ep("cuCtxFromGreenCtx", &fg))
      return;
    ks.get_function = (CUresult(*)(CUfunction*, CUkernel))gf;
    ks.load = (CUresult(*)(CUfunction))ld;
    ks.push = (CUresult(*)(CUcontext))pu;
    ks.pop = (CUresult(*)(CUcontext*))po;
    ks.current = (CUresult(*)(CUcontext*))cur;
    ks.from_green = (CUresult(*)(CUcontext*, CUgreenCtx))fg;
    const void* anchors[] = {kernel_anchor_gemm(),      kernel_anchor_moe(),        kernel_anchor_attention(),
                             kernel_anchor_misc(),      kernel_anchor_decode_tc(),  kernel_anchor_decode_ws(),
                             kernel_anchor_decode_stream(), kernel_anchor_prefill_tc(), kernel_anchor_peer()};
    for (const void* a : anchors) {
      cudaKernel_t k = nullptr;
      if (cudaGetKernel(&k, a) != cudaSuccess) return;
      CUlibrary lib = nullptr;
      unsigned int n = 0;
      if (((CUresult(*)(CUlibrary*, CUkernel))getlib)(&lib, (CUkernel)k) != CUDA_SUCCESS ||
          ((CUresult(*)(unsigned int*, CUlibrary))count)(&n, lib) != CUDA_SUCCESS)
        return;
      std::vector<CUkernel> ks_(n);
      if (n && ((CUresult(*)(CUkernel*, unsigned int, CUlibrary))enumerate)(ks_.data(), n, lib) != CUDA_SUCCESS) return;
      ks.kernels.insert(ks.kernels.end(), ks_.begin(), ks_.end());
    }
    ks.ok = true;
  });
  return ks;
}

cudaError_t preload_into(CUcontext ctx) {
  const KernelSet& ks = kernel_set();
  if (!ks.ok) return cudaErrorNotSupported;
  if (ks.push(ctx) != CUDA_SUCCESS) return cudaErrorUnknown;
  cudaError_t rc = cudaSuccess;
  for (CUkernel k : ks.kernels) {
    CUfunction f = nullptr;
    if (ks.get_function(&f, k) != CUDA_SUCCESS || ks.load(f) != CUDA_SUCCESS) {
      rc = cudaErrorUnknown;
      break;
    }
  }
  CUcontext old;
  ks.pop(&old);
  return rc;
}
}  // namespace

cudaError_t preload_all_kernels() {
  cudaFree(nullptr);  // make sure the runtime's (primary) context exists and is current
  const KernelSet& ks = kernel_set();
  if (!ks.ok) return cudaErrorNotSupported;
  CUcontext ctx = nullptr;
  if (ks.current(&ctx) != CUDA_SUCCESS || !ctx) return cudaErrorUnknown;
  return preload_into(ctx);
}

cudaError_t preload_kernels_green(void* green_ctx) {
  const KernelSet& ks = kernel_set();
  if (!ks.ok) return cudaErrorNotSupported;
  CUcontext ctx = nullptr;
  if (ks.from_green(&ctx, (CUgreenCtx)green_ctx) != CUDA_SUCCESS) return cudaErrorUnknown;
  return preload_into(ctx);
}

// One kernel of this translation unit (preload_all_kernels: its module is loaded eagerly).
const void* kernel_anchor_peer() { return reinterpret_cast<const void*>(peer_reduce_kernel); }

}  // namespace nf
