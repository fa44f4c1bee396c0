// Execution-unit scheduling with hard SM partitions:
// two CUDA green contexts -- a memory partition for decode attention and a
// compute partition for the dense operators -- each with a non-blocking stream.
// Kernels launched on those streams run only on their partition's SMs, so a
// kernel's CTAs can never occupy the other partition.
// Driver entry points are fetched at run time (no -lcuda link).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <algorithm>
#include <string>
#include <vector>

#include "host.h"

namespace nf {
namespace {
struct GreenApi {
  bool tried = false, ok = false;
  PFN_cuDeviceGetDevResource_v12040 getDevResource = nullptr;
  PFN_cuDevSmResourceSplitByCount_v12040 split = nullptr;
  PFN_cuDevResourceGenerateDesc_v12040 genDesc = nullptr;
  PFN_cuGreenCtxCreate_v12040 create = nullptr;
  PFN_cuGreenCtxStreamCreate_v12050 streamCreate = nullptr;
  PFN_cuGreenCtxGetDevResource_v12040 ctxResource = nullptr;
};
GreenApi g_api;

template <typename T>
bool entry(const char* name, T* fn) {
  cudaDriverEntryPointQueryResult q;
  void* p = nullptr;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return false;
  *fn = reinterpret_cast<T>(p);
  return true;
}

bool load_api() {
  if (g_api.tried) return g_api.ok;
  g_api.tried = true;
  g_api.ok = entry("cuDeviceGetDevResource", &g_api.getDevResource) && entry("cuDevSmResourceSplitByCount", &g_api.split) &&
             entry("cuDevResourceGenerateDesc", &g_api.genDesc) && entry("cuGreenCtxCreate", &g_api.create) &&
             entry("cuGreenCtxStreamCreate", &g_api.streamCreate) &&
             entry("cuGreenCtxGetDevResource", &g_api.ctxResource);
  return g_api.ok;
}
}  // namespace

// Creates (once per plan) the memory / compute partitions for an OVERLAP plan,
// plus a network partition of net_sms SMs (TP plans) when
// net_sms > 0.  Returns false (and leaves the plan on ordinary streams) when
// disabled with NF_GREEN=0 or unsupported; p->green_note says why.
bool green_setup(nf_plan* p, int dec_sms, int net_sms) {
  if (p->green_tried) return p->green_ok;
  p->green_tried = true;
  const char* env = getenv("NF_GREEN");
  if (env && env[0] == '0') {
    p->green_note = "disabled (NF_GREEN=0)";
    return false;
  }
  // Nsight Compute cannot replay kernels of green contexts ("Failed to prepare kernel for
  // profiling"): under a profiler the plan runs on ordinary streams (same kernels,
  // SM-bounded persistent grids) unless NF_GREEN=1 forces partitions.  The profiler is
  // recognised by the variables it sets in the target's environment (ncu 2025.2 sets the
  // NV_NSIGHT_INJECTION_* / NV_COMPUTE_PROFILER_* ones; older injection used CUDA_INJECTION64_PATH).
  for (const char* var : {"CUDA_INJECTION64_PATH", "NV_NSIGHT_INJECTION_TRANSPORT_TYPE", "NV_COMPUTE_PROFILER_PERFWORKS_DIR"}) {
    const char* inj = getenv(var);
    if (inj && inj[0] && !(env && env[0] == '1')) {
      p->green_note = std::string("not used under a profiler (") + var + " set)";
      return false;
    }
  }
  if (!load_api()) {
    p->green_note = "driver lacks green-context entry points";
    return false;
  }
  CUdevice dev = p->device;
  CUdevResource all{};
  if (g_api.getDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS) {
    p->green_note = "cuDeviceGetDevResource failed";
    return false;
  }
  // One split of the whole device into groups of the SM granularity (8); the memory and
  // network partitions take whole groups from the front, the compute partition the
  // remaining groups plus the leftover SMs (several SM resources combine into one
  // descriptor).  (Splitting a split's remainder a second time is rejected by the driver.)
  constexpr unsigned kQ = 8;
  CUdevResource groups[64]{}, rest{};
  unsigned int ng = 64;
  if (g_api.split(groups, &ng, &all, &rest, 0, kQ) != CUDA_SUCCESS || ng < 3) {
    p->green_note = "cuDevSmResourceSplitByCount failed";
    return false;
  }
  // dec_sms >= all SMs: no memory partition (decode attention runs on the compute streams;
  // a TP plan that overlaps only the collectives)
  const unsigned n_mem = dec_sms >= (int)all.sm.smCount ? 0u : std::max(1u, (unsigned)((dec_sms + kQ - 1) / kQ));
  const unsigned n_net = net_sms > 0 ? std::max(1u, (unsigned)((net_sms + kQ - 1) / kQ)) : 0u;
  if (n_mem == 0 && n_net == 0) {
    p->green_note = "no partition requested";
    return false;
  }
  if (n_mem + n_net + 1 > ng) {
    p->green_note = "memory + network partitions leave no compute SMs";
    return false;
  }
  std::vector<CUdevResource> cmp(groups + n_mem + n_net, groups + ng);
  if (rest.sm.smCount > 0) cmp.push_back(rest);
  CUdevResourceDesc d_mem, d_cmp, d_net;
  CUgreenCtx g_mem = nullptr, g_cmp, g_net = nullptr;
  if ((n_mem > 0 && (g_api.genDesc(&d_mem, groups, n_mem) != CUDA_SUCCESS ||
                     g_api.create(&g_mem, d_mem, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS)) ||
      g_api.genDesc(&d_cmp, cmp.data(), (unsigned)cmp.size()) != CUDA_SUCCESS ||
      g_api.create(&g_cmp, d_cmp, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS) {
    p->green_note = "green context creation failed";
    return false;
  }
  if (n_net > 0 && (g_api.genDesc(&d_net, groups + n_mem, n_net) != CUDA_SUCCESS ||
                    g_api.create(&g_net, d_net, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS)) {
    p->green_note = "green context creation failed (network partition)";
    return false;
  }
  // every kernel of the library loaded into the new contexts now (no lazy load later, while a
  // spin-waiting kernel may run: see preload_kernels_green)
  for (CUgreenCtx g : {g_mem, g_cmp, g_net})
    if (g && preload_kernels_green((void*)g) != cudaSuccess) {
      p->green_note = "kernel preload into a green context failed";
      return false;
    }
  unsigned sm_mem = 0, sm_net = 0, sm_cmp = 0;
  for (unsigned i = 0; i < n_mem; ++i) sm_mem += groups[i].sm.smCount;
  for (unsigned i = 0; i < n_net; ++i) sm_net += groups[n_mem + i].sm.smCount;
  for (const auto& r : cmp) sm_cmp += r.sm.smCount;
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  CUstream s_mem = nullptr, s_cmp, s_cmp2, s_net = nullptr;
  if ((g_mem && g_api.streamCreate(&s_mem, g_mem, CU_STREAM_NON_BLOCKING, hi) != CUDA_SUCCESS) ||
      g_api.streamCreate(&s_cmp, g_cmp, CU_STREAM_NON_BLOCKING, lo) != CUDA_SUCCESS ||
      g_api.streamCreate(&s_cmp2, g_cmp, CU_STREAM_NON_BLOCKING, lo) != CUDA_SUCCESS ||
      (g_net && g_api.streamCreate(&s_net, g_net, CU_STREAM_NON_BLOCKING, hi) != CUDA_SUCCESS)) {
    p->green_note = "green stream creation failed";
    return false;
  }
  // without a memory partition: two high-priority side streams in the compute partition for decode
  // attention (one per dense group), so a group's decode runs beside its prefill (NF_TP_DEC_SIDE=1)
  CUstream s_d1 = nullptr, s_d2 = nullptr;
  if (!g_mem && (g_api.streamCreate(&s_d1, g_cmp, CU_STREAM_NON_BLOCKING, hi) != CUDA_SUCCESS ||
                 g_api.streamCreate(&s_d2, g_cmp, CU_STREAM_NON_BLOCKING, hi) != CUDA_SUCCESS)) {
    p->green_note = "green stream creation failed";
    return false;
  }
  p->green_ds1 = (cudaStream_t)s_d1;
  p->green_ds2 = (cudaStream_t)s_d2;
  p->green_ms = (cudaStream_t)s_mem;
  p->green_cs = (cudaStream_t)s_cmp;
  p->green_cs2 = (cudaStream_t)s_cmp2;
  p->green_ns = (cudaStream_t)s_net;
  p->green_dec_sms = (int)sm_mem;
  p->green_dense_sms = (int)sm_cmp;
  p->green_net_sms = (int)sm_net;
  p->green_ok = true;
  p->green_note = (g_mem ? "memory partition " + std::to_string(p->green_dec_sms) + " SMs, "
                          : std::string("no memory partition (decode on the compute streams), ")) +
                  "compute partition " + std::to_string(p->green_dense_sms) + " SMs";
  if (g_net) p->green_note += ", network partition " + std::to_string(p->green_net_sms) + " SMs";
  return true;
}

}  // namespace nf
