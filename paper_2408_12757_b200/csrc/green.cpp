// Execution-unit scheduling with hard SM partitions:
// two CUDA green contexts -- a memory partition for decode attention and a
// compute partition for the dense operators -- each with a non-blocking stream.
// Kernels launched on those streams run only on their partition's SMs, so a
// kernel's CTAs can never occupy the other partition.
// Driver entry points are fetched at run time (no -lcuda link).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <string>

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

// Creates (once per plan) the memory / compute partitions for an OVERLAP plan.
// Returns false (and leaves the plan on ordinary streams) when disabled with
// NF_GREEN=0 or unsupported; p->green_note says why.
bool green_setup(nf_plan* p, int dec_sms) {
  if (p->green_tried) return p->green_ok;
  p->green_tried = true;
  const char* env = getenv("NF_GREEN");
  if (env && env[0] == '0') {
    p->green_note = "disabled (NF_GREEN=0)";
    return false;
  }
  if (!load_api()) {
    p->green_note = "driver lacks green-context entry points";
    return false;
  }
  CUdevice dev = p->device;
  CUdevResource all{}, part[1]{}, rest{};
  if (g_api.getDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS) {
    p->green_note = "cuDeviceGetDevResource failed";
    return false;
  }
  unsigned int n = 1;
  const unsigned int want = (unsigned int)((dec_sms + 7) / 8 * 8);
  if (g_api.split(part, &n, &all, &rest, 0, want) != CUDA_SUCCESS || n != 1) {
    p->green_note = "cuDevSmResourceSplitByCount failed";
    return false;
  }
  CUdevResourceDesc d_mem, d_cmp;
  CUgreenCtx g_mem, g_cmp;
  if (g_api.genDesc(&d_mem, part, 1) != CUDA_SUCCESS || g_api.genDesc(&d_cmp, &rest, 1) != CUDA_SUCCESS ||
      g_api.create(&g_mem, d_mem, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS ||
      g_api.create(&g_cmp, d_cmp, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS) {
    p->green_note = "green context creation failed";
    return false;
  }
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  CUstream s_mem, s_cmp;
  if (g_api.streamCreate(&s_mem, g_mem, CU_STREAM_NON_BLOCKING, hi) != CUDA_SUCCESS ||
      g_api.streamCreate(&s_cmp, g_cmp, CU_STREAM_NON_BLOCKING, lo) != CUDA_SUCCESS) {
    p->green_note = "green stream creation failed";
    return false;
  }
  p->green_ms = (cudaStream_t)s_mem;
  p->green_cs = (cudaStream_t)s_cmp;
  p->green_dec_sms = (int)part[0].sm.smCount;
  p->green_dense_sms = (int)rest.sm.smCount;
  p->green_ok = true;
  p->green_note = "memory partition " + std::to_string(p->green_dec_sms) + " SMs, compute partition " +
                  std::to_string(p->green_dense_sms) + " SMs";
  return true;
}

}  // namespace nf
