// Launch-gap probe: the time from one kernel's last CTA exit to the next kernel's first CTA
// entry, two dependent launches captured in a CUDA graph, as a function of the dynamic
// shared memory per CTA, the cluster size and the grid (globaltimer stamps).  Attributes
// the 4-5 us "gap after previous launch" of tools/gemm_phases.py (profiles/r2l_gemm_phases.log).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o launch_gap tools/launch_gap.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// stamps[launch*2 + 0] = min entry over CTAs, stamps[launch*2 + 1] = max exit over CTAs
__global__ void probe(unsigned long long* stamps, int launch, int spin_ns) {
  const uint64_t t0 = gtime();
  if (threadIdx.x == 0) atomicMin(&stamps[launch * 2], (unsigned long long)t0);
  while (gtime() - t0 < (uint64_t)spin_ns) {
  }
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&stamps[launch * 2 + 1], (unsigned long long)gtime());
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64 * sizeof(unsigned long long));
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  const int smems[] = {0, 48 * 1024, 100 * 1024, 200 * 1024, 227 * 1024};
  const int clusters[] = {1, 2};
  const int grids[] = {1, 148};
  printf("%8s %7s %5s %10s %10s\n", "smem_KB", "cluster", "grid", "gap_us", "dur_us");
  for (int g : grids)
    for (int cl : clusters)
      for (int smb : smems) {
        float gsum = 0.f, dsum = 0.f;
        const int reps = 20;
        cudaGraph_t graph;
        cudaGraphExec_t exec;
        cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
        for (int l = 0; l < 2; ++l) {
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3(g == 1 ? cl : g / cl * cl);
          cfg.blockDim = dim3(256);
          cfg.dynamicSmemBytes = smb;
          cfg.stream = st;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeClusterDimension;
          at[0].val.clusterDim.x = cl;
          at[0].val.clusterDim.y = 1;
          at[0].val.clusterDim.z = 1;
          cfg.attrs = at;
          cfg.numAttrs = 1;
          cudaLaunchKernelEx(&cfg, probe, (unsigned long long*)d, l, 5000);
        }
        cudaStreamEndCapture(st, &graph);
        if (cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) {
          printf("instantiate failed smem %d cluster %d\n", smb, cl);
          return 1;
        }
        for (int r = 0; r < reps + 3; ++r) {
          std::vector<unsigned long long> init(8);
          for (int i = 0; i < 4; i += 2) init[i] = ~0ull, init[i + 1] = 0;
          cudaMemcpy(d, init.data(), 4 * sizeof(unsigned long long), cudaMemcpyHostToDevice);
          cudaGraphLaunch(exec, st);
          cudaStreamSynchronize(st);
          unsigned long long h[4];
          cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
          if (r >= 3) {
            gsum += (float)(h[2] - h[1]) / 1e3f;
            dsum += (float)(h[1] - h[0]) / 1e3f;
          }
        }
        cudaError_t e = cudaGetLastError();
        printf("%8d %7d %5d %10.2f %10.2f %s\n", smb / 1024, cl, g, gsum / reps, dsum / reps,
               e == cudaSuccess ? "" : cudaGetErrorString(e));
        cudaGraphExecDestroy(exec);
        cudaGraphDestroy(graph);
      }
  return 0;
}
