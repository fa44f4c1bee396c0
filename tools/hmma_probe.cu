// Throughput of the legacy tensor path (mma.sync.m16n8k16 bf16 -> f32, "HMMA") and of
// FFMA on one B200 SM, to size the decode-attention kernel's per-page instruction budget.
// Build/run: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/hmma_probe.cu -o /tmp/hp && /tmp/hp
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void hmma_kernel(float* out, int iters) {
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  float d[8][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0.f;
  for (int c = 0; c < 8; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void ffma_kernel(float* out, int iters) {
  float x[16];
  for (int c = 0; c < 16; ++c) x[c] = threadIdx.x * 0.001f + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 16; ++c) x[c] = fmaf(x[c], 0.999f, 0.5f);
  }
  float s = 0.f;
  for (int c = 0; c < 16; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 1024 * 4);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps : {4, 8, 16}) {
    const int iters = 4096;
    hmma_kernel<<<148, warps * 32>>>(out, 16);
    cudaEventRecord(e0);
    hmma_kernel<<<148, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double mmas = 148.0 * warps * iters * 8;
    printf("HMMA m16n8k16 bf16: %2d warps/SM: %.1f TFLOP/s, %.2f ns per MMA per SM-subpartition\n", warps,
           mmas * 4096 / (ms * 1e-3) / 1e12, (ms * 1e6) / (mmas / 148.0 / 4.0));
  }
  for (int warps : {8, 16}) {
    const int iters = 4096;
    ffma_kernel<<<148, warps * 32>>>(out, 16);
    cudaEventRecord(e0);
    ffma_kernel<<<148, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double f = 148.0 * warps * 32 * iters * 16;
    printf("FFMA: %2d warps/SM: %.1f TFLOP/s (fp32, 2 flop/FMA)\n", warps, 2 * f / (ms * 1e-3) / 1e12);
  }
  printf("nominal SM clock attribute: %d kHz\n", clk);
  return 0;
}
