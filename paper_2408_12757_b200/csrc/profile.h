#pragma once
#include <cuda_runtime.h>

namespace nf {
void count_launch(int n = 1);
bool profile_active();
// RAII: when profiling is enabled, records CUDA events around the enclosed launches on `st`.
class ProfScope {
 public:
  ProfScope(int op, cudaStream_t st);
  ~ProfScope();

 private:
  int op_;
  cudaStream_t st_;
  cudaEvent_t a_ = nullptr, b_ = nullptr;
};
}  // namespace nf
