// Launch counter and optional per-op CUDA-event timing of every kernel the
// library launches (events recorded on the kernel's own stream).
#include <atomic>
#include <mutex>
#include <vector>

#include "host.h"
#include "profile.h"

namespace nf {
namespace {
std::atomic<long long> g_launches{0};
std::atomic<int> g_prof_on{0};
struct Rec {
  int op;
  cudaStream_t st;
  cudaEvent_t a, b;
  int tag;
};
thread_local int t_tag = -1;
cudaEvent_t g_base = nullptr;
std::mutex g_mu;
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;

cudaEvent_t get_event() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

void count_launch(int n) { g_launches += n; }
bool profile_active() { return g_prof_on.load() != 0; }

ProfScope::ProfScope(int op, cudaStream_t st) : op_(op), st_(st) {
  if (!g_prof_on.load()) return;
  std::lock_guard<std::mutex> lk(g_mu);
  a_ = get_event();
  b_ = get_event();
  cudaEventRecord(a_, st_);
}
ProfScope::~ProfScope() {
  if (!a_) return;
  std::lock_guard<std::mutex> lk(g_mu);
  cudaEventRecord(b_, st_);
  g_recs.push_back(Rec{op_, st_, a_, b_, t_tag});
}

}  // namespace nf

extern "C" {

int64_t nf_kernel_launches(void) { return nf::g_launches.load(); }

nf_status nf_profile_tag(int32_t tag) {
  nf::t_tag = tag;
  return NF_OK;
}

nf_status nf_profile_enable(int32_t on) {
  if (on && !nf::g_prof_on.load()) {
    std::lock_guard<std::mutex> lk(nf::g_mu);
    if (!nf::g_base) cudaEventCreate(&nf::g_base);
    cudaEventRecord(nf::g_base, 0);
  }
  nf::g_prof_on = on ? 1 : 0;
  return NF_OK;
}

nf_status nf_profile_timeline(nf_span* out, int32_t cap, int32_t* n_out) {
  if (!n_out) return nf::set_error(NF_EINVAL, "NULL n_out");
  std::lock_guard<std::mutex> lk(nf::g_mu);
  std::vector<cudaStream_t> streams;
  int n = 0;
  for (auto& r : nf::g_recs) {
    if (out && n < cap) {
      float a = 0.f, b = 0.f;
      cudaError_t e = cudaEventSynchronize(r.b);
      if (e == cudaSuccess) e = cudaEventElapsedTime(&a, nf::g_base, r.a);
      if (e == cudaSuccess) e = cudaEventElapsedTime(&b, nf::g_base, r.b);
      if (e != cudaSuccess) return nf::set_error(NF_ECUDA, "timeline event: %s", cudaGetErrorString(e));
      int si = -1;
      for (size_t i = 0; i < streams.size(); ++i)
        if (streams[i] == r.st) si = (int)i;
      if (si < 0) {
        si = (int)streams.size();
        streams.push_back(r.st);
      }
      out[n] = nf_span{r.op, si, a, b, r.tag};
    }
    ++n;
  }
  *n_out = n;
  return NF_OK;
}

nf_status nf_profile_read(double* ms_out, int64_t* count_out) {
  if (!ms_out || !count_out) return nf::set_error(NF_EINVAL, "NULL output");
  for (int i = 0; i < NF_PROF_COUNT; ++i) {
    ms_out[i] = 0;
    count_out[i] = 0;
  }
  std::lock_guard<std::mutex> lk(nf::g_mu);
  for (auto& r : nf::g_recs) {
    float ms = 0.f;
    cudaError_t e = cudaEventSynchronize(r.b);
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, r.a, r.b);
    if (e != cudaSuccess) return nf::set_error(NF_ECUDA, "profile event: %s", cudaGetErrorString(e));
    if (r.op >= 0 && r.op < NF_PROF_COUNT) {
      ms_out[r.op] += ms;
      count_out[r.op] += 1;
    }
    nf::g_pool.push_back(r.a);
    nf::g_pool.push_back(r.b);
  }
  nf::g_recs.clear();
  return NF_OK;
}

}  // extern "C"
