// Tensor-parallel communicator: NCCL (the process's own libnccl.so.2, loaded
// with dlopen so the library links without it) over NVLink5 / NVSwitch.
// PAPER.md:628 used MSCCL++ SM-constrained kernels (the network
// operation gets its own SM budget).  Here the collectives run on the plan's network
// stream; with nf_comm_create(max_ctas > 0) NCCL's CTA cap (ncclConfig_t.maxCTAs) is
// set, and an OVERLAP plan places that stream in its own green-context SM partition
// of plan sm[NF_OP_NET] SMs when the cap fits in it (api.cu enter_partitions), so the
// collective kernels never run on the compute or memory partitions.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "host.h"
#include "misc.cuh"
#include "peer.cuh"
#include "profile.h"

namespace nf {
// Single-process, single-GPU emulation of a TP group (tests / rank-local
// studies): N ranks are N host threads sharing one device; collectives meet at
// a host barrier and exchange device buffers with stream-ordered copies.
// AllReduce sums the N inputs in rank order with fp32 accumulation, so every
// rank gets bit-identical results.
struct LocalGroup {
  int n;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  std::vector<const void*> src;
  std::vector<cudaStream_t> st;
  std::vector<cudaEvent_t> ev_ready, ev_done;
  std::vector<uint8_t*> sym;  // every rank's symmetric buffer (fused collectives)
  explicit LocalGroup(int n_) : n(n_), src(n_), st(n_), ev_ready(n_), ev_done(n_), sym(n_, nullptr) {
    for (int i = 0; i < n; ++i) {
      cudaEventCreateWithFlags(&ev_ready[i], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&ev_done[i], cudaEventDisableTiming);
    }
  }
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long long g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};
}  // namespace nf

struct nf_comm {
  ncclComm_t comm = nullptr;
  int tp_size = 1, tp_rank = 0;
  int max_ctas = 0;                        // NCCL CTA cap (0 = NCCL default)
  int ar_mode = NF_AR_F32;                 // emulated AllReduce arithmetic
  bool loopback = false;                   // nf_comm_create_loopback: one rank, local copies
  double link_gbs = 0.0;                   // loopback link-time model (nf_comm_loopback_set_link), 0 = off
  std::shared_ptr<nf::LocalGroup> group;  // emulated group (nf_comm_create_local)
  // fused collectives (peer.cuh): this rank's symmetric buffer, every rank's mapping of theirs
  uint8_t* sym = nullptr;
  size_t sym_bytes = 0;
  std::vector<uint8_t*> sym_peer;          // [tp_size] (own entry = sym); IPC-opened for NCCL groups
  uint8_t** sym_peer_dev = nullptr;        // device copy of sym_peer
  nf::PeerGeom* geom = nullptr;
  bool fused = false;
  long long fused_sites = 0;  // fused sites issued (host count)
  long long timeout_ns = 20000000000LL;
};

namespace nf {
namespace {
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRankConfig)(ncclComm_t*, int, ncclUniqueId, int, ncclConfig_t*) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
};
NcclApi g_nccl;

nf_status load_nccl() {
  if (g_nccl.h) return NF_OK;
  const char* env = getenv("NF_NCCL_LIB");
  void* h = dlopen(env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return set_error(NF_ENCCL, "dlopen libnccl.so.2 failed: %s (set NF_NCCL_LIB)", dlerror());
  g_nccl.getUniqueId = (decltype(g_nccl.getUniqueId))dlsym(h, "ncclGetUniqueId");
  g_nccl.commInitRankConfig = (decltype(g_nccl.commInitRankConfig))dlsym(h, "ncclCommInitRankConfig");
  g_nccl.commDestroy = (decltype(g_nccl.commDestroy))dlsym(h, "ncclCommDestroy");
  g_nccl.allGather = (decltype(g_nccl.allGather))dlsym(h, "ncclAllGather");
  g_nccl.allReduce = (decltype(g_nccl.allReduce))dlsym(h, "ncclAllReduce");
  g_nccl.getErrorString = (decltype(g_nccl.getErrorString))dlsym(h, "ncclGetErrorString");
  if (!g_nccl.getUniqueId || !g_nccl.commInitRankConfig || !g_nccl.commDestroy || !g_nccl.allGather ||
      !g_nccl.allReduce || !g_nccl.getErrorString)
    return set_error(NF_ENCCL, "libnccl.so.2 lacks a required symbol");
  g_nccl.h = h;
  return NF_OK;
}
}  // namespace

int comm_size(const nf_comm* c) { return c ? c->tp_size : 1; }
int comm_rank(const nf_comm* c) { return c ? c->tp_rank : 0; }
bool comm_emulated(const nf_comm* c) { return c && (c->group || c->loopback); }
bool comm_host_sync(const nf_comm* c) { return c && c->group; }
int comm_max_ctas(const nf_comm* c) { return c ? c->max_ctas : 0; }
bool comm_fused(const nf_comm* c) { return c && c->fused && c->sym_peer_dev && c->geom; }
// Emulated group with the fused path: the rank threads meet before a step launches any
// spin-waiting kernel, so that no rank is still in a host call that may wait for the device
// to be idle (first pinned-staging allocation, allocator calls) while another rank's reduce
// kernel spins on it.
void comm_count_fused(nf_comm* c) { ++c->fused_sites; }
// Emulated group: every rank has enqueued its producer GEMM of a site before any rank enqueues
// that site's spin-waiting reduce.  (The ranks' streams share the GPU's hardware work queues;
// a reduce queued ahead of another rank's producer in the same queue would wait for it
// forever.  With one rank per GPU each rank enqueues its own GEMM before its reduce, which is
// all that is needed.)
void comm_fused_site_barrier(nf_comm* c) {
  if (c && c->group && comm_fused(c)) c->group->barrier();
}
void comm_fused_step_barrier(nf_comm* c) {
  if (c && c->group && comm_fused(c)) c->group->barrier();
}
const PeerGeom& comm_peer_geom(const nf_comm* c) { return *c->geom; }
uint8_t* const* comm_peer_bases(const nf_comm* c) { return c->sym_peer_dev; }
uint8_t* comm_sym_local(const nf_comm* c) { return c->sym; }
long long comm_peer_timeout_ns(const nf_comm* c) { return c->timeout_ns; }

namespace {
// Loopback link-time model: copy src into `reps` slots of dst (the collective's local HBM
// traffic), then hold until t_ns after the kernel started -- a ring collective over a link of
// the modeled bandwidth ends no earlier (nf_comm_loopback_set_link).
__global__ void paced_copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n16, int reps,
                                  size_t stride16, unsigned long long t_ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int q = 0; q < reps; ++q)
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
      dst[q * stride16 + i] = src[i];
  if (threadIdx.x == 0) {
    do {
      __nanosleep(256);
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    } while (t - t0 < t_ns);
  }
}
}  // namespace

// loopback collective: `reps` copies of `bytes` from src to dst (slot stride `bytes`), lasting at
// least link_bytes / link_gbs when the link model is on
nf_status loopback_copy(nf_comm* c, const void* src, void* dst, size_t bytes, int reps, double link_bytes,
                        cudaStream_t st) {
  const bool paced = c->link_gbs > 0.0;
  const bool vec = bytes % 16 == 0 && ((uintptr_t)src | (uintptr_t)dst) % 16 == 0;
  if (!paced || !vec)
    for (int q = 0; q < reps; ++q)
      if (cudaMemcpyAsync((char*)dst + q * bytes, src, bytes, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return set_error(NF_ECUDA, "loopback copy");
  if (paced) {  // (unaligned buffers: the copies above, then the hold alone)
    const unsigned long long t_ns = (unsigned long long)(link_bytes / c->link_gbs);  // bytes / (GB/s) = ns
    paced_copy_kernel<<<32, 256, 0, st>>>((const uint4*)src, (uint4*)dst, vec ? bytes / 16 : 0, reps, bytes / 16, t_ns);
    count_launch();
    if (cudaGetLastError() != cudaSuccess) return set_error(NF_ECUDA, "loopback paced copy");
  }
  return NF_OK;
}

// recv = [rank 0's send | rank 1's send | ...] (count bf16 elements each)
nf_status comm_all_gather(nf_comm* c, const void* send, void* recv, size_t count_bf16, cudaStream_t st) {
  if (c->loopback)  // this rank's buffer into every slot: the AllGather's bytes, no peers (a ring
                    // AllGather receives N-1 slots per GPU)
    return loopback_copy(c, send, recv, count_bf16 * 2, c->tp_size, (double)(c->tp_size - 1) * count_bf16 * 2, st);
  if (c->group) {
    LocalGroup& g = *c->group;
    const int r = c->tp_rank;
    const size_t bytes = count_bf16 * 2;
    g.src[r] = send;
    g.st[r] = st;
    if (cudaEventRecord(g.ev_ready[r], st) != cudaSuccess) return set_error(NF_ECUDA, "emulated AG record");
    g.barrier();
    for (int q = 0; q < g.n; ++q) {
      cudaStreamWaitEvent(st, g.ev_ready[q], 0);
      if (cudaMemcpyAsync((char*)recv + q * bytes, g.src[q], bytes, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return set_error(NF_ECUDA, "emulated AG copy");
    }
    cudaEventRecord(g.ev_done[r], st);
    g.barrier();
    for (int q = 0; q < g.n; ++q) cudaStreamWaitEvent(st, g.ev_done[q], 0);  // senders reusable after all copies
    g.barrier();
    return NF_OK;
  }
  ncclResult_t r = g_nccl.allGather(send, recv, count_bf16, ncclBfloat16, c->comm, st);
  if (r != ncclSuccess) return set_error(NF_ENCCL, "ncclAllGather: %s", g_nccl.getErrorString(r));
  return NF_OK;
}

// in-place sum over ranks; scratch: count bf16 elements of device memory (emulation only)
nf_status comm_all_reduce_bf16(nf_comm* c, void* buf, size_t count, cudaStream_t st, void* scratch) {
  if (c->loopback)  // a read + write of the buffer (the reduction's local traffic), values unchanged
                    // (a ring AllReduce sends 2 (N-1) / N of the buffer per GPU)
    return loopback_copy(c, buf, scratch, count * 2, 1, 2.0 * (c->tp_size - 1) / c->tp_size * count * 2, st);
  if (c->group) {
    LocalGroup& g = *c->group;
    const int r = c->tp_rank;
    g.src[r] = buf;
    g.st[r] = st;
    if (cudaEventRecord(g.ev_ready[r], st) != cudaSuccess) return set_error(NF_ECUDA, "emulated AR record");
    g.barrier();
    for (int q = 0; q < g.n; ++q) cudaStreamWaitEvent(st, g.ev_ready[q], 0);
    std::vector<const void*> srcs(g.src.begin(), g.src.end());
    if (launch_sum_bf16(srcs.data(), g.n, (__nv_bfloat16*)scratch, count, c->ar_mode == NF_AR_RING, st) != cudaSuccess)
      return set_error(NF_ECUDA, "emulated AR sum");
    cudaEventRecord(g.ev_done[r], st);
    g.barrier();
    for (int q = 0; q < g.n; ++q) cudaStreamWaitEvent(st, g.ev_done[q], 0);  // everyone has read every input
    if (cudaMemcpyAsync(buf, scratch, count * 2, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return set_error(NF_ECUDA, "emulated AR copy");
    g.barrier();
    return NF_OK;
  }
  ncclResult_t r = g_nccl.allReduce(buf, buf, count, ncclBfloat16, ncclSum, c->comm, st);
  if (r != ncclSuccess) return set_error(NF_ENCCL, "ncclAllReduce: %s", g_nccl.getErrorString(r));
  return NF_OK;
}

}  // namespace nf

using namespace nf;

extern "C" {

nf_status nf_comm_unique_id(void* id_out_128) {
  if (!id_out_128) return set_error(NF_EINVAL, "id_out is NULL");
  NF_TRY(load_nccl());
  ncclUniqueId id;
  ncclResult_t r = g_nccl.getUniqueId(&id);
  if (r != ncclSuccess) return set_error(NF_ENCCL, "ncclGetUniqueId: %s", g_nccl.getErrorString(r));
  static_assert(sizeof(ncclUniqueId) == 128, "unique id size");
  std::memcpy(id_out_128, &id, 128);
  return NF_OK;
}

nf_status nf_comm_create(int32_t tp_size, int32_t tp_rank, const void* id_128, int32_t max_ctas, nf_comm** out) {
  if (!out || !id_128) return set_error(NF_EINVAL, "NULL argument");
  if (tp_size < 1 || tp_rank < 0 || tp_rank >= tp_size) return set_error(NF_EINVAL, "bad tp_size/tp_rank");
  if (max_ctas < 0 || max_ctas > 64) return set_error(NF_EINVAL, "max_ctas %d not in [0, 64]", max_ctas);
  NF_TRY(load_nccl());
  ncclUniqueId id;
  std::memcpy(&id, id_128, 128);
  ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
  cfg.blocking = 1;
  if (max_ctas > 0) {
    cfg.minCTAs = 1;
    cfg.maxCTAs = max_ctas;
  }
  nf_comm* c = new nf_comm();
  c->tp_size = tp_size;
  c->tp_rank = tp_rank;
  c->max_ctas = max_ctas;
  ncclResult_t r = g_nccl.commInitRankConfig(&c->comm, tp_size, id, tp_rank, &cfg);
  if (r != ncclSuccess) {
    delete c;
    return set_error(NF_ENCCL, "ncclCommInitRankConfig: %s", g_nccl.getErrorString(r));
  }
  *out = c;
  return NF_OK;
}

nf_status nf_comm_create_local(int32_t tp_size, int32_t ar_mode, nf_comm** comms_out) {
  if (!comms_out || tp_size < 1 || tp_size > 8) return set_error(NF_EINVAL, "bad tp_size (1..8) / output");
  if (ar_mode != NF_AR_F32 && ar_mode != NF_AR_RING) return set_error(NF_EINVAL, "bad ar_mode %d", ar_mode);
  auto g = std::make_shared<LocalGroup>(tp_size);
  for (int r = 0; r < tp_size; ++r) {
    nf_comm* c = new nf_comm();
    c->tp_size = tp_size;
    c->tp_rank = r;
    c->ar_mode = ar_mode;
    c->group = g;
    comms_out[r] = c;
  }
  return NF_OK;
}

nf_status nf_comm_create_loopback(int32_t tp_size, int32_t tp_rank, nf_comm** out) {
  if (!out || tp_size < 1 || tp_size > 64 || tp_rank < 0 || tp_rank >= tp_size)
    return set_error(NF_EINVAL, "bad tp_size/tp_rank/output");
  nf_comm* c = new nf_comm();
  c->tp_size = tp_size;
  c->tp_rank = tp_rank;
  c->loopback = true;
  *out = c;
  return NF_OK;
}

nf_status nf_comm_loopback_set_link(nf_comm* comm, double link_gbs) {
  if (!comm || !comm->loopback) return set_error(NF_EINVAL, "not a loopback communicator");
  if (!(link_gbs >= 0.0) || link_gbs > 1e6) return set_error(NF_EINVAL, "link_gbs %g out of range", link_gbs);
  comm->link_gbs = link_gbs;
  return NF_OK;
}

nf_status nf_comm_sym_bytes(const nf_model_cfg* cfg, int32_t max_tokens, size_t* bytes) {
  if (!cfg || !bytes || max_tokens < 1) return set_error(NF_EINVAL, "NULL argument / max_tokens < 1");
  if (cfg->d_model % PEER_BN) return set_error(NF_EINVAL, "d_model %d not a multiple of %d", cfg->d_model, PEER_BN);
  const int n = std::max(1, (int)cfg->tp_size);
  *bytes = (size_t)peer_geom(n, 0, max_tokens, cfg->d_model).total_bytes;
  return NF_OK;
}

nf_status nf_comm_sym_alloc(nf_comm* c, const nf_model_cfg* cfg, int32_t max_tokens, void* ipc_handle_out_64) {
  if (!c || !cfg) return set_error(NF_EINVAL, "NULL argument");
  if (c->sym) return set_error(NF_EINVAL, "symmetric buffer already allocated");
  if (cfg->tp_size != c->tp_size) return set_error(NF_EINVAL, "cfg tp_size %d != communicator %d", cfg->tp_size, c->tp_size);
  size_t bytes = 0;
  NF_TRY(nf_comm_sym_bytes(cfg, max_tokens, &bytes));
  // a loopback rank has no peers: its fused sites run as a group of one (local staging and result)
  const int n = c->loopback ? 1 : c->tp_size, rank = c->loopback ? 0 : c->tp_rank;
  if (cudaMalloc(&c->sym, bytes) != cudaSuccess) {
    c->sym = nullptr;
    return set_error(NF_ECUDA, "cudaMalloc of %zu symmetric bytes failed", bytes);
  }
  // zeroed and complete before any rank's kernels run (they are on non-blocking streams, which
  // do not order after this legacy-stream memset)
  if (cudaMemset(c->sym, 0, bytes) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess)
    return set_error(NF_ECUDA, "cudaMemset symmetric buffer");
  c->sym_bytes = bytes;
  c->geom = new PeerGeom(peer_geom(n, rank, max_tokens, cfg->d_model));
  if (ipc_handle_out_64) {
    std::memset(ipc_handle_out_64, 0, 64);
    if (!c->group && !c->loopback) {
      cudaIpcMemHandle_t h;
      if (cudaIpcGetMemHandle(&h, c->sym) != cudaSuccess) return set_error(NF_ECUDA, "cudaIpcGetMemHandle failed");
      static_assert(sizeof(cudaIpcMemHandle_t) == 64, "ipc handle size");
      std::memcpy(ipc_handle_out_64, &h, 64);
    }
  }
  if (c->group) {
    std::lock_guard<std::mutex> lk(c->group->mu);
    c->group->sym[c->tp_rank] = c->sym;
  }
  return NF_OK;
}

nf_status nf_comm_sym_open(nf_comm* c, const void* ipc_handles) {
  if (!c || !c->sym) return set_error(NF_EINVAL, "communicator without a symmetric buffer (nf_comm_sym_alloc first)");
  const int n = c->geom->n;
  c->sym_peer.assign(n, nullptr);
  if (c->loopback) {
    c->sym_peer[0] = c->sym;
  } else if (c->group) {
    std::lock_guard<std::mutex> lk(c->group->mu);
    for (int r = 0; r < n; ++r) {
      if (!c->group->sym[r]) return set_error(NF_EINVAL, "rank %d of the emulated group has no symmetric buffer", r);
      c->sym_peer[r] = c->group->sym[r];
    }
  } else {
    if (!ipc_handles) return set_error(NF_EINVAL, "ipc_handles is NULL");
    for (int r = 0; r < n; ++r) {
      if (r == c->tp_rank) {
        c->sym_peer[r] = c->sym;
        continue;
      }
      cudaIpcMemHandle_t h;
      std::memcpy(&h, (const char*)ipc_handles + 64 * r, 64);
      void* p = nullptr;
      if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
        return set_error(NF_ECUDA, "cudaIpcOpenMemHandle of rank %d: %s", r, cudaGetErrorString(cudaGetLastError()));
      c->sym_peer[r] = (uint8_t*)p;
    }
  }
  if (!c->sym_peer_dev && cudaMalloc(&c->sym_peer_dev, sizeof(uint8_t*) * n) != cudaSuccess)
    return set_error(NF_ECUDA, "cudaMalloc peer table");
  if (cudaMemcpy(c->sym_peer_dev, c->sym_peer.data(), sizeof(uint8_t*) * n, cudaMemcpyHostToDevice) != cudaSuccess)
    return set_error(NF_ECUDA, "peer table upload");
  if (preload_all_kernels() != cudaSuccess) return set_error(NF_ECUDA, "preloading the library's kernels failed");
  const char* e = getenv("NF_PEER_TIMEOUT_MS");
  if (e) c->timeout_ns = std::max(1LL, atoll(e)) * 1000000LL;
  c->fused = true;
  return NF_OK;
}

nf_status nf_comm_set_fused(nf_comm* c, int32_t on) {
  if (!c) return set_error(NF_EINVAL, "NULL communicator");
  if (on && !c->sym_peer_dev) return set_error(NF_EINVAL, "symmetric buffers not open (nf_comm_sym_open)");
  c->fused = on != 0;
  return NF_OK;
}

nf_status nf_comm_sym_status(nf_comm* c, int32_t* timeouts_out, int64_t* fused_sites_out) {
  if (!c || !timeouts_out) return set_error(NF_EINVAL, "NULL argument");
  *timeouts_out = 0;
  if (fused_sites_out) *fused_sites_out = c->fused_sites;
  if (!c->sym) return NF_OK;
  uint32_t v[16 + 8 * 16] = {};
  if (cudaMemcpy(v, c->sym, sizeof(v), cudaMemcpyDeviceToHost) != cudaSuccess) return set_error(NF_ECUDA, "status read");
  *timeouts_out = (int32_t)v[0];
  if (getenv("NF_PEER_DEBUG")) {
    fprintf(stderr, "[nf peer] rank %d: timeouts %u, longest flag wait %u us, longest done wait %u us\n", c->tp_rank,
            v[0], v[8], v[9]);
  }
  if (v[0]) {  // the first timeout's record, for the caller's error report (nf_last_error)
    set_error(NF_OK, "peer wait timeout: site %u %s block %u src %u observed %u target %u (%u timeouts)", v[16],
              v[17] == 2 ? "all-gather done" : v[17] ? "done" : "flag", v[18] / 16, v[18] % 16, v[19], v[20], v[0]);
  }
  return NF_OK;
}

void nf_comm_destroy(nf_comm* c) {
  if (!c) return;
  if (!c->group && !c->loopback)
    for (int r = 0; r < (int)c->sym_peer.size(); ++r)
      if (r != c->tp_rank && c->sym_peer[r]) cudaIpcCloseMemHandle(c->sym_peer[r]);
  if (c->group && c->sym) {
    std::lock_guard<std::mutex> lk(c->group->mu);
    c->group->sym[c->tp_rank] = nullptr;
  }
  if (c->sym_peer_dev) cudaFree(c->sym_peer_dev);
  if (c->sym) cudaFree(c->sym);
  delete c->geom;
  if (!c->group && !c->loopback && c->comm && g_nccl.commDestroy) g_nccl.commDestroy(c->comm);
  delete c;
}

}  // extern "C"
