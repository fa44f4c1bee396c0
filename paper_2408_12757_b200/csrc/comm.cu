// Tensor-parallel communicator: NCCL (the process's own libnccl.so.2, loaded
// with dlopen so the library links without it) over NVLink5 / NVSwitch.
// PAPER.md:628 used MSCCL++ SM-constrained kernels; here the collectives run
// on the plan's network stream with NCCL's CTA cap (ncclConfig_t.maxCTAs) set
// to the plan's network SM budget.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>

#include "host.h"

struct nf_comm {
  ncclComm_t comm = nullptr;
  int tp_size = 1, tp_rank = 0;
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

nf_status comm_all_gather(nf_comm* c, const void* send, void* recv, size_t count_bf16, cudaStream_t st) {
  ncclResult_t r = g_nccl.allGather(send, recv, count_bf16, ncclBfloat16, c->comm, st);
  if (r != ncclSuccess) return set_error(NF_ENCCL, "ncclAllGather: %s", g_nccl.getErrorString(r));
  return NF_OK;
}
nf_status comm_all_reduce_bf16(nf_comm* c, void* buf, size_t count, cudaStream_t st) {
  ncclResult_t r = g_nccl.allReduce(buf, buf, count, ncclBfloat16, ncclSum, c->comm, st);
  if (r != ncclSuccess) return set_error(NF_ENCCL, "ncclAllReduce: %s", g_nccl.getErrorString(r));
  return NF_OK;
}
nf_status comm_all_reduce_f32(nf_comm* c, void* buf, size_t count, cudaStream_t st) {
  ncclResult_t r = g_nccl.allReduce(buf, buf, count, ncclFloat32, ncclSum, c->comm, st);
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

nf_status nf_comm_create(int32_t tp_size, int32_t tp_rank, const void* id_128, nf_comm** out) {
  if (!out || !id_128) return set_error(NF_EINVAL, "NULL argument");
  if (tp_size < 1 || tp_rank < 0 || tp_rank >= tp_size) return set_error(NF_EINVAL, "bad tp_size/tp_rank");
  NF_TRY(load_nccl());
  ncclUniqueId id;
  std::memcpy(&id, id_128, 128);
  ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
  cfg.blocking = 1;
  nf_comm* c = new nf_comm();
  c->tp_size = tp_size;
  c->tp_rank = tp_rank;
  ncclResult_t r = g_nccl.commInitRankConfig(&c->comm, tp_size, id, tp_rank, &cfg);
  if (r != ncclSuccess) {
    delete c;
    return set_error(NF_ENCCL, "ncclCommInitRankConfig: %s", g_nccl.getErrorString(r));
  }
  *out = c;
  return NF_OK;
}

void nf_comm_destroy(nf_comm* c) {
  if (!c) return;
  if (c->comm && g_nccl.commDestroy) g_nccl.commDestroy(c->comm);
  delete c;
}

}  // extern "C"
