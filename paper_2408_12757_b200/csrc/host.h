// Host-side internals shared by the ABI translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/nf.h"
#include "attention.cuh"

namespace nf {

nf_status set_error(nf_status s, const char* fmt, ...);
inline nf_status ok() { return NF_OK; }

#define NF_CUDA(call)                                                                                  \
  do {                                                                                                 \
    cudaError_t _e = (call);                                                                           \
    if (_e != cudaSuccess) return set_error(NF_ECUDA, "%s failed: %s", #call, cudaGetErrorString(_e)); \
  } while (0)
#define NF_TRY(call)                   \
  do {                                 \
    nf_status _s = (call);             \
    if (_s != NF_OK) return _s;        \
  } while (0)

nf_status validate_cfg(const nf_model_cfg* c);
nf_status validate_batch(const nf_model_cfg* c, const nf_batch* b);
int64_t batch_tokens(const nf_batch* b);

struct NanoRange {
  int r0, r1;        // requests [r0, r1) in the internal (permuted) order
  int t0, t1;        // token rows
  int dec_off, dec_n;  // decode items
  int dec_cs_n = 0;    // OVERLAP: this many of the shortest decode items run on the compute partition
  int dec_rows_off = 0;  // offset of this nano-batch's decode row streams in the workspace (ROWS loader)
  int pf_off, pf_n;    // prefill items
};

// Per-step metadata in the internal token order (request permutation `order`).
struct StepMeta {
  std::vector<int32_t> buf;   // int32 words uploaded to the workspace
  size_t off_pos = 0, off_slot = 0, off_pages = 0, off_dec = 0, off_pf = 0, off_emit_row = 0, off_emit_req = 0,
         off_tok_src = 0, off_emit_sorted = 0;  // emit rows in ascending caller-request order (logits output)
  int T = 0, n_req = 0, n_emit = 0;
  std::vector<NanoRange> nanos;
};

// Upper bound of StepMeta words for a batch (workspace sizing).
size_t meta_words_bound(const nf_model_cfg* c, const nf_batch* b);
// order: internal request order (size n_req); req_cuts: nano-batch boundaries in that order.
void build_meta(const nf_model_cfg* c, const nf_batch* b, const std::vector<int>& order, const std::vector<int>& req_cuts,
                StepMeta* m, const std::vector<int32_t>* caller_row0 = nullptr,
                const std::vector<int32_t>* caller_req = nullptr);
void balance_requests(const nf_batch* b, int nn, const int32_t* share, std::vector<std::vector<int>>* groups);
std::vector<int> snap_cuts_impl(const std::vector<int64_t>& row_start_of_boundary, int n_nano, const int32_t* share);

struct Workspace {
  int32_t* meta;
  __nv_bfloat16 *q, *o, *o_full, *h1, *m, *xa, *xb, *lm_rows;
  float *part_a, *part_b, *part_h1, *lm_part, *am_val;
  int* am_idx;
  float* red;  // TP partial sums (f32)
  __nv_bfloat16 *ag, *ag2, *ocat, *hcol;  // TP: gathered (rank-major) attention output / O-col output staging,
                                          // interleaved O input, O-col output
  float* am_pair;      // TP: per-row (max, global argmax) of this rank's vocab shard [n_req] (float, int)
  float* am_pair_all;  // TP: AllGather of am_pair [tp][n_req]
  float* sk_part;  // stream-K partial tiles [148][128][256] f32
  int* sk_flag;    // stream-K tile counters
  int sk_flag_n;
  float* sk_part2;  // TP: a second stream-K set for the second dense nano-batch's compute stream
  int* sk_flag2;
  int sk_flag_total;  // flags to zero per step (both sets)
  int sk_slots;
  // MoE FFN (n_experts > 0): routing, grouping and the grouped GEMM operands (moe.cu)
  int* mo_ids;
  float* mo_wts;
  float* mo_inv;
  int* mo_grp;       // [E+1] segment offsets, then [E] segment ends
  int* mo_dst;
  int* mo_rowtok;
  float *mo_roww, *mo_rowinv;
  __nv_bfloat16 *mo_x, *mo_m, *mo_y;
  int* mo_cta;       // per-router-CTA expert counts, then bases (moe.cuh MoeGroupArgs)
  int* dec_rows;     // decode row streams of every nano-batch (sum of decode pages x kv heads)
  int* dec_wstart;   // [NF_MAX_NANO][2049] per-warp stream offsets
  int64_t mo_cap;    // grouped rows capacity
  size_t total;
};
Workspace carve_workspace(const nf_model_cfg* c, const nf_batch* b, void* base);

}  // namespace nf

namespace nf {
bool green_setup(nf_plan* p, int dec_sms, int net_sms);
int comm_size(const nf_comm* c);
int comm_rank(const nf_comm* c);
bool comm_emulated(const nf_comm* c);   // emulated group or loopback (no NCCL kernels)
bool comm_host_sync(const nf_comm* c);  // collectives meet at host barriers (not capturable)
int comm_max_ctas(const nf_comm* c);
nf_status comm_all_gather(nf_comm* c, const void* send, void* recv, size_t count_bf16, cudaStream_t st);
nf_status comm_all_reduce_bf16(nf_comm* c, void* buf, size_t count, cudaStream_t st, void* scratch);
// Fused GEMM -> AllReduce over peer memory (peer.cuh; NEXT-3): active once the communicator's
// symmetric buffers are open (nf_comm_sym_open) and not switched off (nf_comm_set_fused).
struct PeerGeom;
bool comm_fused(const nf_comm* c);
void comm_fused_step_barrier(nf_comm* c);
void comm_count_fused(nf_comm* c);
void comm_fused_site_barrier(nf_comm* c);
cudaError_t preload_kernels_green(void* green_ctx);  // peer.cu: load the library's kernels into a green context  // one fused site issued (nf_comm_sym_status reports the count)
const PeerGeom& comm_peer_geom(const nf_comm* c);
uint8_t* const* comm_peer_bases(const nf_comm* c);  // device array [geom.n]
uint8_t* comm_sym_local(const nf_comm* c);          // this rank's buffer
long long comm_peer_timeout_ns(const nf_comm* c);
}  // namespace nf

// A captured nf_model_step (plan spec.graph): replayed while the launch structure
// (key: shapes, item counts, metadata offsets, buffers) is unchanged.
struct NfGraph {
  std::vector<int64_t> key;
  cudaGraphExec_t exec = nullptr;
};

struct nf_plan {
  nf_model_cfg cfg;
  nf_plan_spec spec;
  std::string csv;
  // runtime resources (lazily created)
  int device = -1;
  cudaStream_t mem_stream = nullptr;
  cudaEvent_t ev_kqv[NF_MAX_NANO] = {};
  cudaEvent_t ev_att[NF_MAX_NANO] = {};
  cudaEvent_t ev_join = nullptr;
  cudaStream_t net_stream = nullptr;
  cudaEvent_t ev_c2n = nullptr, ev_n2c = nullptr;
  // TP pipeline edges, one per dense nano-batch (api.cu tp_* stages)
  cudaEvent_t ev_pre[NF_MAX_NANO] = {}, ev_agattn = nullptr, ev_o[NF_MAX_NANO] = {}, ev_ago = nullptr,
              ev_aro[NF_MAX_NANO] = {}, ev_d[NF_MAX_NANO] = {}, ev_ard[NF_MAX_NANO] = {};
  cudaEvent_t ev_join_n = nullptr;
  cudaStream_t green_ns = nullptr;  // network partition (TP OVERLAP plans)
  int green_net_sms = 0;
  std::vector<NfGraph> graphs;      // CUDA-graph cache (spec.graph)
  cudaStream_t cap_stream = nullptr;  // capture stream
  std::string graph_note = "not used";
  std::string note;                 // nf_plan_runtime_note buffer
  // green-context SM partitions (OVERLAP plans; green.cpp)
  bool green_tried = false, green_ok = false;
  std::string green_note = "not used";
  cudaStream_t green_cs = nullptr, green_ms = nullptr, green_cs2 = nullptr;
  cudaStream_t green_ds1 = nullptr, green_ds2 = nullptr;  // no memory partition: decode side streams (compute partition)
  cudaStream_t cs2 = nullptr;  // second compute stream (TP OVERLAP: one per dense nano-batch) outside green contexts
  cudaEvent_t ev_fork2 = nullptr, ev_join_c2 = nullptr;
  int green_dec_sms = 0, green_dense_sms = 0;
  cudaEvent_t ev_fork = nullptr, ev_join_c = nullptr, ev_join_m = nullptr, ev_join_m2 = nullptr;
  cudaEvent_t ev_upload[2] = {};
  void* pinned[2] = {nullptr, nullptr};
  size_t pinned_cap[2] = {0, 0};
  int upload_idx = 0;
};
