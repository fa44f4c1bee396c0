/*
 * nf.h — C ABI of the B200-native NanoFlow hot path (arXiv 2408.12757).
 *
 * One thing is exported: the forward pass of a LLaMA-style decoder layer over
 * a dense batch that mixes prefill chunks and decode tokens (PAPER.md:155,
 * :504), with a paged KV cache, split into nano-batches whose
 * dense projections, paged attention and tensor-parallel collectives are
 * issued as an operation-level pipeline on SM-bounded kernels
 * (PAPER.md:537-563, :602-614), plus the model step around it.
 *
 * Conventions (all entry points):
 *  - Plain C types only.  Device buffers are `void*` device pointers owned by
 *    the caller; `stream` is a `cudaStream_t` passed as `void*`.  Host arrays
 *    are read during the call only.
 *  - bf16 tensors are row-major [rows, cols] with the stated shapes.
 *  - Calls are stream-ordered and do not synchronise the host, except
 *    nf_plan_* / nf_comm_* (host only) and the pack calls (stream-ordered).
 *  - Every argument is validated on the host before any launch.  On error the
 *    call returns a non-zero nf_status, launches nothing (validation errors) and
 *    nf_last_error() describes it.  No exception crosses the ABI.
 *  - The library never allocates device memory inside nf_layer_forward /
 *    nf_model_step / nf_attention / nf_gemm_bf16: scratch comes from the
 *    caller's workspace (size from nf_workspace_size).
 */
#ifndef NF_H_
#define NF_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NF_ABI_VERSION 3

typedef enum {
  NF_OK = 0,
  NF_EINVAL = 1,        /* invalid argument (shape, batch, buffer size) */
  NF_EUNSUPPORTED = 2,  /* valid but not implemented (e.g. head_dim not in {64,128}) */
  NF_EINFEASIBLE = 3,   /* planner: no SM assignment fits the budget */
  NF_ECUDA = 4,         /* a CUDA call failed; nf_last_error names it */
  NF_ENCCL = 5,         /* an NCCL call failed */
  NF_ENOMEM = 6         /* host allocation failed */
} nf_status;

/* Thread-local description of the last error on this thread; valid until the
 * next nf_* call on the same thread.  Never NULL. */
const char* nf_last_error(void);
int32_t nf_abi_version(void);

/* Model shape and this rank's place in tensor parallelism.
 * head-parallel TP: tp_size must divide n_kv_heads
 * and d_ffn; head_dim in {64, 128}; d_model % 256 == 0; page_size == 16. */
typedef struct {
  int32_t d_model, n_layers, n_q_heads, n_kv_heads, head_dim, d_ffn, vocab;
  float rms_eps;    /* RMSNorm epsilon (reading A-2: 1e-5) */
  float rope_theta; /* RoPE base (reading A-4) */
  int32_t page_size;
  int32_t tp_size, tp_rank;
  /* MoE FFN (Mixtral-8x7B shape; "the gating operation is required for
   * expert selection"; readings A-20..A-23): n_experts = 0 is the dense FFN.
   * 1 <= top_k <= min(n_experts, 4), n_experts <= 16 (NF_EUNSUPPORTED above). */
  int32_t n_experts, top_k;
} nf_model_cfg;

/* One step's global batch (PAPER.md:155 chunked prefill co-batched with
 * decode).  Token rows are request-major in this order: request r owns rows
 * [sum(q_len[0..r)), +q_len[r]).  Token i of request r has position
 * kv_prefix[r] + i; its K/V go to logical page (pos / page_size) of the
 * request, slot pos % page_size.  All arrays are HOST arrays.
 * NF_EINVAL: n_req < 1, q_len < 1, kv_prefix < 0, fewer than
 * ceil((kv_prefix+q_len)/page_size) pages for a request, page id outside
 * [0, n_pages_pool). */
typedef struct {
  int32_t n_req;
  const int32_t* q_len;       /* [n_req]  1 = decode, >1 = prefill chunk */
  const int32_t* kv_prefix;   /* [n_req]  tokens cached before this step */
  const int32_t* page_indptr; /* [n_req+1] CSR into page_ids */
  const int32_t* page_ids;    /* [page_indptr[n_req]] physical page of logical page i */
  int32_t n_pages_pool;       /* pages in each layer's pool */
  const int32_t* emit;        /* [n_req] or NULL (= all): 1 if the request samples a token */
} nf_batch;

/* ------------------------------------------------------------------ host-only metadata (a1) */
/* pos_out[t] = kv_prefix[r] + i; slot_out[t] = page_ids[page_indptr[r] + pos/page] * page + pos % page.
 * Arrays sized [T = sum q_len].  Bit-exact contract with oracle/metadata.py. */
nf_status nf_batch_metadata(const nf_model_cfg* cfg, const nf_batch* b, int32_t* pos_out, int32_t* slot_out);
/* Nano-batch cut snapping (reading A-10): share[k] are integer token-share
 * weights of n_nano nano-batches; cut k is the request boundary nearest to
 * T * (share[0]+..+share[k-1]) / sum(share), ties to the lower one.
 * req_cuts_out: [n_nano+1] request indices (0 .. n_req). */
nf_status nf_snap_cuts(const nf_batch* b, int32_t n_nano, const int32_t* share, int32_t* req_cuts_out);

/* ------------------------------------------------------------------ plans */
enum { NF_SEQUENTIAL = 0, NF_NANO_ONLY = 1, NF_OVERLAP = 2 }; /* ablation modes */
enum {
  NF_OP_KQV = 0,
  NF_OP_DECODE_ATTN = 1,
  NF_OP_PREFILL_ATTN = 2,
  NF_OP_O = 3,
  NF_OP_UG = 4,
  NF_OP_DOWN = 5,
  NF_OP_NET = 6,
  NF_OP_COUNT = 7
};
#define NF_MAX_NANO 4
/* A nano-batch plan: "the size of each nano-batch and the allocation of
 * execution units to the operations".  share: token-share
 * weights of the nano-batches (snapped to requests per batch); sm: SM budget
 * per op kind (1..148).  SEQUENTIAL ignores n_nano/share (one nano-batch). */
typedef struct {
  int32_t mode;
  int32_t n_nano;              /* 1..NF_MAX_NANO */
  int32_t share[NF_MAX_NANO];
  int32_t sm[NF_OP_COUNT];
  int32_t balance;             /* model step only: 0 request-order cuts (A-10); 1 requests balanced by tokens
                                  and decode KV (A-10b); 2 exact token shares + decode-KV balance, prefill
                                  requests split across nano-batches where needed (A-10c) */
  int32_t colocate;            /* 1: attention CTAs co-reside with GEMM CTAs on the same SMs (3-stage GEMM ring,
                                  4-warp decode CTAs) instead of disjoint SM partitions */
  int32_t n_dense;             /* dense (O / UGD / network) nano-batches; 0 = n_nano.  At tp_size > 1 the
                                  n_nano attention nano-batches are grouped into n_dense contiguous dense
                                  nano-batches (n_nano % n_dense == 0): the paper's 4-way KQV/attention and
                                  2-way O/UGD/network split is n_nano 4, n_dense 2.  Dense
                                  nano-batch 0 runs column-parallel O + AllGather, the others row-parallel O +
                                  AllReduce.  At tp_size 1 it must be 0 or n_nano. */
  int32_t graph;               /* nf_model_step only: 1 = capture the step's launches in a CUDA graph per
                                  (batch structure, buffers) and replay it; the step metadata is uploaded
                                  outside the graph.  Ignored with an emulated communicator. */
} nf_plan_spec;

/* One measured kernel-curve sample, CSV `op_kind,resource_class,units,work,latency_s`. */
typedef struct {
  int32_t op_kind;   /* NF_OP_* */
  int32_t units;     /* SMs */
  double work;       /* tokens (dense/net) or KV keys (attention) */
  double latency_s;
} nf_curve_point;

typedef struct {
  int32_t sm_budget;  /* total SMs (148) */
  int32_t sm_quantum; /* assignment granularity (8) */
  int32_t mode;
  int32_t n_nano;     /* 2 single GPU, 4 attention / 2 dense at TP>1 */
  int32_t max_iters;  /* greedy iterations (200) */
} nf_plan_opts;

typedef struct nf_plan nf_plan;
/* Explicit plan (tests, ablations).  NF_EINVAL on out-of-range fields. */
nf_status nf_plan_create_explicit(const nf_model_cfg* cfg, const nf_plan_spec* spec, nf_plan** out);
/* Autosearch: critical-path greedy SM assignment per
 * candidate split over measured curves; keeps the shortest per-layer period.
 * NF_EINFEASIBLE if no candidate fits opts->sm_budget. */
nf_status nf_plan_create(const nf_model_cfg* cfg, const nf_batch* shape, const nf_curve_point* pts, int32_t n_pts,
                         const nf_plan_opts* opts, nf_plan** out);
nf_status nf_plan_get_spec(const nf_plan* plan, nf_plan_spec* out);
/* Gantt CSV `node_id,kind,nano_index,units,start_s,end_s` of the searched schedule. */
nf_status nf_plan_export_csv(const nf_plan* plan, char* buf, size_t cap, size_t* len);
void nf_plan_destroy(nf_plan* plan);
/* 64-bit hash of the plan's launch decisions and model config (tp_rank excluded).  The
 * ranks of one TP group must hold plans with equal hashes: they then issue the same
 * collectives in the same order (callers check it with one AllGather at setup). */
uint64_t nf_plan_hash(const nf_plan* plan);
/* How an OVERLAP plan partitions the GPU at run time (green-context SM
 * partitions, or why they are not used).  Valid until the plan is destroyed. */
const char* nf_plan_runtime_note(const nf_plan* plan);

/* ------------------------------------------------------------------ tensor-parallel communicator */
typedef struct nf_comm nf_comm;
/* 128-byte NCCL unique id, created on rank 0 and broadcast by the caller. */
nf_status nf_comm_unique_id(void* id_out_128);
/* NCCL communicator (bf16 AllGather / AllReduce over NVLink / NVSwitch).  max_ctas > 0 caps the
 * CTAs of every collective (ncclConfig_t.maxCTAs): an OVERLAP plan's network partition
 * (plan sm[NF_OP_NET]) is only used when max_ctas fits in it, so that
 * the collective kernels can never occupy the compute or memory partitions.  0 = NCCL default. */
nf_status nf_comm_create(int32_t tp_size, int32_t tp_rank, const void* id_128, int32_t max_ctas, nf_comm** out);
/* tp_size communicators of one emulated group living in this process on one
 * GPU (tests, rank-local studies): rank r's calls run on host thread r;
 * collectives meet at a host barrier and exchange device buffers with
 * stream-ordered copies.  ar_mode selects the AllReduce arithmetic:
 *   NF_AR_F32  : sum of the bf16 inputs in fp32 in rank order, one rounding;
 *   NF_AR_RING : NCCL's ring order with a bf16 rounding after every hop (chunk c of N
 *                starts at rank (c+1) mod N, adds ranks c+2, ..., c in turn).
 * Both are bit-identical on all ranks.  comms_out: [tp_size]. */
enum { NF_AR_F32 = 0, NF_AR_RING = 1 };
nf_status nf_comm_create_local(int32_t tp_size, int32_t ar_mode, nf_comm** comms_out);
/* Performance proxy of one rank of a tp_size group on one GPU (bench --config c3loop):
 * collectives move this rank's bytes locally (AllGather: its buffer copied into every
 * slot; AllReduce: a local copy, values unchanged) -- the rank's compute, pipeline and
 * local copy traffic without peers.  Results are NOT the model's (no reduction). */
nf_status nf_comm_create_loopback(int32_t tp_size, int32_t tp_rank, nf_comm** out);
/* Link-time model for a loopback communicator (bench --config c3loop --net-model nvlink): every
 * collective lasts at least the bytes a ring moves per GPU divided by link_gbs (GB/s).  An
 * AllGather of N slots of S bytes moves (N-1) S; an AllReduce of B bytes moves 2 (N-1)/N B.
 * The local copy runs first; one thread per block then holds until that time has passed since
 * the copy kernel started, on the collective's stream.  This models the link's duration; it
 * is not a measurement of NVLink.  link_gbs = 0 (the default) turns the model off.
 * NF_EINVAL if comm is not a loopback communicator, or if link_gbs is negative or > 1e6. */
nf_status nf_comm_loopback_set_link(nf_comm* comm, double link_gbs);
void nf_comm_destroy(nf_comm* comm);

/* ---- Fused collectives over peer memory (PAPER.md:628 used
 * MSCCL++ SM-constrained collective kernels, PAPER.md:612-614 the network SM budget).
 * With symmetric buffers open, every row-parallel GEMM whose output the TP group sums
 * (O2 row-parallel O projection, Down projection) runs a fused
 * epilogue that stores each 128x256 bf16 partial block directly into the block owner's
 * staging slot (owner = block % tp_size; a peer store over NVLink), and the owner's
 * reduce kernel on the network stream sums the tp_size partials in rank order in fp32
 * (one bf16 rounding: the NF_AR_F32 arithmetic) and pushes the block to every rank
 * (all-gather), replacing the NCCL AllReduce of that site (Down: dense FFN only, MoE layers
 * keep the communicator's AllReduce).  The O column-parallel projection's AllGather
 * is fused the same way: its residual epilogue stores the rank's output
 * slice into every rank's all-gather region.  The attention-output AllGather stays on
 * the communicator.  All ranks of a group must enable it together.
 *
 * nf_comm_sym_bytes: size of one rank's symmetric buffer for steps of at most max_tokens
 *   rows (d_model % 256 == 0).
 * nf_comm_sym_alloc: allocates this rank's buffer (cudaMalloc; owned by the communicator,
 *   freed by nf_comm_destroy) and writes its 64-byte CUDA IPC handle to ipc_handle_out_64
 *   (may be NULL; all-zero for emulated / loopback communicators).  The caller gathers the
 *   tp_size handles (rank order) and passes them to nf_comm_sym_open.
 * nf_comm_sym_open: maps the other ranks' buffers (cudaIpcOpenMemHandle; emulated groups
 *   use their shared registry and ignore ipc_handles, which may then be NULL; a loopback
 *   rank runs its sites as a group of one) and switches the fused path on.
 *   NF_EINVAL before nf_comm_sym_alloc or when an emulated rank has no buffer yet.
 * nf_comm_set_fused: 0 = back to the plain AllReduce (A/B), 1 = fused (buffers must be open).
 * nf_comm_sym_status: number of bounded waits that timed out so far (0 = healthy; a
 *   timeout means a peer never delivered -- results of that step are invalid, nothing
 *   hangs; NF_PEER_TIMEOUT_MS sets the bound, default 20000; nf_last_error() then names the
 *   first one) and, if fused_sites_out is not NULL, how many fused sites this rank issued.
 *   Synchronous.
 * Where it runs: the owner reduce spins until the partials arrive, so it is used only where
 * it cannot hold SMs a producer needs: SEQUENTIAL / NANO_ONLY plans (single compute stream,
 * the reduce follows the GEMM in stream order) and OVERLAP plans whose network operation has
 * its own green-context partition (plan sm[NF_OP_NET]); other OVERLAP plans keep the
 * AllReduce of the communicator. */
nf_status nf_comm_sym_bytes(const nf_model_cfg* cfg, int32_t max_tokens, size_t* bytes);
nf_status nf_comm_sym_alloc(nf_comm* comm, const nf_model_cfg* cfg, int32_t max_tokens, void* ipc_handle_out_64);
nf_status nf_comm_sym_open(nf_comm* comm, const void* ipc_handles);
nf_status nf_comm_set_fused(nf_comm* comm, int32_t on);
nf_status nf_comm_sym_status(nf_comm* comm, int32_t* timeouts_out, int64_t* fused_sites_out);

/* Evidence of execution-unit partitioning: launches a probe kernel
 * (4 CTAs per SM of the device) on each of the plan's partition streams -- memory,
 * compute, network -- as an OVERLAP step would use them, and writes, per partition,
 * smids_out[part * n_sm + sm] = number of probe CTAs that ran on SM `sm` (%smid).
 * n_sm = device SM count (148); partitions the plan does not use are all-zero.
 * Synchronises `stream`.  NF_EINVAL if the plan is not an OVERLAP plan. */
nf_status nf_plan_probe_partitions(nf_plan* plan, nf_comm* comm, int32_t* smids_out, int32_t n_sm, void* stream);

/* ------------------------------------------------------------------ weights */
/* This rank's shards in canonical [out, in] row-major bf16 (device):
 * w_q [qh/N*hd, D], w_k/w_v [kh/N*hd, D], w_o [D, qh*hd] FULL (TP1) or NULL,
 * w_o_col [D/N, qh*hd] and w_o_row [D, qh/N*hd] (TP>1), w_gate/w_up [F/N, D],
 * w_down [D, F/N], norms [D].
 * MoE (n_experts = E > 0): w_router [E, D] (replicated), w_gate/w_up [E][F/N, D] and
 * w_down [E][D, F/N] expert-major (each expert's F columns split across ranks). */
typedef struct {
  const void *attn_norm, *w_q, *w_k, *w_v, *w_o, *w_o_col, *w_o_row, *ffn_norm, *w_gate, *w_up, *w_down;
  const void* w_router; /* MoE only, else NULL */
} nf_layer_weights;
/* Packed, kernel-ready layer (caller-allocated device buffers, sizes from nf_packed_layer_bytes):
 * w_qkv [(qh+2kh)/N*hd, D] with gamma_attn folded into columns;
 * w_o: TP1 [D, qh*hd]; TP>1 w_o = w_o_col [D/N, D] and w_o_row [D, D/N];
 * w_gate_up [ceil(F/N/128)*256, D] gate/up interleaved in 128-row blocks, gamma_ffn folded;
 * w_down [D, F/N].
 * MoE: w_gate_up [E][ceil(F/N/128)*256, D], w_down [E][D, F/N], w_router fp32 [E, D] = W_r * gamma_ffn
 * (exact: a product of two bf16 values). */
typedef struct {
  void *w_qkv, *w_o, *w_o_row, *w_gate_up, *w_down;
  void* w_router; /* MoE only (bytes_out[5] > 0) */
} nf_packed_layer;
nf_status nf_packed_layer_bytes(const nf_model_cfg* cfg, size_t bytes_out[6]);
nf_status nf_pack_layer(const nf_model_cfg* cfg, const nf_layer_weights* src, const nf_packed_layer* dst, void* stream);
/* Vocab-parallel LM head: lm_head is this rank's vocab shard [V/N, D]
 * (rows tp_rank*V/N .. +V/N of the full [V, D] head; the full head at tp_size 1);
 * dst [V/N, D] = lm_head * gamma_final.  NF_EUNSUPPORTED unless (V/N) % 32 == 0. */
nf_status nf_pack_lm_head(const nf_model_cfg* cfg, const void* lm_head, const void* final_norm, void* dst, void* stream);

typedef struct {
  const void* embed;               /* [V, D] full, replicated */
  const nf_packed_layer* layers;   /* host array [n_layers] of device pointers */
  const void* lm_head_packed;      /* [V/N, D] this rank's vocab shard (nf_pack_lm_head) */
} nf_model_weights;

/* ------------------------------------------------------------------ forward */
/* Workspace bytes for nf_layer_forward / nf_model_step / nf_attention with this batch. */
nf_status nf_workspace_size(const nf_model_cfg* cfg, const nf_batch* b, size_t* bytes);

/* One decoder layer: x_out = layer(x_in), appending this
 * step's K/V into kv_pool (layout [n_pages_pool][2][kh/N][page][hd] bf16).
 * x_in, x_out: [T, D] bf16, replicated on every rank.  comm may be NULL at TP1. */
nf_status nf_layer_forward(const nf_plan* plan, nf_comm* comm, const nf_packed_layer* w, void* kv_pool,
                           const nf_batch* b, const void* x_in, void* x_out, void* ws, size_t ws_bytes, void* stream);

/* Embedding gather -> n_layers decoder layers -> final RMSNorm -> LM head on
 * the last row of each emitting request -> greedy argmax (ties: lowest id).
 * token_ids: device int32 [T]; next_ids: device int32 [n_req] (-1 if not emitted).
 * kv_pools: host array [n_layers] of device pool pointers. */
nf_status nf_model_step(const nf_plan* plan, nf_comm* comm, const nf_model_weights* w, void* const* kv_pools,
                        const nf_batch* b, const int32_t* token_ids, int32_t* next_ids, void* ws, size_t ws_bytes,
                        void* stream);
/* nf_model_step with optional inspection outputs (parity tests; not on the hot path):
 *  logits: device bf16 [n_emit, V/N]: this rank's vocab shard of the logits of every emitting
 *          request's last row (the final-RMSNorm-ed hidden state times the packed LM head), rows in
 *          caller request order of the emitting requests; NULL = not written.
 *  hidden: host array [n_layers + 1] of device bf16 [T, D] buffers (or NULL entries):
 *          hidden[0] = the embedding rows, hidden[l + 1] = decoder layer l's output, rows in caller
 *          token order; NULL = none written.  Copies are taken as each layer's rows complete.
 * Writing them does not change next_ids or any other result. */
typedef struct {
  int32_t* next_ids;      /* device [n_req] (required) */
  void* logits;           /* device bf16 [n_emit, V/N] or NULL */
  void* const* hidden;    /* host [n_layers + 1] of device [T, D] bf16, or NULL */
} nf_step_outputs;
nf_status nf_model_step_ex(const nf_plan* plan, nf_comm* comm, const nf_model_weights* w, void* const* kv_pools,
                           const nf_batch* b, const int32_t* token_ids, const nf_step_outputs* out, void* ws,
                           size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------ op-level entry points (tests, profiling) */
/* C[M, N] = A[M, K] . B[N, K]^T, bf16 in/out, f32 accumulation (tcgen05).
 * Leading dimensions in elements, multiples of 8; N % 32 == 0.  ws (device,
 * 256-byte aligned, >= nf_gemm_workspace_bytes(M, N)) enables the stream-K
 * tail schedule; ws == NULL runs whole tiles only.  The fp32 summation order
 * depends on the grid (SM budget) when stream-K is active. */
nf_status nf_gemm_bf16(const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc, int32_t M,
                       int32_t N, int32_t K, int32_t sm_budget, void* ws, size_t ws_bytes, void* stream);
size_t nf_gemm_workspace_bytes(int32_t M, int32_t N);
/* Paged causal GQA attention of PAPER.md:161 for every token of the batch:
 * q [T, qh, hd] (post-RoPE), kv_pool already holding this step's K/V,
 * o [T, qh*hd].  Decode tokens (q_len == 1) run on the decode kernel with
 * sm_decode SMs, prefill chunks on the prefill kernel with sm_prefill SMs. */
nf_status nf_attention(const nf_model_cfg* cfg, const nf_batch* b, const void* q, const void* kv_pool, void* o,
                       void* ws, size_t ws_bytes, int32_t sm_decode, int32_t sm_prefill, void* stream);

/* MoE gating and token grouping of one batch of rows (readings A-21, A-23),
 * the first two steps of the MoE FFN that nf_layer_forward runs, exposed for the
 * bit-exact index tests.  h1 [T, D] bf16 (device); router_packed fp32 [E, D] (from
 * nf_pack_layer).  Outputs (device): ids/wts [T, top_k] (experts by descending logit,
 * lowest index on ties; weights = softmax over the selected logits), grp_off [E+1]
 * (expert segments padded to 128 rows), dst [T, top_k] (grouped row of each
 * assignment, token-major within an expert), row_tok [nf_moe_rows_cap(T)] (token of
 * each grouped row, -1 = padding; rows >= grp_off[E] untouched).  ws: device scratch
 * of nf_moe_route_ws_bytes bytes. */
int64_t nf_moe_rows_cap(const nf_model_cfg* cfg, int32_t T);
size_t nf_moe_route_ws_bytes(const nf_model_cfg* cfg, int32_t T);
nf_status nf_moe_route(const nf_model_cfg* cfg, const void* h1, const void* router_packed, int32_t T, int32_t* ids,
                       float* wts, int32_t* grp_off, int32_t* dst, int32_t* row_tok, void* ws, size_t ws_bytes,
                       void* stream);

/* Inspection (parity tests): device pointer to the routing ids [T, top_k] that the most
 * recent nf_layer_forward with this workspace and batch chose (rows in the caller's token
 * order; the experts of each row by descending logit).  Valid until the workspace is reused. */
nf_status nf_moe_last_ids(const nf_model_cfg* cfg, const nf_batch* b, const void* ws, size_t ws_bytes,
                          const int32_t** ids_out);

/* ------------------------------------------------------------------ serving loop (NEXT-4) */
/* Global batch scheduler + KV-cache manager (host, C++): continuous batching with
 * chunked prefill, discrete dense batch sizes,
 * peak-memory admission and eviction, asynchronous EOS
 * detection one step late; readings A-25..A-29 in DESIGN.md,
 * bit-exact contract with oracle/serving.py.  Protocol per step i:
 *   nf_sched_next -> (upload tok_src, nf_assemble_tokens, nf_model_step of step i)
 *   -> nf_sched_complete(i - 1, next_ids of step i - 1) -> nf_sched_next ...
 * i.e. step i+1 is formed before step i's tokens are read; a decode whose input
 * token was produced by the previous step gets tok_src = -(1 + row) (row of that
 * step's next_ids), every other token id is known on the host. */
typedef struct {
  int32_t n_pages;       /* pages of the KV pool (per layer) */
  int32_t page_size;     /* 16 */
  int32_t n_bdense;      /* allowed dense batch sizes (tokens), any order, 1..16 of them */
  const int32_t* bdense;
  int32_t avg_decode;    /* average decode length for the peak-memory estimate */
  int32_t eos_id;        /* token id ending a request, or -1 */
} nf_sched_cfg;
typedef struct nf_sched nf_sched;
/* One formed step; arrays are owned by the scheduler and valid until the next
 * nf_sched_next.  n_req == 0: nothing runnable (idle or blocked). */
typedef struct {
  int64_t step;
  int32_t n_req, n_tokens;
  const int64_t* req_ids;                 /* [n_req] */
  const int32_t *q_len, *kv_prefix, *emit; /* [n_req] (nf_batch fields) */
  const int32_t *page_indptr, *page_ids;  /* [n_req+1], [page_indptr[n_req]] */
  const int32_t* tok_src;                 /* [n_tokens]: >= 0 token id; < 0: next_ids[-(1+v)] of step - 1 */
} nf_sched_step;
typedef struct {
  int64_t steps, tokens, prefill_tokens, decode_tokens, finished, generated, useless, evictions;
  int32_t peak_pages_used, running, queued;
} nf_sched_stats;
nf_status nf_sched_create(const nf_sched_cfg* cfg, nf_sched** out);
/* Queue a request (first come, first served).  prompt: host [prompt_len] token ids
 * (copied); out_len: the position of its EOS (synthetic traces).  NF_EINVAL on a
 * duplicate id or empty prompt / out_len < 1. */
nf_status nf_sched_submit(nf_sched* s, int64_t req_id, const int32_t* prompt, int32_t prompt_len, int32_t out_len);
/* NF_EINVAL if the protocol above was not followed (a step older than the previous
 * one still not completed when a decode needs its token); the scheduler is then
 * unusable (destroy it). */
nf_status nf_sched_next(nf_sched* s, nf_sched_step* out);
/* next_ids: host [n_req of that step] (the step's nf_model_step output).  NF_EINVAL
 * if the step is not pending. */
nf_status nf_sched_complete(nf_sched* s, int64_t step, const int32_t* next_ids);
nf_status nf_sched_get_stats(const nf_sched* s, nf_sched_stats* out);
void nf_sched_destroy(nf_sched* s);
/* token_ids[t] = tok_src[t] >= 0 ? tok_src[t] : prev_next_ids[-(1 + tok_src[t])]  (device arrays, one launch). */
nf_status nf_assemble_tokens(const int32_t* tok_src, const int32_t* prev_next_ids, int32_t* token_ids, int32_t T,
                             void* stream);

/* ------------------------------------------------------------------ instrumentation */
/* Cumulative number of CUDA kernels this process launched through libnf. */
int64_t nf_kernel_launches(void);
/* Op kinds of the per-kernel timing (NF_OP_* plus the LM head and small kernels). */
enum { NF_PROF_LMHEAD = NF_OP_COUNT, NF_PROF_MISC = NF_OP_COUNT + 1, NF_PROF_COUNT = NF_OP_COUNT + 2 };
/* on != 0: record CUDA events on the launching stream around every kernel
 * launch (adds ~1 us host time per launch). */
nf_status nf_profile_enable(int32_t on);
/* Synchronises the recorded events and returns, per op kind, the summed
 * event-to-event milliseconds (ms_out[NF_PROF_COUNT]) and the number of
 * launches (count_out[NF_PROF_COUNT]); clears the records. */
nf_status nf_profile_read(double* ms_out, int64_t* count_out);
/* One recorded kernel span: op kind, stream index (order of first use), start/end in ms
 * since profiling was enabled. */
typedef struct {
  int32_t op, stream;
  float start_ms, end_ms;
  int32_t tag;  /* the launching thread's nf_profile_tag (-1 if none) */
} nf_span;
/* Tag the spans recorded from the calling thread (e.g. its rank in an emulated TP group). */
nf_status nf_profile_tag(int32_t tag);
/* Copies up to cap spans recorded since the last nf_profile_read (call before it);
 * *n_out = number recorded.  Synchronises the events. */
nf_status nf_profile_timeline(nf_span* out, int32_t cap, int32_t* n_out);

#ifdef __cplusplus
}
#endif
#endif /* NF_H_ */
