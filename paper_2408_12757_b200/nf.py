"""Thin ctypes binding of include/nf.h (argument marshalling only).

Every compute step runs in libnf.so's CUDA kernels; there is no Python or CPU
fallback.  If the library is missing, importing this module raises.
Device buffers are passed as integer device pointers (e.g. torch
``tensor.data_ptr()``), streams as integer ``cudaStream_t`` handles.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NF_LIB", os.path.join(_HERE, "libnf.so"))
if not os.path.exists(LIB_PATH):
    raise ImportError(f"libnf.so not built at {LIB_PATH}: run `python -m paper_2408_12757_b200.build` "
                      "(there is no CPU fallback)")
lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)

NF_OK, NF_EINVAL, NF_EUNSUPPORTED, NF_EINFEASIBLE, NF_ECUDA, NF_ENCCL, NF_ENOMEM = range(7)
SEQUENTIAL, NANO_ONLY, OVERLAP = 0, 1, 2
OP_KQV, OP_DECODE_ATTN, OP_PREFILL_ATTN, OP_O, OP_UG, OP_DOWN, OP_NET, OP_COUNT = range(8)
MAX_NANO = 4
P_i32 = C.POINTER(C.c_int32)


class NFError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"nf status {status}: {msg}")
        self.status = status


class ModelCfg(C.Structure):
    _fields_ = [("d_model", C.c_int32), ("n_layers", C.c_int32), ("n_q_heads", C.c_int32),
                ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("d_ffn", C.c_int32),
                ("vocab", C.c_int32), ("rms_eps", C.c_float), ("rope_theta", C.c_float),
                ("page_size", C.c_int32), ("tp_size", C.c_int32), ("tp_rank", C.c_int32),
                ("n_experts", C.c_int32), ("top_k", C.c_int32)]


class _Batch(C.Structure):
    _fields_ = [("n_req", C.c_int32), ("q_len", P_i32), ("kv_prefix", P_i32), ("page_indptr", P_i32),
                ("page_ids", P_i32), ("n_pages_pool", C.c_int32), ("emit", P_i32)]


class PlanSpec(C.Structure):
    _fields_ = [("mode", C.c_int32), ("n_nano", C.c_int32), ("share", C.c_int32 * MAX_NANO),
                ("sm", C.c_int32 * OP_COUNT), ("balance", C.c_int32), ("colocate", C.c_int32),
                ("n_dense", C.c_int32), ("graph", C.c_int32)]


class CurvePoint(C.Structure):
    _fields_ = [("op_kind", C.c_int32), ("units", C.c_int32), ("work", C.c_double), ("latency_s", C.c_double)]


class PlanOpts(C.Structure):
    _fields_ = [("sm_budget", C.c_int32), ("sm_quantum", C.c_int32), ("mode", C.c_int32),
                ("n_nano", C.c_int32), ("max_iters", C.c_int32)]


class LayerWeights(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("attn_norm", "w_q", "w_k", "w_v", "w_o", "w_o_col", "w_o_row",
                                          "ffn_norm", "w_gate", "w_up", "w_down", "w_router")]


class PackedLayer(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("w_qkv", "w_o", "w_o_row", "w_gate_up", "w_down", "w_router")]


class ModelWeights(C.Structure):
    _fields_ = [("embed", C.c_void_p), ("layers", C.POINTER(PackedLayer)), ("lm_head_packed", C.c_void_p)]


def _sig(name, restype, *args):
    f = getattr(lib, name)
    f.restype = restype
    f.argtypes = list(args)
    return f


_sig("nf_last_error", C.c_char_p)
_sig("nf_abi_version", C.c_int32)
_sig("nf_batch_metadata", C.c_int, C.POINTER(ModelCfg), C.POINTER(_Batch), P_i32, P_i32)
_sig("nf_snap_cuts", C.c_int, C.POINTER(_Batch), C.c_int32, P_i32, P_i32)
_sig("nf_plan_create_explicit", C.c_int, C.POINTER(ModelCfg), C.POINTER(PlanSpec), C.POINTER(C.c_void_p))
_sig("nf_plan_create", C.c_int, C.POINTER(ModelCfg), C.POINTER(_Batch), C.POINTER(CurvePoint), C.c_int32,
     C.POINTER(PlanOpts), C.POINTER(C.c_void_p))
_sig("nf_plan_get_spec", C.c_int, C.c_void_p, C.POINTER(PlanSpec))
_sig("nf_plan_export_csv", C.c_int, C.c_void_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t))
_sig("nf_plan_destroy", None, C.c_void_p)
_sig("nf_plan_hash", C.c_uint64, C.c_void_p)
_sig("nf_plan_runtime_note", C.c_char_p, C.c_void_p)
_sig("nf_plan_probe_partitions", C.c_int, C.c_void_p, C.c_void_p, P_i32, C.c_int32, C.c_void_p)
_sig("nf_comm_unique_id", C.c_int, C.c_void_p)
_sig("nf_comm_create", C.c_int, C.c_int32, C.c_int32, C.c_void_p, C.c_int32, C.POINTER(C.c_void_p))
_sig("nf_comm_destroy", None, C.c_void_p)
_sig("nf_comm_create_local", C.c_int, C.c_int32, C.c_int32, C.POINTER(C.c_void_p))
AR_F32, AR_RING = 0, 1
_sig("nf_comm_create_loopback", C.c_int, C.c_int32, C.c_int32, C.POINTER(C.c_void_p))
_sig("nf_comm_loopback_set_link", C.c_int, C.c_void_p, C.c_double)
_sig("nf_comm_sym_bytes", C.c_int, C.c_void_p, C.c_int32, C.POINTER(C.c_size_t))
_sig("nf_comm_sym_alloc", C.c_int, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p)
_sig("nf_comm_sym_open", C.c_int, C.c_void_p, C.c_void_p)
_sig("nf_comm_set_fused", C.c_int, C.c_void_p, C.c_int32)
_sig("nf_comm_sym_status", C.c_int, C.c_void_p, P_i32, C.POINTER(C.c_int64))
_sig("nf_packed_layer_bytes", C.c_int, C.POINTER(ModelCfg), C.POINTER(C.c_size_t))
_sig("nf_pack_layer", C.c_int, C.POINTER(ModelCfg), C.POINTER(LayerWeights), C.POINTER(PackedLayer), C.c_void_p)
_sig("nf_pack_lm_head", C.c_int, C.POINTER(ModelCfg), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p)
_sig("nf_workspace_size", C.c_int, C.POINTER(ModelCfg), C.POINTER(_Batch), C.POINTER(C.c_size_t))
_sig("nf_layer_forward", C.c_int, C.c_void_p, C.c_void_p, C.POINTER(PackedLayer), C.c_void_p, C.POINTER(_Batch),
     C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)
_sig("nf_model_step", C.c_int, C.c_void_p, C.c_void_p, C.POINTER(ModelWeights), C.POINTER(C.c_void_p),
     C.POINTER(_Batch), C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)


class StepOutputs(C.Structure):
    _fields_ = [("next_ids", C.c_void_p), ("logits", C.c_void_p), ("hidden", C.POINTER(C.c_void_p))]


_sig("nf_model_step_ex", C.c_int, C.c_void_p, C.c_void_p, C.POINTER(ModelWeights), C.POINTER(C.c_void_p),
     C.POINTER(_Batch), C.c_void_p, C.POINTER(StepOutputs), C.c_void_p, C.c_size_t, C.c_void_p)
_sig("nf_gemm_bf16", C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int32,
     C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_size_t, C.c_void_p)
_sig("nf_gemm_workspace_bytes", C.c_size_t, C.c_int32, C.c_int32)
_sig("nf_attention", C.c_int, C.POINTER(ModelCfg), C.POINTER(_Batch), C.c_void_p, C.c_void_p, C.c_void_p,
     C.c_void_p, C.c_size_t, C.c_int32, C.c_int32, C.c_void_p)

_sig("nf_moe_rows_cap", C.c_int64, C.POINTER(ModelCfg), C.c_int32)
_sig("nf_moe_route_ws_bytes", C.c_size_t, C.POINTER(ModelCfg), C.c_int32)
_sig("nf_moe_last_ids", C.c_int, C.POINTER(ModelCfg), C.POINTER(_Batch), C.c_void_p, C.c_size_t,
     C.POINTER(C.c_void_p))
_sig("nf_moe_route", C.c_int, C.POINTER(ModelCfg), C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
     C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)

class SchedCfg(C.Structure):
    _fields_ = [("n_pages", C.c_int32), ("page_size", C.c_int32), ("n_bdense", C.c_int32), ("bdense", P_i32),
                ("avg_decode", C.c_int32), ("eos_id", C.c_int32)]


class SchedStep(C.Structure):
    _fields_ = [("step", C.c_int64), ("n_req", C.c_int32), ("n_tokens", C.c_int32),
                ("req_ids", C.POINTER(C.c_int64)), ("q_len", P_i32), ("kv_prefix", P_i32), ("emit", P_i32),
                ("page_indptr", P_i32), ("page_ids", P_i32), ("tok_src", P_i32)]


class SchedStats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("steps", "tokens", "prefill_tokens", "decode_tokens", "finished",
                                         "generated", "useless", "evictions")] + \
               [("peak_pages_used", C.c_int32), ("running", C.c_int32), ("queued", C.c_int32)]


_sig("nf_sched_create", C.c_int, C.POINTER(SchedCfg), C.POINTER(C.c_void_p))
_sig("nf_sched_submit", C.c_int, C.c_void_p, C.c_int64, P_i32, C.c_int32, C.c_int32)
_sig("nf_sched_next", C.c_int, C.c_void_p, C.POINTER(SchedStep))
_sig("nf_sched_complete", C.c_int, C.c_void_p, C.c_int64, P_i32)
_sig("nf_sched_get_stats", C.c_int, C.c_void_p, C.POINTER(SchedStats))
_sig("nf_sched_destroy", None, C.c_void_p)
_sig("nf_assemble_tokens", C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p)

_sig("nf_kernel_launches", C.c_int64)
_sig("nf_profile_enable", C.c_int, C.c_int32)
_sig("nf_profile_read", C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_int64))
PROF_LMHEAD, PROF_MISC, PROF_COUNT = OP_COUNT, OP_COUNT + 1, OP_COUNT + 2


class Span(C.Structure):
    _fields_ = [("op", C.c_int32), ("stream", C.c_int32), ("start_ms", C.c_float), ("end_ms", C.c_float),
                ("tag", C.c_int32)]


_sig("nf_profile_timeline", C.c_int, C.POINTER(Span), C.c_int32, P_i32)
_sig("nf_profile_tag", C.c_int, C.c_int32)
PROF_NAMES = ["kqv", "decode_attn", "prefill_attn", "o_proj", "up_gate", "down", "net", "lm_head", "misc"]

EXPORTED = ["nf_plan_runtime_note", "nf_plan_probe_partitions", "nf_comm_create_local", "nf_gemm_workspace_bytes", "nf_profile_timeline", "nf_profile_tag", "nf_kernel_launches", "nf_profile_enable", "nf_profile_read", "nf_last_error", "nf_abi_version", "nf_batch_metadata", "nf_snap_cuts", "nf_plan_create_explicit",
            "nf_plan_create", "nf_plan_get_spec", "nf_plan_export_csv", "nf_plan_destroy", "nf_plan_hash", "nf_comm_unique_id",
            "nf_comm_create", "nf_comm_destroy", "nf_comm_create_loopback", "nf_comm_loopback_set_link", "nf_comm_sym_bytes", "nf_comm_sym_alloc",
            "nf_comm_sym_open", "nf_comm_set_fused", "nf_comm_sym_status", "nf_packed_layer_bytes", "nf_pack_layer", "nf_pack_lm_head",
            "nf_workspace_size", "nf_layer_forward", "nf_model_step", "nf_model_step_ex", "nf_gemm_bf16", "nf_attention",
            "nf_moe_rows_cap", "nf_moe_route_ws_bytes", "nf_moe_route", "nf_moe_last_ids", "nf_sched_create", "nf_sched_submit",
            "nf_sched_next", "nf_sched_complete", "nf_sched_get_stats", "nf_sched_destroy", "nf_assemble_tokens"]


def _check(status: int):
    if status != NF_OK:
        raise NFError(status, lib.nf_last_error().decode())


def last_error() -> str:
    return lib.nf_last_error().decode()


def model_cfg(d_model, n_layers, n_q_heads, n_kv_heads, head_dim, d_ffn, vocab, rms_eps=1e-5, rope_theta=1e4,
              page_size=16, tp_size=1, tp_rank=0, n_experts=0, top_k=2) -> ModelCfg:
    return ModelCfg(d_model, n_layers, n_q_heads, n_kv_heads, head_dim, d_ffn, vocab, rms_eps, rope_theta,
                    page_size, tp_size, tp_rank, n_experts, top_k)


class Batch:
    """Host-side nf_batch; keeps its int32 arrays alive."""

    def __init__(self, q_len, kv_prefix, page_indptr, page_ids, n_pages_pool: int, emit=None):
        self.q_len = np.ascontiguousarray(q_len, dtype=np.int32)
        self.kv_prefix = np.ascontiguousarray(kv_prefix, dtype=np.int32)
        self.page_indptr = np.ascontiguousarray(page_indptr, dtype=np.int32)
        self.page_ids = np.ascontiguousarray(page_ids, dtype=np.int32)
        self.emit = None if emit is None else np.ascontiguousarray(emit, dtype=np.int32)
        p = lambda a: a.ctypes.data_as(P_i32)
        self.c = _Batch(len(self.q_len), p(self.q_len), p(self.kv_prefix), p(self.page_indptr), p(self.page_ids),
                        int(n_pages_pool), p(self.emit) if self.emit is not None else None)

    @classmethod
    def from_any(cls, b, emit=None) -> "Batch":
        return cls(b.q_len, b.kv_prefix, b.page_indptr, b.page_ids, b.n_pages_pool, emit)

    @property
    def n_tokens(self) -> int:
        return int(self.q_len.sum())


def batch_metadata(cfg: ModelCfg, b: Batch):
    T = b.n_tokens
    pos = np.zeros(T, np.int32)
    slot = np.zeros(T, np.int32)
    _check(lib.nf_batch_metadata(C.byref(cfg), C.byref(b.c), pos.ctypes.data_as(P_i32), slot.ctypes.data_as(P_i32)))
    return pos, slot


def snap_cuts(b: Batch, shares: Sequence[int]):
    sh = np.ascontiguousarray(shares, dtype=np.int32)
    out = np.zeros(len(sh) + 1, np.int32)
    _check(lib.nf_snap_cuts(C.byref(b.c), len(sh), sh.ctypes.data_as(P_i32), out.ctypes.data_as(P_i32)))
    return out


class Plan:
    def __init__(self, handle: int):
        self.h = C.c_void_p(handle)

    @classmethod
    def explicit(cls, cfg: ModelCfg, mode: int = SEQUENTIAL, shares: Sequence[int] = (1,),
                 sm: Optional[Sequence[int]] = None, balance: bool = False, colocate: bool = False,
                 n_dense: int = 0, graph: bool = False) -> "Plan":
        spec = PlanSpec()
        spec.mode = mode
        spec.n_nano = len(shares)
        for i, s in enumerate(shares):
            spec.share[i] = int(s)
        sm = [148] * OP_COUNT if sm is None else list(sm)
        for i in range(OP_COUNT):
            spec.sm[i] = int(sm[i])
        spec.balance = int(balance)  # bool True -> 1
        spec.colocate = int(colocate)
        spec.n_dense = int(n_dense)
        spec.graph = int(graph)
        h = C.c_void_p()
        _check(lib.nf_plan_create_explicit(C.byref(cfg), C.byref(spec), C.byref(h)))
        return cls(h.value)

    @classmethod
    def search(cls, cfg: ModelCfg, shape: Batch, points: Sequence[tuple], sm_budget=148, sm_quantum=8,
               mode=OVERLAP, n_nano=2, max_iters=200) -> "Plan":
        arr = (CurvePoint * len(points))(*[CurvePoint(int(k), int(u), float(w), float(t)) for k, u, w, t in points])
        opts = PlanOpts(sm_budget, sm_quantum, mode, n_nano, max_iters)
        h = C.c_void_p()
        _check(lib.nf_plan_create(C.byref(cfg), C.byref(shape.c), arr, len(points), C.byref(opts), C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_spec(cls, cfg: ModelCfg, spec: PlanSpec) -> "Plan":
        h = C.c_void_p()
        _check(lib.nf_plan_create_explicit(C.byref(cfg), C.byref(spec), C.byref(h)))
        return cls(h.value)

    def probe_partitions(self, stream: int, comm: Optional[int] = None, n_sm: int = 148):
        """[3][n_sm] probe-CTA counts per SM for the memory / compute / network partitions."""
        out = np.zeros(3 * n_sm, np.int32)
        _check(lib.nf_plan_probe_partitions(self.h, C.c_void_p(comm), out.ctypes.data_as(P_i32), n_sm,
                                            C.c_void_p(stream)))
        return out.reshape(3, n_sm)

    def hash(self) -> int:
        """nf_plan_hash: equal on every rank of a TP group."""
        return int(lib.nf_plan_hash(self.h))

    def runtime_note(self) -> str:
        return lib.nf_plan_runtime_note(self.h).decode()

    def spec(self) -> PlanSpec:
        s = PlanSpec()
        _check(lib.nf_plan_get_spec(self.h, C.byref(s)))
        return s

    def csv(self) -> str:
        n = C.c_size_t()
        _check(lib.nf_plan_export_csv(self.h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        _check(lib.nf_plan_export_csv(self.h, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    def __del__(self):
        if getattr(self, "h", None) and self.h.value:
            lib.nf_plan_destroy(self.h)
            self.h = C.c_void_p()


def packed_layer_bytes(cfg: ModelCfg):
    out = (C.c_size_t * 6)()
    _check(lib.nf_packed_layer_bytes(C.byref(cfg), out))
    return list(out)


def pack_layer(cfg: ModelCfg, src: dict, dst: dict, stream: int):
    lw = LayerWeights(*[src.get(n) for n, _ in LayerWeights._fields_])
    pl = PackedLayer(*[dst.get(n) for n, _ in PackedLayer._fields_])
    _check(lib.nf_pack_layer(C.byref(cfg), C.byref(lw), C.byref(pl), C.c_void_p(stream)))


def pack_lm_head(cfg: ModelCfg, lm_head: int, final_norm: int, dst: int, stream: int):
    _check(lib.nf_pack_lm_head(C.byref(cfg), C.c_void_p(lm_head), C.c_void_p(final_norm), C.c_void_p(dst),
                               C.c_void_p(stream)))


def workspace_size(cfg: ModelCfg, b: Batch) -> int:
    n = C.c_size_t()
    _check(lib.nf_workspace_size(C.byref(cfg), C.byref(b.c), C.byref(n)))
    return n.value


def layer_forward(plan: Plan, packed: dict, kv_pool: int, b: Batch, x_in: int, x_out: int, ws: int, ws_bytes: int,
                  stream: int, comm: Optional[int] = None):
    pl = PackedLayer(*[packed.get(n) for n, _ in PackedLayer._fields_])
    _check(lib.nf_layer_forward(plan.h, C.c_void_p(comm), C.byref(pl), C.c_void_p(kv_pool), C.byref(b.c),
                                C.c_void_p(x_in), C.c_void_p(x_out), C.c_void_p(ws), ws_bytes, C.c_void_p(stream)))


class ModelHandle:
    """Keeps the ctypes arrays of nf_model_weights alive."""

    def __init__(self, embed: int, layers: Sequence[dict], lm_head_packed: int):
        self.layers = (PackedLayer * len(layers))(*[PackedLayer(*[d.get(n) for n, _ in PackedLayer._fields_])
                                                    for d in layers])
        self.c = ModelWeights(embed, C.cast(self.layers, C.POINTER(PackedLayer)), lm_head_packed)


def model_step(plan: Plan, model: ModelHandle, kv_pools: Sequence[int], b: Batch, token_ids: int, next_ids: int,
               ws: int, ws_bytes: int, stream: int, comm: Optional[int] = None):
    pools = (C.c_void_p * len(kv_pools))(*kv_pools)
    _check(lib.nf_model_step(plan.h, C.c_void_p(comm), C.byref(model.c), pools, C.byref(b.c), C.c_void_p(token_ids),
                             C.c_void_p(next_ids), C.c_void_p(ws), ws_bytes, C.c_void_p(stream)))


def model_step_ex(plan: Plan, model: ModelHandle, kv_pools: Sequence[int], b: Batch, token_ids: int, next_ids: int,
                  ws: int, ws_bytes: int, stream: int, comm: Optional[int] = None, logits: int = 0,
                  hidden: Optional[Sequence[int]] = None):
    pools = (C.c_void_p * len(kv_pools))(*kv_pools)
    hid = (C.c_void_p * len(hidden))(*[h or None for h in hidden]) if hidden is not None else None
    out = StepOutputs(next_ids, logits or None, C.cast(hid, C.POINTER(C.c_void_p)) if hid is not None else None)
    _check(lib.nf_model_step_ex(plan.h, C.c_void_p(comm), C.byref(model.c), pools, C.byref(b.c), C.c_void_p(token_ids),
                                C.byref(out), C.c_void_p(ws), ws_bytes, C.c_void_p(stream)))


def gemm_workspace_bytes(M: int, N: int) -> int:
    return int(lib.nf_gemm_workspace_bytes(M, N))


def gemm_bf16(A: int, lda: int, B: int, ldb: int, Cp: int, ldc: int, M: int, N: int, K: int, sm_budget: int,
              stream: int, ws: int = 0, ws_bytes: int = 0):
    _check(lib.nf_gemm_bf16(C.c_void_p(A), lda, C.c_void_p(B), ldb, C.c_void_p(Cp), ldc, M, N, K, sm_budget,
                            C.c_void_p(ws or None), ws_bytes, C.c_void_p(stream)))


def attention(cfg: ModelCfg, b: Batch, q: int, kv_pool: int, o: int, ws: int, ws_bytes: int, sm_decode: int,
              sm_prefill: int, stream: int):
    _check(lib.nf_attention(C.byref(cfg), C.byref(b.c), C.c_void_p(q), C.c_void_p(kv_pool), C.c_void_p(o),
                            C.c_void_p(ws), ws_bytes, sm_decode, sm_prefill, C.c_void_p(stream)))


def moe_rows_cap(cfg: ModelCfg, T: int) -> int:
    return int(lib.nf_moe_rows_cap(C.byref(cfg), T))


def moe_route_ws_bytes(cfg: ModelCfg, T: int) -> int:
    return int(lib.nf_moe_route_ws_bytes(C.byref(cfg), T))


def moe_route(cfg: ModelCfg, h1: int, router_packed: int, T: int, ids: int, wts: int, grp_off: int, dst: int,
              row_tok: int, ws: int, ws_bytes: int, stream: int):
    _check(lib.nf_moe_route(C.byref(cfg), C.c_void_p(h1), C.c_void_p(router_packed), T, C.c_void_p(ids),
                            C.c_void_p(wts), C.c_void_p(grp_off), C.c_void_p(dst), C.c_void_p(row_tok),
                            C.c_void_p(ws), ws_bytes, C.c_void_p(stream)))


def moe_last_ids(cfg: ModelCfg, b: Batch, ws: int, ws_bytes: int) -> int:
    """Device pointer of the [T, top_k] routing ids of the last nf_layer_forward on this workspace."""
    p = C.c_void_p()
    _check(lib.nf_moe_last_ids(C.byref(cfg), C.byref(b.c), C.c_void_p(ws), ws_bytes, C.byref(p)))
    return p.value


def kernel_launches() -> int:
    return int(lib.nf_kernel_launches())


def profile_enable(on: bool = True):
    _check(lib.nf_profile_enable(1 if on else 0))


def profile_timeline(with_tag: bool = False):
    """[(op name, stream index, start ms, end ms[, tag])] recorded since the last profile_read()."""
    n = C.c_int32()
    _check(lib.nf_profile_timeline(None, 0, C.byref(n)))
    arr = (Span * max(n.value, 1))()
    _check(lib.nf_profile_timeline(arr, n.value, C.byref(n)))
    if with_tag:
        return [(PROF_NAMES[s.op], s.stream, s.start_ms, s.end_ms, s.tag) for s in arr[:n.value]]
    return [(PROF_NAMES[s.op], s.stream, s.start_ms, s.end_ms) for s in arr[:n.value]]


def profile_tag(tag: int):
    """Tag the profile spans recorded from this thread (e.g. its emulated rank)."""
    _check(lib.nf_profile_tag(tag))


def profile_read():
    """{op name: (total ms, launches)} since the last read (synchronises)."""
    ms = (C.c_double * PROF_COUNT)()
    cnt = (C.c_int64 * PROF_COUNT)()
    _check(lib.nf_profile_read(ms, cnt))
    return {PROF_NAMES[i]: (ms[i], cnt[i]) for i in range(PROF_COUNT)}


def comm_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib.nf_comm_unique_id(buf))
    return buf.raw


def comm_create_local(tp_size: int, ar_mode: int = AR_RING):
    """Handles of an emulated single-GPU TP group (one per rank; drive rank r from thread r).
    ar_mode: AR_RING (NCCL ring order, bf16 rounding per hop; default) or AR_F32 (fp32 sum, one rounding)."""
    arr = (C.c_void_p * tp_size)()
    _check(lib.nf_comm_create_local(tp_size, ar_mode, arr))
    return [arr[i] for i in range(tp_size)]


def comm_create_loopback(tp_size: int, tp_rank: int = 0) -> int:
    """One-rank performance proxy of a tp_size group (local copies instead of peers)."""
    h = C.c_void_p()
    _check(lib.nf_comm_create_loopback(tp_size, tp_rank, C.byref(h)))
    return h.value


def comm_loopback_set_link(comm: int, link_gbs: float):
    """Link-time model of a loopback communicator (0 = off): collectives last >= ring bytes / link_gbs."""
    _check(lib.nf_comm_loopback_set_link(C.c_void_p(comm), float(link_gbs)))


def comm_destroy(h: int):
    lib.nf_comm_destroy(C.c_void_p(h))


def comm_create(tp_size: int, tp_rank: int, uid: bytes, max_ctas: int = 0) -> int:
    """NCCL communicator; max_ctas > 0 caps NCCL's CTAs per collective (the plan's network SM budget)."""
    h = C.c_void_p()
    buf = C.create_string_buffer(uid, 128)
    _check(lib.nf_comm_create(tp_size, tp_rank, buf, max_ctas, C.byref(h)))
    return h.value


def comm_sym_bytes(cfg, max_tokens: int) -> int:
    """Bytes of one rank's symmetric buffer for the fused GEMM->AllReduce (NEXT-3)."""
    n = C.c_size_t()
    _check(lib.nf_comm_sym_bytes(C.byref(cfg), max_tokens, C.byref(n)))
    return n.value


def comm_sym_alloc(h: int, cfg, max_tokens: int) -> bytes:
    """Allocate this rank's symmetric buffer; returns its 64-byte CUDA IPC handle (zeros when emulated)."""
    buf = C.create_string_buffer(64)
    _check(lib.nf_comm_sym_alloc(C.c_void_p(h), C.byref(cfg), max_tokens, buf))
    return buf.raw


def comm_sym_open(h: int, handles: Optional[Sequence[bytes]] = None):
    """Map the group's buffers (handles: every rank's 64-byte IPC handle in rank order; None when
    emulated / loopback) and switch the fused GEMM->AllReduce on."""
    buf = C.create_string_buffer(b"".join(handles), 64 * len(handles)) if handles else None
    _check(lib.nf_comm_sym_open(C.c_void_p(h), buf))


def comm_set_fused(h: int, on: bool):
    _check(lib.nf_comm_set_fused(C.c_void_p(h), 1 if on else 0))


def comm_sym_status(h: int, with_sites: bool = False):
    """Number of bounded peer waits that timed out (0 = healthy); with_sites: (timeouts, fused
    sites this rank issued)."""
    v = C.c_int32()
    n = C.c_int64()
    _check(lib.nf_comm_sym_status(C.c_void_p(h), C.byref(v), C.byref(n)))
    return (v.value, n.value) if with_sites else v.value


def comm_enable_fused_local(comms: Sequence[int], cfgs, max_tokens: int):
    """Emulated group: allocate every rank's buffer, then open them (one thread)."""
    for h, c in zip(comms, cfgs):
        comm_sym_alloc(h, c, max_tokens)
    for h in comms:
        comm_sym_open(h, None)


class Scheduler:
    """nf_sched_* (serving loop: batch scheduler + KV-cache manager, host C++)."""

    def __init__(self, n_pages: int, page_size: int, bdense: Sequence[int], avg_decode: int, eos_id: int = -1):
        self._bd = np.ascontiguousarray(bdense, dtype=np.int32)
        cfg = SchedCfg(n_pages, page_size, len(self._bd), self._bd.ctypes.data_as(P_i32), avg_decode, eos_id)
        self.h = C.c_void_p()
        _check(lib.nf_sched_create(C.byref(cfg), C.byref(self.h)))

    def submit(self, rid: int, prompt, out_len: int):
        p = np.ascontiguousarray(prompt, dtype=np.int32)
        _check(lib.nf_sched_submit(self.h, int(rid), p.ctypes.data_as(P_i32), len(p), int(out_len)))

    def next(self) -> dict:
        """The formed step as numpy copies (nf_batch arrays + token sources)."""
        st = SchedStep()
        _check(lib.nf_sched_next(self.h, C.byref(st)))
        n, T = st.n_req, st.n_tokens
        a = lambda ptr, k: np.ctypeslib.as_array(ptr, shape=(k,)).copy() if k > 0 else np.zeros(0, np.int32)
        ind = a(st.page_indptr, n + 1)
        return {"step": st.step, "req_ids": a(st.req_ids, n).astype(np.int64) if n else np.zeros(0, np.int64),
                "q_len": a(st.q_len, n), "kv_prefix": a(st.kv_prefix, n), "emit": a(st.emit, n),
                "page_indptr": ind, "page_ids": a(st.page_ids, int(ind[-1])) if n else np.zeros(0, np.int32),
                "tok_src": a(st.tok_src, T)}

    def complete(self, step: int, next_ids):
        ids = np.ascontiguousarray(next_ids, dtype=np.int32)
        _check(lib.nf_sched_complete(self.h, int(step), ids.ctypes.data_as(P_i32)))

    def stats(self) -> dict:
        s = SchedStats()
        _check(lib.nf_sched_get_stats(self.h, C.byref(s)))
        return {n: getattr(s, n) for n, _ in SchedStats._fields_}

    def __del__(self):
        if getattr(self, "h", None) and self.h.value:
            lib.nf_sched_destroy(self.h)
            self.h = C.c_void_p()


def assemble_tokens(tok_src: int, prev_next_ids: int, token_ids: int, T: int, stream: int):
    _check(lib.nf_assemble_tokens(C.c_void_p(tok_src), C.c_void_p(prev_next_ids), C.c_void_p(token_ids), T,
                                  C.c_void_p(stream)))
