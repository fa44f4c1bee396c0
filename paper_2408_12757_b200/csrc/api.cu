// C ABI of the NanoFlow hot path: validation, step metadata, workspace,
// weight packing, the nano-batch pipeline executor and the op-level entries.
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <ctime>
#include <cstring>
#include <mutex>
#include <numeric>
#include <string>

#include "attention.cuh"
#include "gemm.cuh"
#include "host.h"
#include "moe.cuh"
#include "misc.cuh"
#include "peer.cuh"
#include "profile.h"

namespace nf {

namespace {
thread_local std::string g_err = "no error";
int g_num_sms = 0;

int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0, n = 148;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess)
      g_num_sms = n;
    else
      g_num_sms = 148;
  }
  return g_num_sms;
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
}  // namespace

nf_status set_error(nf_status s, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

int64_t batch_tokens(const nf_batch* b) {
  int64_t T = 0;
  for (int r = 0; r < b->n_req; ++r) T += b->q_len[r];
  return T;
}

nf_status validate_cfg(const nf_model_cfg* c) {
  if (!c) return set_error(NF_EINVAL, "cfg is NULL");
  if (c->tp_size < 1 || c->tp_rank < 0 || c->tp_rank >= c->tp_size)
    return set_error(NF_EINVAL, "bad tp_size/tp_rank %d/%d", c->tp_size, c->tp_rank);
  if (c->d_model <= 0 || c->n_q_heads <= 0 || c->n_kv_heads <= 0 || c->d_ffn <= 0 || c->vocab <= 0 || c->n_layers <= 0)
    return set_error(NF_EINVAL, "non-positive model dimension");
  if (c->n_q_heads % c->n_kv_heads) return set_error(NF_EINVAL, "n_kv_heads must divide n_q_heads");
  if (c->n_kv_heads % c->tp_size) return set_error(NF_EINVAL, "tp_size must divide n_kv_heads");
  if (c->d_ffn % c->tp_size || c->d_model % c->tp_size) return set_error(NF_EINVAL, "tp_size must divide d_ffn and d_model");
  if (c->head_dim != 64 && c->head_dim != 128) return set_error(NF_EUNSUPPORTED, "head_dim %d not in {64,128}", c->head_dim);
  if (c->page_size != 16) return set_error(NF_EUNSUPPORTED, "page_size must be 16");
  if (c->d_model % 256) return set_error(NF_EUNSUPPORTED, "d_model must be a multiple of 256");
  if ((c->d_ffn / c->tp_size) % 32) return set_error(NF_EUNSUPPORTED, "d_ffn/tp_size must be a multiple of 32");
  if (c->vocab % c->tp_size) return set_error(NF_EINVAL, "tp_size must divide vocab (vocab-parallel LM head)");
  if ((c->vocab / c->tp_size) % 32) return set_error(NF_EUNSUPPORTED, "vocab/tp_size must be a multiple of 32");
  if (c->n_q_heads / c->n_kv_heads > 8) return set_error(NF_EUNSUPPORTED, "GQA group > 8 (decode kernel N = 8)");
  if (!(c->rms_eps > 0) || !(c->rope_theta > 1)) return set_error(NF_EINVAL, "bad rms_eps / rope_theta");
  if (c->n_experts < 0) return set_error(NF_EINVAL, "n_experts %d < 0", c->n_experts);
  if (c->n_experts > 0) {
    if (c->top_k < 1 || c->top_k > c->n_experts) return set_error(NF_EINVAL, "top_k %d not in [1, n_experts]", c->top_k);
    if (c->n_experts > MOE_MAX_EXPERTS || c->top_k > MOE_MAX_TOPK)
      return set_error(NF_EUNSUPPORTED, "MoE with %d experts / top-%d (max %d / %d)", c->n_experts, c->top_k,
                       MOE_MAX_EXPERTS, MOE_MAX_TOPK);
  }
  return NF_OK;
}

// Packed-layer pointers the forward pass dereferences (NF_EINVAL instead of a device fault).
nf_status validate_packed(const nf_model_cfg* c, const nf_packed_layer* w, int layer) {
  if (!w->w_qkv || !w->w_o || !w->w_gate_up || !w->w_down)
    return set_error(NF_EINVAL, "layer %d: NULL packed weight", layer);
  if (c->tp_size > 1 && !w->w_o_row) return set_error(NF_EINVAL, "layer %d: w_o_row required at tp_size > 1", layer);
  if (c->n_experts > 0 && !w->w_router) return set_error(NF_EINVAL, "layer %d: MoE layer without w_router", layer);
  return NF_OK;
}

int64_t moe_rows_cap(const nf_model_cfg* c, int64_t T) {
  return c->n_experts > 0 ? ((T * c->top_k + GEMM_BM - 1) / GEMM_BM + c->n_experts) * GEMM_BM : 0;
}

nf_status validate_batch(const nf_model_cfg* c, const nf_batch* b) {
  if (!b) return set_error(NF_EINVAL, "batch is NULL");
  if (b->n_req < 1) return set_error(NF_EINVAL, "n_req must be >= 1");
  if (!b->q_len || !b->kv_prefix || !b->page_indptr || !b->page_ids)
    return set_error(NF_EINVAL, "batch arrays must be non-NULL");
  if (b->page_indptr[0] != 0) return set_error(NF_EINVAL, "page_indptr[0] must be 0");
  const int P = c ? c->page_size : 16;
  for (int r = 0; r < b->n_req; ++r) {
    if (b->q_len[r] < 1) return set_error(NF_EINVAL, "q_len[%d] = %d < 1", r, b->q_len[r]);
    if (b->kv_prefix[r] < 0) return set_error(NF_EINVAL, "kv_prefix[%d] = %d < 0", r, b->kv_prefix[r]);
    const int64_t need = ((int64_t)b->kv_prefix[r] + b->q_len[r] + P - 1) / P;
    const int64_t have = (int64_t)b->page_indptr[r + 1] - b->page_indptr[r];
    if (have < need) return set_error(NF_EINVAL, "request %d has %lld pages, needs %lld", r, (long long)have, (long long)need);
  }
  const int64_t np = b->page_indptr[b->n_req];
  for (int64_t i = 0; i < np; ++i)
    if (b->page_ids[i] < 0 || b->page_ids[i] >= b->n_pages_pool)
      return set_error(NF_EINVAL, "page id %d at %lld outside pool of %d", b->page_ids[i], (long long)i, b->n_pages_pool);
  if (batch_tokens(b) > (1 << 24)) return set_error(NF_EINVAL, "too many tokens");
  return NF_OK;
}

// Balanced request -> nano-batch assignment (reading A-10b): prefill
// chunks by tokens (largest first, to the nano-batch with the most remaining
// token share), then decode requests by KV length (longest first, to the
// nano-batch with the least accumulated attention work).
void balance_requests(const nf_batch* b, int nn, const int32_t* share, std::vector<std::vector<int>>* groups) {
  const int n_req = b->n_req;
  int64_t T = batch_tokens(b), tot = 0;
  for (int k = 0; k < nn; ++k) tot += share[k];
  std::vector<double> cap(nn), kv(nn, 0.0);
  for (int k = 0; k < nn; ++k) cap[k] = (double)T * share[k] / tot;
  std::vector<std::vector<int>>& grp = *groups;
  grp.assign(nn, {});
  std::vector<int> pre, dec;
  for (int r = 0; r < n_req; ++r) (b->q_len[r] > 1 ? pre : dec).push_back(r);
  std::stable_sort(pre.begin(), pre.end(), [&](int x, int y) { return b->q_len[x] > b->q_len[y]; });
  std::stable_sort(dec.begin(), dec.end(), [&](int x, int y) { return b->kv_prefix[x] > b->kv_prefix[y]; });
  for (int r : pre) {
    int best = 0;
    for (int k = 1; k < nn; ++k)
      if (cap[k] > cap[best]) best = k;
    grp[best].push_back(r);
    cap[best] -= b->q_len[r];
    kv[best] += (double)b->q_len[r] * (b->kv_prefix[r] + b->q_len[r] / 2.0) / 64.0;
  }
  for (int r : dec) {
    int best = 0;
    for (int k = 1; k < nn; ++k)
      if (kv[k] < kv[best]) best = k;
    grp[best].push_back(r);
    cap[best] -= 1;
    kv[best] += b->kv_prefix[r] + 1;
  }
  for (auto& g : grp) std::sort(g.begin(), g.end());
}

std::vector<int> snap_cuts_impl(const std::vector<int64_t>& bound, int n_nano, const int32_t* share) {
  // bound[b] = token offset of request boundary b (b = 0..n_req); reading A-10
  const int n_req = (int)bound.size() - 1;
  const int64_t T = bound[n_req];
  int64_t tot = 0;
  for (int k = 0; k < n_nano; ++k) tot += share[k];
  std::vector<int> cuts{0};
  int64_t acc = 0;
  for (int k = 0; k + 1 < n_nano; ++k) {
    acc += share[k];
    // target = T*acc/tot; compare |bound*tot - T*acc| exactly in integers
    int best = 0;
    __int128 bd = -1;
    for (int b = 0; b <= n_req; ++b) {
      __int128 d = (__int128)bound[b] * tot - (__int128)T * acc;
      if (d < 0) d = -d;
      if (bd < 0 || d < bd) { bd = d; best = b; }
    }
    cuts.push_back(std::max(best, cuts.back()));
  }
  cuts.push_back(n_req);
  return cuts;
}

size_t meta_words_bound(const nf_model_cfg* c, const nf_batch* b) {
  const int64_t T = batch_tokens(b);
  const int qh = c->n_q_heads / c->tp_size, kh = c->n_kv_heads / c->tp_size;
  int64_t pf_tiles = 0;
  for (int r = 0; r < b->n_req; ++r)
    if (b->q_len[r] > 1) pf_tiles += (b->q_len[r] + 63) / 64;
  // (x2 pages and + NF_MAX_NANO requests/tiles: split prefill requests duplicate their page list)
  const int64_t words = 3 * T + 2 * (int64_t)b->page_indptr[b->n_req] + 4 * ((int64_t)b->n_req + NF_MAX_NANO) * kh +
                        8 * (pf_tiles + NF_MAX_NANO) * qh + 3 * ((int64_t)b->n_req + NF_MAX_NANO) + 64;
  return (size_t)words;
}

void build_meta(const nf_model_cfg* c, const nf_batch* b, const std::vector<int>& order, const std::vector<int>& req_cuts,
                StepMeta* m, const std::vector<int32_t>* caller_row0, const std::vector<int32_t>* caller_req) {
  const int P = c->page_size;
  const int qh = c->n_q_heads / c->tp_size, kh = c->n_kv_heads / c->tp_size;
  const int n_req = b->n_req;
  int64_t T = batch_tokens(b);
  m->T = (int)T;
  m->n_req = n_req;
  const int64_t npg = b->page_indptr[n_req];
  m->off_pos = 0;
  m->off_slot = T;
  m->off_tok_src = 2 * T;
  m->off_pages = 3 * T;
  m->off_dec = m->off_pages + npg;
  // token rows in internal order
  std::vector<int64_t> caller_start(n_req + 1, 0);
  for (int r = 0; r < n_req; ++r) caller_start[r + 1] = caller_start[r] + b->q_len[r];
  std::vector<int> row_start(n_req);
  {
    int t = 0;
    for (int i = 0; i < n_req; ++i) {
      row_start[order[i]] = t;
      t += b->q_len[order[i]];
    }
  }
  std::vector<int32_t> head(3 * T + npg);
  for (int r = 0; r < n_req; ++r) {
    for (int i = 0; i < b->q_len[r]; ++i) {
      const int t = row_start[r] + i;
      const int pos = b->kv_prefix[r] + i;
      head[t] = pos;
      head[T + t] = b->page_ids[b->page_indptr[r] + pos / P] * P + pos % P;
      head[2 * T + t] = (int32_t)((caller_row0 ? (*caller_row0)[r] : caller_start[r]) + i);
    }
  }
  std::memcpy(head.data() + 3 * T, b->page_ids, npg * sizeof(int32_t));
  std::vector<DecodeItem> dec;
  std::vector<PrefillItem> pf;
  m->nanos.clear();
  for (size_t k = 0; k + 1 < req_cuts.size(); ++k) {
    NanoRange nr;
    nr.r0 = req_cuts[k];
    nr.r1 = req_cuts[k + 1];
    nr.t0 = nr.r0 < n_req ? row_start[order[nr.r0]] : (int)T;
    nr.t1 = nr.r1 < n_req ? row_start[order[nr.r1]] : (int)T;
    if (nr.r0 == nr.r1) nr.t1 = nr.t0;
    nr.dec_off = (int)dec.size();
    nr.pf_off = (int)pf.size();
    for (int i = nr.r0; i < nr.r1; ++i) {
      const int r = order[i];
      const int kvl = b->kv_prefix[r] + b->q_len[r];
      if (b->q_len[r] == 1) {
        for (int g = 0; g < kh; ++g) dec.push_back(DecodeItem{row_start[r], g, kvl, b->page_indptr[r]});
      } else {
        const int rows = prefill_rows(c->head_dim);
        for (int i0 = 0; i0 < b->q_len[r]; i0 += rows)
          for (int h = 0; h < qh; ++h)
            pf.push_back(PrefillItem{row_start[r] + i0, std::min(rows, b->q_len[r] - i0), b->kv_prefix[r] + i0, h, kvl,
                                     b->page_indptr[r], 0, 0});
      }
    }
    nr.dec_n = (int)dec.size() - nr.dec_off;
    nr.pf_n = (int)pf.size() - nr.pf_off;
    nr.dec_rows_off = m->nanos.empty() ? 0 : m->nanos.back().dec_rows_off;
    if (!m->nanos.empty())
      for (int q = m->nanos.back().dec_off; q < m->nanos.back().dec_off + m->nanos.back().dec_n; ++q)
        nr.dec_rows_off += (dec[q].kv_len + P - 1) / P;
    // longest first: static round-robin over warps/CTAs is then LPT-like
    std::stable_sort(dec.begin() + nr.dec_off, dec.end(),
                     [](const DecodeItem& x, const DecodeItem& y) { return x.kv_len > y.kv_len; });
    {
      // (opt-in, NF_DEC_CS_FRAC = f) the shortest items holding a fraction f of the nano-batch's
      // decode KV run on the compute partition in OVERLAP plans, to balance the two partitions
      static double cs_frac = -1.0;
      if (cs_frac < 0.0) {
        const char* e = getenv("NF_DEC_CS_FRAC");
        cs_frac = e ? std::max(0.0, std::min(0.9, atof(e))) : 0.0;
      }
      if (cs_frac > 0.0 && nr.dec_n > 0) {
        int64_t tot = 0, acc = 0;
        for (int q = nr.dec_off; q < nr.dec_off + nr.dec_n; ++q) tot += dec[q].kv_len;
        int n = 0;
        for (int q = nr.dec_off + nr.dec_n - 1; q >= nr.dec_off; --q) {
          if ((double)(acc + dec[q].kv_len) > cs_frac * (double)tot) break;
          acc += dec[q].kv_len;
          ++n;
        }
        nr.dec_cs_n = std::min(n, nr.dec_n - 1);
      }
    }
    std::stable_sort(pf.begin() + nr.pf_off, pf.end(),
                     [](const PrefillItem& x, const PrefillItem& y) { return x.pos0 + x.n > y.pos0 + y.n; });
    m->nanos.push_back(nr);
  }
  m->off_pf = m->off_dec + dec.size() * 4;
  m->off_emit_row = m->off_pf + pf.size() * 8;
  std::vector<int32_t> erow, ereq;
  for (int i = 0; i < n_req; ++i) {
    const int r = order[i];
    if (b->emit == nullptr || b->emit[r]) {
      erow.push_back(row_start[r] + b->q_len[r] - 1);
      ereq.push_back(caller_req ? (*caller_req)[r] : r);
    }
  }
  m->n_emit = (int)erow.size();
  m->off_emit_req = m->off_emit_row + erow.size();
  m->off_emit_sorted = m->off_emit_req + ereq.size();
  std::vector<int32_t> esort(erow.size());
  {
    std::vector<int> ix(erow.size());
    std::iota(ix.begin(), ix.end(), 0);
    std::stable_sort(ix.begin(), ix.end(), [&](int a, int b2) { return ereq[a] < ereq[b2]; });
    for (size_t i = 0; i < ix.size(); ++i) esort[i] = erow[ix[i]];
  }
  m->buf.resize(m->off_emit_sorted + esort.size());
  std::memcpy(m->buf.data() + m->off_emit_sorted, esort.data(), esort.size() * 4);
  std::memcpy(m->buf.data(), head.data(), head.size() * 4);
  std::memcpy(m->buf.data() + m->off_dec, dec.data(), dec.size() * sizeof(DecodeItem));
  std::memcpy(m->buf.data() + m->off_pf, pf.data(), pf.size() * sizeof(PrefillItem));
  std::memcpy(m->buf.data() + m->off_emit_row, erow.data(), erow.size() * 4);
  std::memcpy(m->buf.data() + m->off_emit_req, ereq.data(), ereq.size() * 4);
}

Workspace carve_workspace(const nf_model_cfg* c, const nf_batch* b, void* base) {
  const int64_t T = batch_tokens(b);
  const int N = c->tp_size;
  const int64_t qd = (int64_t)c->n_q_heads / N * c->head_dim, D = c->d_model, F = c->d_ffn / N;
  const int64_t NP = D / GEMM_NORM_COLS;
  const int64_t VT = (c->vocab / N + GEMM_BN - 1) / GEMM_BN;
  const int64_t R = b->n_req;
  Workspace w{};
  size_t off = 0;
  char* p = static_cast<char*>(base);
  auto take = [&](size_t bytes) -> void* {
    void* r = p ? p + off : nullptr;
    off = align_up(off + bytes, 256);
    return r;
  };
  w.meta = (int32_t*)take(meta_words_bound(c, b) * 4);
  w.q = (__nv_bfloat16*)take(T * qd * 2);
  w.o = (__nv_bfloat16*)take(T * qd * 2);
  w.o_full = N > 1 ? (__nv_bfloat16*)take(T * (int64_t)c->n_q_heads * c->head_dim * 2) : nullptr;
  w.h1 = (__nv_bfloat16*)take(T * D * 2);
  w.m = (__nv_bfloat16*)take(T * F * 2);
  w.xa = (__nv_bfloat16*)take(T * D * 2);
  w.xb = (__nv_bfloat16*)take(T * D * 2);
  w.part_a = (float*)take(NP * T * 4);
  w.part_b = (float*)take(NP * T * 4);
  w.part_h1 = (float*)take(NP * T * 4);
  w.lm_rows = (__nv_bfloat16*)take(R * D * 2);
  w.lm_part = (float*)take(R * 4);
  w.am_val = (float*)take(VT * R * 4);
  w.am_idx = (int*)take(VT * R * 4);
  w.red = N > 1 ? (float*)take(T * D * 4) : nullptr;
  const int64_t qd_full = (int64_t)c->n_q_heads * c->head_dim;
  w.ag = N > 1 ? (__nv_bfloat16*)take(T * qd_full * 2) : nullptr;
  w.ag2 = N > 1 ? (__nv_bfloat16*)take(T * D * 2) : nullptr;
  w.am_pair = N > 1 ? (float*)take(R * 8) : nullptr;
  w.am_pair_all = N > 1 ? (float*)take(R * 8 * N) : nullptr;
  w.ocat = N > 1 ? (__nv_bfloat16*)take(T * qd_full * 2) : nullptr;
  w.hcol = N > 1 ? (__nv_bfloat16*)take(T * (D / N) * 2) : nullptr;
  // stream-K / split-K partial slots: max(148 CTAs, tiles of the largest non-SiLU GEMM)
  const int64_t qkv_n = (int64_t)(c->n_q_heads + 2 * c->n_kv_heads) / N * c->head_dim;
  w.sk_slots = (int)std::max<int64_t>(148, ((T + GEMM_BM - 1) / GEMM_BM) * ((std::max(qkv_n, D) + 255) / 256));
  w.sk_part = (float*)take((size_t)w.sk_slots * GEMM_BM * GEMM_SK_LD * 4);
  w.sk_part2 = N > 1 ? (float*)take((size_t)w.sk_slots * GEMM_BM * GEMM_SK_LD * 4) : nullptr;
  const int64_t maxN = std::max<int64_t>({qkv_n, D, ((F + 127) / 128) * 256});
  w.sk_flag_n = (int)(((T + GEMM_BM - 1) / GEMM_BM) * ((maxN + 127) / 128) +
                      ((R + GEMM_BM - 1) / GEMM_BM) * VT + 64);
  if (c->n_experts > 0)  // grouped expert GEMMs: up to cap/128 m-tiles
    w.sk_flag_n = std::max<int>(w.sk_flag_n, (int)(moe_rows_cap(c, T) / GEMM_BM * ((maxN + 127) / 128) + 64));
  w.sk_flag = (int*)take((size_t)w.sk_flag_n * (N > 1 ? 2 : 1) * 4);
  w.sk_flag2 = (N > 1 && w.sk_flag) ? w.sk_flag + w.sk_flag_n : nullptr;
  w.sk_flag_total = w.sk_flag_n * (N > 1 ? 2 : 1);
  {
    int64_t dec_pages = 0;
    for (int r = 0; r < b->n_req; ++r)
      if (b->q_len[r] == 1) dec_pages += ((int64_t)b->kv_prefix[r] + 1 + c->page_size - 1) / c->page_size;
    w.dec_rows = (int*)take((size_t)(dec_pages * (c->n_kv_heads / N) + 64) * 4);
    w.dec_wstart = (int*)take((size_t)NF_MAX_NANO * 2049 * 4);
  }
  if (c->n_experts > 0) {
    const int64_t cap = moe_rows_cap(c, T), nk = T * c->top_k;
    w.mo_cap = cap;
    w.mo_ids = (int*)take(nk * 4);
    w.mo_wts = (float*)take(nk * 4);
    w.mo_inv = (float*)take(T * 4);
    w.mo_grp = (int*)take((2 * c->n_experts + 1) * 4);
    w.mo_dst = (int*)take(nk * 4);
    w.mo_rowtok = (int*)take(cap * 4);
    w.mo_roww = (float*)take(cap * 4);
    w.mo_rowinv = (float*)take(cap * 4);
    w.mo_x = (__nv_bfloat16*)take(cap * D * 2);
    w.mo_m = (__nv_bfloat16*)take(cap * F * 2);
    w.mo_y = (__nv_bfloat16*)take(cap * D * 2);
    w.mo_cta = (int*)take(moe_group_ints(T, c->n_experts) * 4);
  }
  w.total = off;
  return w;
}

}  // namespace nf

using namespace nf;

extern "C" {

const char* nf_last_error(void) { return g_err.c_str(); }
int32_t nf_abi_version(void) { return NF_ABI_VERSION; }

nf_status nf_batch_metadata(const nf_model_cfg* cfg, const nf_batch* b, int32_t* pos_out, int32_t* slot_out) {
  NF_TRY(validate_cfg(cfg));
  NF_TRY(validate_batch(cfg, b));
  if (!pos_out || !slot_out) return set_error(NF_EINVAL, "output arrays are NULL");
  std::vector<int> order(b->n_req);
  std::iota(order.begin(), order.end(), 0);
  StepMeta m;
  build_meta(cfg, b, order, {0, b->n_req}, &m);
  std::memcpy(pos_out, m.buf.data() + m.off_pos, m.T * 4);
  std::memcpy(slot_out, m.buf.data() + m.off_slot, m.T * 4);
  return NF_OK;
}

nf_status nf_snap_cuts(const nf_batch* b, int32_t n_nano, const int32_t* share, int32_t* req_cuts_out) {
  NF_TRY(validate_batch(nullptr, b));
  if (n_nano < 1 || n_nano > NF_MAX_NANO || !share || !req_cuts_out) return set_error(NF_EINVAL, "bad n_nano/share");
  int64_t tot = 0;
  for (int k = 0; k < n_nano; ++k) {
    if (share[k] < 0) return set_error(NF_EINVAL, "negative share");
    tot += share[k];
  }
  if (tot <= 0) return set_error(NF_EINVAL, "shares sum to zero");
  std::vector<int64_t> bound(b->n_req + 1, 0);
  for (int r = 0; r < b->n_req; ++r) bound[r + 1] = bound[r] + b->q_len[r];
  auto cuts = snap_cuts_impl(bound, n_nano, share);
  for (int k = 0; k <= n_nano; ++k) req_cuts_out[k] = cuts[k];
  return NF_OK;
}

nf_status nf_workspace_size(const nf_model_cfg* cfg, const nf_batch* b, size_t* bytes) {
  NF_TRY(validate_cfg(cfg));
  NF_TRY(validate_batch(cfg, b));
  if (!bytes) return set_error(NF_EINVAL, "bytes is NULL");
  *bytes = carve_workspace(cfg, b, nullptr).total;
  return NF_OK;
}

// ------------------------------------------------------------------ packing
nf_status nf_packed_layer_bytes(const nf_model_cfg* c, size_t out[6]) {
  NF_TRY(validate_cfg(c));
  if (!out) return set_error(NF_EINVAL, "out is NULL");
  const int N = c->tp_size;
  const size_t D = c->d_model, hd = c->head_dim, qh = c->n_q_heads / N, kh = c->n_kv_heads / N;
  const size_t F = c->d_ffn / N, E = c->n_experts > 0 ? c->n_experts : 1;
  out[0] = (qh + 2 * kh) * hd * D * 2;
  out[1] = N == 1 ? D * c->n_q_heads * hd * 2 : (D / N) * c->n_q_heads * hd * 2;
  out[2] = N == 1 ? 0 : D * qh * hd * 2;
  out[3] = E * ((F + 127) / 128) * 256 * D * 2;
  out[4] = E * D * F * 2;
  out[5] = c->n_experts > 0 ? (size_t)c->n_experts * D * 4 : 0;
  return NF_OK;
}

nf_status nf_pack_layer(const nf_model_cfg* c, const nf_layer_weights* s, const nf_packed_layer* d, void* stream) {
  NF_TRY(validate_cfg(c));
  if (!s || !d) return set_error(NF_EINVAL, "NULL weights");
  const int N = c->tp_size;
  if (!s->attn_norm || !s->w_q || !s->w_k || !s->w_v || !s->ffn_norm || !s->w_gate || !s->w_up || !s->w_down)
    return set_error(NF_EINVAL, "NULL source weight");
  if (N == 1 && !s->w_o) return set_error(NF_EINVAL, "w_o required at tp_size 1");
  if (N > 1 && (!s->w_o_col || !s->w_o_row)) return set_error(NF_EINVAL, "w_o_col and w_o_row required at tp_size > 1");
  if (!d->w_qkv || !d->w_o || !d->w_gate_up || !d->w_down || (N > 1 && !d->w_o_row))
    return set_error(NF_EINVAL, "NULL destination buffer");
  cudaStream_t st = (cudaStream_t)stream;
  using B = __nv_bfloat16;
  const int64_t D = c->d_model, hd = c->head_dim, qh = c->n_q_heads / N, kh = c->n_kv_heads / N, F = c->d_ffn / N;
  B* qkv = (B*)d->w_qkv;
  NF_CUDA(launch_scale_cols((const B*)s->w_q, (const B*)s->attn_norm, qh * hd, (int)D, qkv, st));
  NF_CUDA(launch_scale_cols((const B*)s->w_k, (const B*)s->attn_norm, kh * hd, (int)D, qkv + qh * hd * D, st));
  NF_CUDA(launch_scale_cols((const B*)s->w_v, (const B*)s->attn_norm, kh * hd, (int)D, qkv + (qh + kh) * hd * D, st));
  if (N == 1) {
    NF_CUDA(cudaMemcpyAsync(d->w_o, s->w_o, (size_t)D * c->n_q_heads * hd * 2, cudaMemcpyDeviceToDevice, st));
  } else {
    NF_CUDA(cudaMemcpyAsync(d->w_o, s->w_o_col, (size_t)(D / N) * c->n_q_heads * hd * 2, cudaMemcpyDeviceToDevice, st));
    NF_CUDA(cudaMemcpyAsync(d->w_o_row, s->w_o_row, (size_t)D * qh * hd * 2, cudaMemcpyDeviceToDevice, st));
  }
  const int64_t E = c->n_experts > 0 ? c->n_experts : 1, Ngu = ((F + 127) / 128) * 256;
  if (c->n_experts > 0) {
    if (!s->w_router || !d->w_router) return set_error(NF_EINVAL, "MoE layer needs w_router (source and packed)");
    NF_CUDA(launch_pack_router((const B*)s->w_router, (const B*)s->ffn_norm, (int)E, (int)D, (float*)d->w_router, st));
  }
  for (int64_t e = 0; e < E; ++e)
    NF_CUDA(launch_pack_gate_up((const B*)s->w_gate + e * F * D, (const B*)s->w_up + e * F * D, (const B*)s->ffn_norm,
                                (int)F, (int)D, (B*)d->w_gate_up + e * Ngu * D, st));
  NF_CUDA(cudaMemcpyAsync(d->w_down, s->w_down, (size_t)E * D * F * 2, cudaMemcpyDeviceToDevice, st));
  return NF_OK;
}

nf_status nf_pack_lm_head(const nf_model_cfg* c, const void* lm_head, const void* final_norm, void* dst, void* stream) {
  NF_TRY(validate_cfg(c));
  if (!lm_head || !final_norm || !dst) return set_error(NF_EINVAL, "NULL pointer");
  NF_CUDA(launch_scale_cols((const __nv_bfloat16*)lm_head, (const __nv_bfloat16*)final_norm, c->vocab / c->tp_size,
                            c->d_model, (__nv_bfloat16*)dst, (cudaStream_t)stream));
  return NF_OK;
}

// ------------------------------------------------------------------ plans
nf_status nf_plan_create_explicit(const nf_model_cfg* cfg, const nf_plan_spec* spec, nf_plan** out) {
  NF_TRY(validate_cfg(cfg));
  if (!spec || !out) return set_error(NF_EINVAL, "NULL spec/out");
  if (spec->mode < NF_SEQUENTIAL || spec->mode > NF_OVERLAP) return set_error(NF_EINVAL, "bad mode %d", spec->mode);
  if (spec->n_nano < 1 || spec->n_nano > NF_MAX_NANO) return set_error(NF_EINVAL, "n_nano %d out of range", spec->n_nano);
  int64_t tot = 0;
  for (int k = 0; k < spec->n_nano; ++k) {
    if (spec->share[k] <= 0) return set_error(NF_EINVAL, "share[%d] must be > 0", k);
    tot += spec->share[k];
  }
  for (int o = 0; o < NF_OP_COUNT; ++o)
    if (spec->sm[o] < 1 || spec->sm[o] > 1024) return set_error(NF_EINVAL, "sm[%d] = %d out of range", o, spec->sm[o]);
  if (spec->balance < 0 || spec->balance > 2) return set_error(NF_EINVAL, "balance must be 0, 1 or 2");
  if (spec->graph < 0 || spec->graph > 1) return set_error(NF_EINVAL, "graph must be 0 or 1");
  const int nd = spec->n_dense > 0 ? spec->n_dense : spec->n_nano;
  if (spec->n_dense < 0 || nd > spec->n_nano || spec->n_nano % nd)
    return set_error(NF_EINVAL, "n_dense %d must divide n_nano %d", spec->n_dense, spec->n_nano);
  if (cfg->tp_size == 1 && nd != spec->n_nano && spec->mode != NF_SEQUENTIAL)
    return set_error(NF_EINVAL, "n_dense != n_nano needs tp_size > 1");
  nf_plan* p = new (std::nothrow) nf_plan();
  if (!p) return set_error(NF_ENOMEM, "plan allocation failed");
  p->cfg = *cfg;
  p->spec = *spec;
  p->spec.n_dense = nd;
  if (spec->mode == NF_SEQUENTIAL) {
    p->spec.n_nano = 1;
    p->spec.n_dense = 1;
    p->spec.share[0] = 1;
  }
  *out = p;
  return NF_OK;
}

nf_status nf_plan_get_spec(const nf_plan* plan, nf_plan_spec* out) {
  if (!plan || !out) return set_error(NF_EINVAL, "NULL plan/out");
  *out = plan->spec;
  return NF_OK;
}

nf_status nf_plan_export_csv(const nf_plan* plan, char* buf, size_t cap, size_t* len) {
  if (!plan || !len) return set_error(NF_EINVAL, "NULL plan/len");
  *len = plan->csv.size();
  if (buf && cap > 0) {
    const size_t n = std::min(cap - 1, plan->csv.size());
    std::memcpy(buf, plan->csv.data(), n);
    buf[n] = 0;
  }
  return NF_OK;
}

uint64_t nf_plan_hash(const nf_plan* p) {
  if (!p) return 0;
  // FNV-1a over the model config and the plan spec (the executor's launch decisions);
  // ranks of one TP group must agree on it (collective issue order)
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](const void* d, size_t n) {
    const unsigned char* b = static_cast<const unsigned char*>(d);
    for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
  };
  nf_model_cfg c = p->cfg;
  c.tp_rank = 0;  // the rank differs by design
  mix(&c, sizeof(c));
  mix(&p->spec, sizeof(p->spec));
  return h;
}

const char* nf_plan_runtime_note(const nf_plan* p) {
  if (!p) return "";
  nf_plan* q = const_cast<nf_plan*>(p);
  q->note = q->green_note + (q->spec.graph ? "; CUDA graph: " + q->graph_note : std::string());
  return q->note.c_str();
}

void nf_plan_destroy(nf_plan* p) {
  if (!p) return;
  if (p->mem_stream) cudaStreamDestroy(p->mem_stream);
  for (int k = 0; k < NF_MAX_NANO; ++k) {
    if (p->ev_kqv[k]) cudaEventDestroy(p->ev_kqv[k]);
    if (p->ev_att[k]) cudaEventDestroy(p->ev_att[k]);
  }
  if (p->ev_join) cudaEventDestroy(p->ev_join);
  if (p->net_stream) cudaStreamDestroy(p->net_stream);
  if (p->cap_stream) cudaStreamDestroy(p->cap_stream);
  if (p->ev_c2n) cudaEventDestroy(p->ev_c2n);
  if (p->ev_n2c) cudaEventDestroy(p->ev_n2c);
  for (int k = 0; k < NF_MAX_NANO; ++k)
    for (cudaEvent_t e : {p->ev_pre[k], p->ev_o[k], p->ev_aro[k], p->ev_d[k], p->ev_ard[k]})
      if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : {p->ev_agattn, p->ev_ago, p->ev_join_n, p->ev_fork, p->ev_join_c, p->ev_join_m, p->ev_join_m2, p->ev_fork2,
                        p->ev_join_c2})
    if (e) cudaEventDestroy(e);
  if (p->cs2) cudaStreamDestroy(p->cs2);
  for (auto& g : p->graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  for (int i = 0; i < 2; ++i) {
    if (p->ev_upload[i]) cudaEventDestroy(p->ev_upload[i]);
    if (p->pinned[i]) cudaFreeHost(p->pinned[i]);
  }
  delete p;
}

}  // extern "C"

// ------------------------------------------------------------------ executor
namespace nf {

namespace {

nf_status ensure_runtime(nf_plan* p) {
  if (p->mem_stream) return NF_OK;
  NF_CUDA(cudaGetDevice(&p->device));
  int lo = 0, hi = 0;
  NF_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  // attention stream at higher priority: its CTAs are admitted first when both are pending
  NF_CUDA(cudaStreamCreateWithPriority(&p->mem_stream, cudaStreamNonBlocking, hi));
  for (int k = 0; k < NF_MAX_NANO; ++k) {
    NF_CUDA(cudaEventCreateWithFlags(&p->ev_kqv[k], cudaEventDisableTiming));
    NF_CUDA(cudaEventCreateWithFlags(&p->ev_att[k], cudaEventDisableTiming));
  }
  NF_CUDA(cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming));
  NF_CUDA(cudaStreamCreateWithPriority(&p->net_stream, cudaStreamNonBlocking, hi));
  NF_CUDA(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming));
  NF_CUDA(cudaEventCreateWithFlags(&p->ev_join_c, cudaEventDisableTiming));
  NF_CUDA(cudaEventCreateWithFlags(&p->ev_join_m, cudaEventDisableTiming));
  NF_CUDA(cudaEventCreateWithFlags(&p->ev_join_m2, cudaEventDisableTiming));
  NF_CUDA(cudaEventCreateWithFlags(&p->ev_c2n, cudaEventDisableTiming));
  NF_CUDA(cudaEventCreateWithFlags(&p->ev_n2c, cudaEventDisableTiming));
  for (int k = 0; k < NF_MAX_NANO; ++k)
    for (cudaEvent_t* e : {&p->ev_pre[k], &p->ev_o[k], &p->ev_aro[k], &p->ev_d[k], &p->ev_ard[k]})
      NF_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  for (cudaEvent_t* e : {&p->ev_agattn, &p->ev_ago, &p->ev_join_n, &p->ev_fork2, &p->ev_join_c2})
    NF_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  NF_CUDA(cudaStreamCreateWithPriority(&p->cs2, cudaStreamNonBlocking, lo));
  for (int i = 0; i < 2; ++i) NF_CUDA(cudaEventCreateWithFlags(&p->ev_upload[i], cudaEventDisableTiming));
  return NF_OK;
}

// Copy the step metadata into the workspace through a double-buffered pinned staging buffer.
nf_status upload_meta(nf_plan* p, const StepMeta& m, int32_t* dev, cudaStream_t st) {
  const size_t bytes = m.buf.size() * 4;
  const int i = p->upload_idx;
  p->upload_idx ^= 1;
  NF_CUDA(cudaEventSynchronize(p->ev_upload[i]));
  if (p->pinned_cap[i] < bytes) {
    if (p->pinned[i]) NF_CUDA(cudaFreeHost(p->pinned[i]));
    const size_t cap = bytes * 2 + 4096;
    NF_CUDA(cudaHostAlloc(&p->pinned[i], cap, cudaHostAllocDefault));
    p->pinned_cap[i] = cap;
  }
  std::memcpy(p->pinned[i], m.buf.data(), bytes);
  NF_CUDA(cudaMemcpyAsync(dev, p->pinned[i], bytes, cudaMemcpyHostToDevice, st));
  NF_CUDA(cudaEventRecord(p->ev_upload[i], st));
  return NF_OK;
}

// Internal request order and nano-batch cuts for this plan and batch.
// Internal view of a caller batch in which prefill requests may be split into
// consecutive parts living in successive nano-batches (reading A-10c): part j
// keeps the request's page list, starts at kv_prefix + (tokens of parts < j),
// and only the last part samples.  Equivalent to the unsplit request by T7
// (chunked prefill == whole prefill): an earlier part's K/V are appended by an
// earlier nano-batch's KQV, which precedes the later parts on the compute stream.
struct BatchView {
  std::vector<int32_t> q_len, kv_prefix, page_indptr, page_ids, emit, caller_req, caller_row0;
  nf_batch b{};
  void finish() {
    b.n_req = (int32_t)q_len.size();
    b.q_len = q_len.data();
    b.kv_prefix = kv_prefix.data();
    b.page_indptr = page_indptr.data();
    b.page_ids = page_ids.data();
    b.emit = emit.data();
  }
};

// balance == 2: every nano-batch gets exactly its token share (so GEMM tile
// counts split evenly) and decode requests are assigned longest-context first
// to the nano-batch with the least decode KV that still has token room; the
// prefill requests (largest first) then fill the remaining room in nano-batch
// order, split across nano-batches where they do not fit.
void split_view(const nf_batch* b, int nn, const int32_t* share, BatchView* v, std::vector<int>* order,
                std::vector<int>* cuts) {
  const int n_req = b->n_req;
  const int64_t T = batch_tokens(b);
  int64_t tot = 0;
  for (int k = 0; k < nn; ++k) tot += share[k];
  std::vector<int64_t> cap(nn);
  int64_t acc = 0;
  for (int k = 0; k < nn; ++k) {
    const int64_t next = (k + 1 == nn) ? T : (T * (acc + share[k])) / tot;
    cap[k] = next - (T * acc) / tot;
    acc += share[k];
  }
  std::vector<int64_t> caller_start(n_req + 1, 0);
  for (int r = 0; r < n_req; ++r) caller_start[r + 1] = caller_start[r] + b->q_len[r];
  std::vector<int> pre, dec;
  for (int r = 0; r < n_req; ++r) (b->q_len[r] > 1 ? pre : dec).push_back(r);
  std::stable_sort(dec.begin(), dec.end(), [&](int x, int y) { return b->kv_prefix[x] > b->kv_prefix[y]; });
  std::stable_sort(pre.begin(), pre.end(), [&](int x, int y) { return b->q_len[x] > b->q_len[y]; });
  struct Part { int r, off, len; };
  std::vector<std::vector<Part>> grp(nn);
  std::vector<double> kv(nn, 0.0);
  for (int r : dec) {
    int best = -1;
    for (int k = 0; k < nn; ++k)
      if (cap[k] > 0 && (best < 0 || kv[k] < kv[best])) best = k;
    if (best < 0) best = nn - 1;
    grp[best].push_back({r, 0, 1});
    cap[best] -= 1;
    kv[best] += b->kv_prefix[r] + 1;
  }
  int k = 0;
  for (int r : pre) {
    int off = 0;
    while (off < b->q_len[r]) {
      while (k < nn - 1 && cap[k] <= 0) ++k;
      const int len = (int)std::min<int64_t>(b->q_len[r] - off, k == nn - 1 ? INT32_MAX : cap[k]);
      grp[k].push_back({r, off, len});
      cap[k] -= len;
      off += len;
    }
  }
  order->clear();
  cuts->assign(1, 0);
  for (int kk = 0; kk < nn; ++kk) {
    std::stable_sort(grp[kk].begin(), grp[kk].end(), [](const Part& x, const Part& y) { return x.r < y.r; });
    for (const Part& pt : grp[kk]) {
      const int r = pt.r;
      const int idx = (int)v->q_len.size();
      v->q_len.push_back(pt.len);
      v->kv_prefix.push_back(b->kv_prefix[r] + pt.off);
      v->page_indptr.push_back((int32_t)v->page_ids.size());
      for (int i = b->page_indptr[r]; i < b->page_indptr[r + 1]; ++i) v->page_ids.push_back(b->page_ids[i]);
      const bool last = pt.off + pt.len == b->q_len[r];
      v->emit.push_back(last && (b->emit == nullptr || b->emit[r]) ? 1 : 0);
      v->caller_req.push_back(r);
      v->caller_row0.push_back((int32_t)(caller_start[r] + pt.off));
      order->push_back(idx);
    }
    cuts->push_back((int)order->size());
  }
  v->page_indptr.push_back((int32_t)v->page_ids.size());
  v->finish();
}

// Internal request order and nano-batch cuts for this plan and batch.  With
// balance == 2 (model step) the batch is re-expressed as a split view.
void plan_order(const nf_plan* p, const nf_batch* b, bool allow_balance, std::vector<int>* order, std::vector<int>* cuts,
                BatchView* view = nullptr, bool* use_view = nullptr) {
  const int n_req = b->n_req;
  const int nn = p->spec.n_nano;
  if (use_view) *use_view = false;
  order->resize(n_req);
  std::iota(order->begin(), order->end(), 0);
  if (nn == 1) {
    *cuts = {0, n_req};
    return;
  }
  if (!(allow_balance && p->spec.balance)) {
    std::vector<int64_t> bound(n_req + 1, 0);
    for (int r = 0; r < n_req; ++r) bound[r + 1] = bound[r] + b->q_len[r];
    *cuts = snap_cuts_impl(bound, nn, p->spec.share);
    return;
  }
  if (p->spec.balance == 2 && view) {
    split_view(b, nn, p->spec.share, view, order, cuts);
    if (use_view) *use_view = true;
    return;
  }
  std::vector<std::vector<int>> grp;
  balance_requests(b, nn, p->spec.share, &grp);
  order->clear();
  cuts->assign(1, 0);
  for (int k = 0; k < nn; ++k) {
    for (int r : grp[k]) order->push_back(r);
    cuts->push_back((int)order->size());
  }
}

struct LayerCtx {
  const nf_plan* p;
  const nf_model_cfg* c;
  const StepMeta* m;
  const Workspace* w;
  const int32_t* meta_dev;
  CUtensorMap pool_map;
  CUtensorMap page_map;
  cudaStream_t cs, ms;  // compute / memory streams
  cudaStream_t ns;      // network stream (TP collectives; == cs outside OVERLAP)
  cudaStream_t cs2 = nullptr;  // TP OVERLAP: compute stream of the second dense nano-batch (null: cs)
  bool dec_on_cs = false;      // no memory partition: decode attention on the (group's) compute stream
  bool dec_side = false;       // no memory partition: decode on side streams of the compute partition
  cudaStream_t ms2 = nullptr;  // dec_side: the second dense group's decode stream
  mutable bool rows_built[NF_MAX_NANO] = {};  // decode row streams written this step (ROWS loader)
  nf_comm* comm;
  int cap_dense = 0, cap_dec = 0;  // partition sizes when green contexts are active (0: whole GPU)
};

int clampsm(int v) { return std::max(1, std::min(v, num_sms())); }
int clamp_dense(const LayerCtx& L, int v) { return clampsm(L.cap_dense ? std::min(v, L.cap_dense) : v); }
int clamp_dec(const LayerCtx& L, int v) { return clampsm(L.cap_dec ? std::min(v, L.cap_dec) : v); }

// Decode kernel choice: the mma.sync kernel (8 independent warps per SM, one
// 4-D TMA box per page) is the default: it reaches the HBM roofline at ~80 SMs.
// The tcgen05 kernel (decode_tc.cu, one item in flight per CTA) is selectable
// with NF_DECODE_IMPL=tc for head_dim 128 / GQA <= 8 (not in co-located plans).
// Default: the stream kernel (decode_stream.cu) when its row streams fit; NF_DECODE_IMPL=fused
// selects the item-walking kernel (attention.cu), =tc / =ws the tcgen05 / warp-specialised ones.
int decode_impl_env() {  // read per launch (tests switch it at run time)
  const char* e = getenv("NF_DECODE_IMPL");
  if (!e) return 0;
  const std::string v(e);
  return v == "tc" ? 1 : v == "ws" ? 2 : v == "fused" ? 3 : 0;
}
bool use_tc_decode(const nf_model_cfg* c, const nf_plan* p) {
  return decode_impl_env() == 1 && !p->spec.colocate && c->head_dim == 128 && c->n_q_heads / c->n_kv_heads <= 8;
}
// warp-specialised decode (decode_ws.cu): NF_DECODE_IMPL=ws, not in co-located plans
bool use_ws_decode(const nf_plan* p) { return decode_impl_env() == 2 && !p->spec.colocate; }
// row-stream loader of the default decode kernel: opt-in with NF_DEC_ROWS=1 (measured
// 9 % (8B) / 10 % (70B rank) slower per SM than the item-walking loader at 32 SMs,
// profiles/r2e_attn_rows_ab.log)
bool use_rows_decode() {
  const char* e = getenv("NF_DEC_ROWS");
  return e && e[0] == '1';
}

nf_status run_kqv(const LayerCtx& L, const NanoRange& nr, const __nv_bfloat16* x, const float* part, int nparts,
                  const nf_packed_layer* wt, void* pool) {
  const nf_model_cfg* c = L.c;
  const int N = c->tp_size;
  const int M = nr.t1 - nr.t0;
  if (M <= 0) return NF_OK;
  GemmArgs a{};
  a.epi = EPI_QKV;
  a.sk_part = L.w->sk_part;
  a.sk_slots = L.w->sk_slots;
  a.sk_flag = L.w->sk_flag;
  a.stages = L.p->spec.colocate ? 3 : 4;
  a.M = M;
  a.N = (c->n_q_heads + 2 * c->n_kv_heads) / N * c->head_dim;
  a.K = c->d_model;
  a.n_valid = a.N;
  a.norm_part = part + nr.t0;
  a.norm_nparts = nparts;
  a.norm_stride = L.m->T;
  a.inv_d = 1.f / c->d_model;
  a.eps = c->rms_eps;
  a.qh = c->n_q_heads / N;
  a.kh = c->n_kv_heads / N;
  a.hd = c->head_dim;
  a.page_size = c->page_size;
  a.log2_theta = (float)std::log2((double)c->rope_theta);
  a.tok_pos = L.meta_dev + L.m->off_pos + nr.t0;
  a.tok_slot = L.meta_dev + L.m->off_slot + nr.t0;
  a.q_out = L.w->q + (int64_t)nr.t0 * a.qh * a.hd;
  a.kv_pool = (__nv_bfloat16*)pool;
  ProfScope ps(NF_OP_KQV, L.cs);
  NF_CUDA(launch_gemm(x + (int64_t)nr.t0 * c->d_model, c->d_model, (const __nv_bfloat16*)wt->w_qkv, c->d_model, a,
                      clamp_dense(L, L.p->spec.sm[NF_OP_KQV]), L.cs));
  return NF_OK;
}

AttnArgs attn_args(const LayerCtx& L) {
  const nf_model_cfg* c = L.c;
  AttnArgs a{};
  a.q = L.w->q;
  a.o = L.w->o;
  a.page_ids = L.meta_dev + L.m->off_pages;
  a.qh = c->n_q_heads / c->tp_size;
  a.kh = c->n_kv_heads / c->tp_size;
  a.hd = c->head_dim;
  a.page_size = c->page_size;
  a.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)c->head_dim));
  a.dec_warps = L.p->spec.colocate ? 4 : 8;
  a.n_rows = L.m->T;
  return a;
}

// Prefill attention of one nano-batch: compute-bound, so it runs on the compute
// stream right after the nano-batch's KQV (reading A-11), within the GEMMs' SM
// budget; its small multi-CTA-per-SM grid must not spill onto the memory partition.
nf_status run_prefill(const LayerCtx& L, const NanoRange& nr, cudaStream_t st) {
  if (nr.pf_n <= 0) return NF_OK;
  const AttnArgs a = attn_args(L);
  const PrefillItem* pf = reinterpret_cast<const PrefillItem*>(L.meta_dev + L.m->off_pf) + nr.pf_off;
  ProfScope ps(NF_OP_PREFILL_ATTN, st);
  NF_CUDA(launch_prefill_attention(L.pool_map, a, pf, nr.pf_n, clamp_dense(L, L.p->spec.sm[NF_OP_PREFILL_ATTN]), st));
  return NF_OK;
}

// Decode attention of one nano-batch: HBM-bound, on the memory stream in OVERLAP mode.
// part 0: all decode items of the nano-batch; 1: all but the dec_cs_n shortest (memory
// partition); 2: the dec_cs_n shortest, on the compute partition (OVERLAP balance option)
nf_status run_decode(const LayerCtx& L, const NanoRange& nr, cudaStream_t st, int part = 0) {
  const int off = part == 2 ? nr.dec_n - nr.dec_cs_n : 0;
  const int n = part == 0 ? nr.dec_n : (part == 1 ? nr.dec_n - nr.dec_cs_n : nr.dec_cs_n);
  if (n <= 0) return NF_OK;
  const nf_model_cfg* c = L.c;
  AttnArgs a = attn_args(L);
  const DecodeItem* dec = reinterpret_cast<const DecodeItem*>(L.meta_dev + L.m->off_dec) + nr.dec_off + off;
  const int sms = part == 2     ? clamp_dense(L, L.p->spec.sm[NF_OP_KQV])
                  : (L.dec_on_cs || L.dec_side) ? clamp_dense(L, L.p->spec.sm[NF_OP_DECODE_ATTN])
                                : clamp_dec(L, L.p->spec.sm[NF_OP_DECODE_ATTN]);
  ProfScope ps(NF_OP_DECODE_ATTN, st);
  if (use_tc_decode(c, L.p)) {
    NF_CUDA(launch_decode_attention_tc(L.pool_map, a, dec, n, sms, st));
  } else if (use_ws_decode(L.p)) {
    NF_CUDA(launch_decode_attention_ws(L.page_map, a, dec, n, sms, st));
  } else if (part != 2 && decode_impl_env() == 0 && a.dec_warps != 4 && L.w->dec_rows && decode_stream_supported(a) &&
             decode_grid(n, sms, a.hd == 128 ? decode_stream_warps() : 12) * (a.hd == 128 ? decode_stream_warps() : 12) <=
                 2048) {
    // stream kernel: row streams of this nano-batch's launch geometry, written once per step
    // (every layer of a step has the same items, pages and grid)
    const int W = a.hd == 128 ? decode_stream_warps() : 12;
    const int k = (int)(&nr - &L.m->nanos[0]);
    const int grid = decode_grid(n, sms, W);
    int* rows = L.w->dec_rows + nr.dec_rows_off;
    int* wst = L.w->dec_wstart + k * 2049;
    if (k < 0 || k >= NF_MAX_NANO || !L.rows_built[k]) {
      NF_CUDA(launch_build_dec_rows(dec, n, grid, W, a.page_ids, a.kh, rows, wst, st));
      if (k >= 0 && k < NF_MAX_NANO) L.rows_built[k] = true;
    }
    a.dec_rows = rows;
    a.dec_wstart = wst;
    NF_CUDA(launch_decode_attention_stream(L.page_map, a, dec, n, sms, st));
  } else if (part != 2 && use_rows_decode() && a.dec_warps != 4 && L.w->dec_rows) {
    // row streams of this nano-batch's launch geometry, written once per step (every layer
    // of a step has the same items, pages and grid)
    const int k = (int)(&nr - &L.m->nanos[0]);
    const int W = decode_warps(c->head_dim, a.dec_warps);
    const int grid = decode_grid(n, sms, W);
    int* rows = L.w->dec_rows + nr.dec_rows_off;
    int* wst = L.w->dec_wstart + k * 2049;
    if (grid * W <= 2048) {
      if (k < 0 || k >= NF_MAX_NANO || !L.rows_built[k]) {
        NF_CUDA(launch_build_dec_rows(dec, n, grid, W, a.page_ids, a.kh, rows, wst, st));
        if (k >= 0 && k < NF_MAX_NANO) L.rows_built[k] = true;
      }
      a.dec_rows = rows;
      a.dec_wstart = wst;
    }
    NF_CUDA(launch_decode_attention(L.pool_map, L.page_map, a, dec, n, sms, st));
  } else
    NF_CUDA(launch_decode_attention(L.pool_map, L.page_map, a, dec, n, sms, st));
  return NF_OK;
}

nf_status run_attn(const LayerCtx& L, const NanoRange& nr, cudaStream_t st) {
  NF_TRY(run_prefill(L, nr, st));
  return run_decode(L, nr, st);
}

nf_status run_moe_ffn(const LayerCtx& L, const NanoRange& nr, const __nv_bfloat16* h1, const nf_packed_layer* wt,
                      const __nv_bfloat16* resid, __nv_bfloat16* out, float* part_out);

// O + residual, RMS(FFN) fold, Up/Gate + SiLU, Down + residual for one nano-batch (TP1).
nf_status run_dense_tail(const LayerCtx& L, const NanoRange& nr, const __nv_bfloat16* x, const nf_packed_layer* wt,
                         __nv_bfloat16* x_out, float* part_out) {
  const nf_model_cfg* c = L.c;
  const int M = nr.t1 - nr.t0;
  if (M <= 0) return NF_OK;
  const int64_t D = c->d_model, F = c->d_ffn, qd = (int64_t)c->n_q_heads * c->head_dim;
  const int T = L.m->T;
  const int NP = (int)(D / GEMM_NORM_COLS);
  // O projection + residual: h1 = x + o W_o^T, with sum-of-squares partials of h1
  GemmArgs a{};
  a.epi = EPI_RESID;
  a.sk_part = L.w->sk_part;
  a.sk_slots = L.w->sk_slots;
  a.sk_flag = L.w->sk_flag;
  a.stages = L.p->spec.colocate ? 3 : 4;
  a.M = M;
  a.N = (int)D;
  a.K = (int)qd;
  a.n_valid = (int)D;
  a.out = L.w->h1 + nr.t0 * D;
  a.ldo = D;
  a.resid = x + nr.t0 * D;
  a.ldr = D;
  a.sq_out = L.w->part_h1 + nr.t0;
  a.sq_stride = T;
  {
    ProfScope ps(NF_OP_O, L.cs);
    NF_CUDA(launch_gemm(L.w->o + nr.t0 * qd, qd, (const __nv_bfloat16*)wt->w_o, qd, a, clamp_dense(L, L.p->spec.sm[NF_OP_O]), L.cs));
  }
  if (c->n_experts > 0) return run_moe_ffn(L, nr, L.w->h1, wt, L.w->h1, x_out, part_out);
  // Up/Gate + SiLU(gate) * up, RMSNorm(h1) folded as a row scale
  GemmArgs u{};
  u.epi = EPI_SILU;
  u.sk_part = L.w->sk_part;
  u.sk_slots = L.w->sk_slots;
  u.sk_flag = L.w->sk_flag;
  u.stages = L.p->spec.colocate ? 3 : 4;
  u.M = M;
  u.N = (int)(((F + 127) / 128) * 256);
  u.K = (int)D;
  u.n_valid = (int)F;
  u.out = L.w->m + nr.t0 * F;
  u.ldo = F;
  u.norm_part = L.w->part_h1 + nr.t0;
  u.norm_nparts = NP;
  u.norm_stride = T;
  u.inv_d = 1.f / D;
  u.eps = c->rms_eps;
  {
    ProfScope ps(NF_OP_UG, L.cs);
    NF_CUDA(launch_gemm(L.w->h1 + nr.t0 * D, D, (const __nv_bfloat16*)wt->w_gate_up, D, u, clamp_dense(L, L.p->spec.sm[NF_OP_UG]),
                        L.cs));
  }
  // Down + residual: x_out = h1 + m W_d^T, partials of x_out for the next layer's norm
  GemmArgs d{};
  d.epi = EPI_RESID;
  d.sk_part = L.w->sk_part;
  d.sk_slots = L.w->sk_slots;
  d.sk_flag = L.w->sk_flag;
  d.stages = L.p->spec.colocate ? 3 : 4;
  d.M = M;
  d.N = (int)D;
  d.K = (int)F;
  d.n_valid = (int)D;
  d.out = x_out + nr.t0 * D;
  d.ldo = D;
  d.resid = L.w->h1 + nr.t0 * D;
  d.ldr = D;
  d.sq_out = part_out ? part_out + nr.t0 : nullptr;
  d.sq_stride = T;
  {
    ProfScope ps(NF_OP_DOWN, L.cs);
    NF_CUDA(launch_gemm(L.w->m + nr.t0 * F, F, (const __nv_bfloat16*)wt->w_down, F, d, clamp_dense(L, L.p->spec.sm[NF_OP_DOWN]),
                        L.cs));
  }
  return NF_OK;
}

// MoE FFN of one nano-batch (readings A-20..A-23): gating, grouping,
// grouped Up/Gate + SiLU (1/rms row scale), grouped Down (routing-weight row scale,
// bf16), weighted combine (fp32 sum).  resid != null: out = bf16(resid + sum) with RMS partials
// (TP1); resid == null: out = bf16(sum), this rank's partial for the AllReduce (TP>1).
// Routing buffers are reused by every nano-batch: all of it runs on the compute stream.
nf_status run_moe_ffn(const LayerCtx& L, const NanoRange& nr, const __nv_bfloat16* h1, const nf_packed_layer* wt,
                      const __nv_bfloat16* resid, __nv_bfloat16* out, float* part_out) {
  const nf_model_cfg* c = L.c;
  const Workspace* w = L.w;
  const int M = nr.t1 - nr.t0;
  if (M <= 0) return NF_OK;
  const int64_t D = c->d_model, Fl = c->d_ffn / c->tp_size;
  const int E = c->n_experts, k = c->top_k, T = L.m->T;
  const int cap = (int)moe_rows_cap(c, M);
  int* grp_off = w->mo_grp;
  int* grp_end = w->mo_grp + E + 1;
  {
    ProfScope ps(NF_PROF_MISC, L.cs);
    MoeGroupArgs g{};
    g.cta_cnt = w->mo_cta;
    g.cta_base = w->mo_cta + moe_group_ints(M, E) / 2;
    g.counter = w->sk_flag + (w->sk_flag_n - 1);  // zeroed with the step's flags, self-resetting
    g.grp_off = grp_off;
    g.grp_end = grp_end;
    g.row_tok = w->mo_rowtok;
    g.row_w = w->mo_roww;
    g.row_inv = w->mo_rowinv;
    g.tile = GEMM_BM;
    // routing of the nano-batch's rows at their row offset (the whole batch's routing stays
    // in the workspace after a layer: nf_moe_last_ids)
    NF_CUDA(launch_moe_route(h1 + nr.t0 * D, M, (int)D, (const float*)wt->w_router, E, k, c->rms_eps,
                             w->mo_ids + (int64_t)nr.t0 * k, w->mo_wts + (int64_t)nr.t0 * k, w->mo_inv + nr.t0, g,
                             L.cs));
    NF_CUDA(launch_moe_scatter(h1 + nr.t0 * D, M, (int)D, k, E, w->mo_ids + (int64_t)nr.t0 * k,
                               w->mo_wts + (int64_t)nr.t0 * k, w->mo_inv + nr.t0, g, w->mo_dst + (int64_t)nr.t0 * k,
                               w->mo_x, L.cs));
  }
  const int stages = L.p->spec.colocate ? 3 : 4;
  GemmArgs u{};
  u.epi = EPI_SILU;
  u.stages = stages;
  u.M = cap;
  u.N = (int)(((Fl + 127) / 128) * 256);
  u.K = (int)D;
  u.n_valid = (int)Fl;
  u.out = w->mo_m;
  u.ldo = Fl;
  u.row_scale = w->mo_rowinv;
  u.sk_part = w->sk_part;
  u.sk_slots = w->sk_slots;
  u.sk_flag = w->sk_flag;
  u.grp_off = grp_off;
  u.grp_end = grp_end;
  u.n_groups = E;
  {
    ProfScope ps(NF_OP_UG, L.cs);
    NF_CUDA(launch_gemm(w->mo_x, D, (const __nv_bfloat16*)wt->w_gate_up, D, u, clamp_dense(L, L.p->spec.sm[NF_OP_UG]),
                        L.cs));
  }
  GemmArgs d{};
  d.epi = EPI_STORE;  // y = bf16(weight * expert output); summed in fp32 by the combine
  d.stages = stages;
  d.M = cap;
  d.N = (int)D;
  d.K = (int)Fl;
  d.n_valid = (int)D;
  d.out = w->mo_y;
  d.ldo = D;
  d.row_scale = w->mo_roww;
  d.sk_part = w->sk_part;
  d.sk_slots = w->sk_slots;
  d.sk_flag = w->sk_flag;
  d.grp_off = grp_off;
  d.grp_end = grp_end;
  d.n_groups = E;
  {
    ProfScope ps(NF_OP_DOWN, L.cs);
    NF_CUDA(launch_gemm(w->mo_m, Fl, (const __nv_bfloat16*)wt->w_down, Fl, d, clamp_dense(L, L.p->spec.sm[NF_OP_DOWN]),
                        L.cs));
  }
  {
    ProfScope ps(NF_PROF_MISC, L.cs);
    NF_CUDA(launch_moe_combine(w->mo_y, w->mo_dst + (int64_t)nr.t0 * k, M, k, (int)D, resid ? resid + nr.t0 * D : nullptr, out + nr.t0 * D,
                               part_out ? part_out + nr.t0 : nullptr, T, nullptr, L.cs));
  }
  return NF_OK;
}

// Record `ev` on `from` and make `to` wait on it (no-op when both are the same stream).
nf_status edge(cudaEvent_t ev, cudaStream_t from, cudaStream_t to) {
  if (from == to) return NF_OK;
  NF_CUDA(cudaEventRecord(ev, from));
  NF_CUDA(cudaStreamWaitEvent(to, ev, 0));
  return NF_OK;
}

// ------------------------------------------------------------------ tensor-parallel pipeline
// PAPER.md:183, :547-548 and SURVEY.md §8 (a6-a10 DAG).  The n_nano attention
// nano-batches (KQV, decode/prefill attention) are grouped into n_dense contiguous
// dense nano-batches ("groups").  Group 0 (H1) runs column-parallel O:
//   AG(attention out) -> O_col (+ x columns) -> AG -> h1,
// the other groups (H2) row-parallel O:
//   O_row partial -> AR -> h1 = x + sum.
// Every group then runs column Up/Gate + SiLU and a row-parallel Down partial,
// AR, and x_out = h1 + sum (A-12b: the residual is added after the AllReduce in
// fp32 with one rounding; one RMS part per row).  Collectives run on the network
// stream ns; the compute stream cs waits only right before the op that reads a
// collective's output, so a group's AllGather / AllReduce is in flight while the
// compute stream runs the other group's GEMMs (O2 under AG_o1, UG1 under AR_o2,
// D2 under AR_d1, the next layer's KQV under AR_d2).  The host issue order of the
// collectives is the same on every rank (NCCL's ordering requirement).
struct Group {
  NanoRange nr;  // token rows / requests of the group (t0..t1, r0..r1)
  int k0, k1;    // its attention nano-batches
  bool col;
};

std::vector<Group> dense_groups(const nf_plan* p, const StepMeta& m) {
  const int nn = (int)m.nanos.size();
  int nd = p->spec.n_dense > 0 ? std::min(p->spec.n_dense, nn) : nn;
  if (nd < 1 || nn % nd) nd = nn;
  const int per = nn / nd;
  std::vector<Group> g(nd);
  for (int i = 0; i < nd; ++i) {
    g[i].k0 = i * per;
    g[i].k1 = (i + 1) * per;
    g[i].nr = m.nanos[g[i].k0];
    g[i].nr.r1 = m.nanos[g[i].k1 - 1].r1;
    g[i].nr.t1 = m.nanos[g[i].k1 - 1].t1;
    g[i].col = i == 0;
  }
  return g;
}

// TP OVERLAP: the dense nano-batches alternate between two compute streams on the compute
// partition (each with its own stream-K scratch), so a group whose next op waits on a
// collective or on decode attention does not hold back the other group's ready GEMMs:
// the hardware runs whichever is ready (the in-order single stream stalled on every wait).
LayerCtx group_ctx(const LayerCtx& L, int g, Workspace* wg) {
  LayerCtx c = L;
  if ((g & 1) && L.cs2) {
    *wg = *L.w;
    wg->sk_part = L.w->sk_part2;
    wg->sk_flag = L.w->sk_flag2;
    c.w = wg;
    c.cs = L.cs2;
  }
  if (L.dec_on_cs) c.ms = c.cs;
  else if ((g & 1) && L.ms2) c.ms = L.ms2;
  return c;
}

// Fused GEMM -> AllReduce sites (peer.cuh, NEXT-3): the O row-parallel projection of dense
// group g uses site g, its Down projection site NF_MAX_NANO + g.  The decision is a pure
// function of the communicator and the group's shape, so stages b/c/d agree on it.
// The owner reduce spins until the group's partials arrive, so it must never hold SMs that a
// kernel it (transitively) waits for needs: it runs either in stream order on the single
// compute stream (SEQUENTIAL / NANO_ONLY: ns == cs) or inside the OVERLAP plan's network
// green-context partition, whose SMs no GEMM uses.  An OVERLAP plan without a network
// partition keeps the plain AllReduce.
bool fused_site_ok(const LayerCtx& L, int M) {
  if (!comm_fused(L.comm) || M <= 0) return false;
  const bool streams_ok = L.ns == L.cs || (L.p->green_ns && L.ns == L.p->green_ns);
  const PeerGeom& g = comm_peer_geom(L.comm);
  const bool ok = streams_ok && M <= g.max_rows && g.cols == L.c->d_model;
  static const bool dbg = getenv("NF_PEER_DEBUG") != nullptr;
  if (dbg) {
    timespec ts;
    clock_gettime(CLOCK_REALTIME, &ts);
    fprintf(stderr, "[nf peer] rank %d M %d streams_ok %d -> %s at host %lld ms\n", comm_rank(L.comm), M,
            (int)streams_ok, ok ? "fused" : "plain", ((long long)ts.tv_sec * 1000 + ts.tv_nsec / 1000000) % 1000000);
  }
  return ok;
}
int site_of(bool down, int gi) { return (down ? NF_MAX_NANO : 0) + gi; }
void set_peer_args(GemmArgs* a, const LayerCtx& L, int site, int M) {
  const PeerGeom& g = comm_peer_geom(L.comm);
  a->epi = EPI_PEER;
  a->peer_bases = comm_peer_bases(L.comm);
  a->peer_site_off = g.site(site);
  a->peer_stage_off = g.stage_off;
  a->peer_flags_off = g.flags_off;
  a->peer_n = g.n;
  a->peer_rank = g.rank;
  a->peer_maxown = g.maxown;
  a->peer_mb = (M + PEER_BM - 1) / PEER_BM;
}
// Fused AllGather of the O column-parallel projection (group 0): its EPI_RESID epilogue
// writes the rank's slice into every rank's site-0 result region (site 0 = the O-row site
// of group 0, which the column group never uses) -- peer.cuh.
bool fused_ag_ok(const LayerCtx& L, int M) {
  return fused_site_ok(L, M) && (L.c->d_model / L.c->tp_size) % 64 == 0;
}
void set_peer_ag_args(GemmArgs* a, const LayerCtx& L, int M) {
  set_peer_args(a, L, 0, M);
  a->epi = EPI_RESID;
  a->peer_mode = 1;
  a->peer_result_off = comm_peer_geom(L.comm).result_off;
}
const __nv_bfloat16* peer_result(const LayerCtx& L, int site) {
  const PeerGeom& g = comm_peer_geom(L.comm);
  return reinterpret_cast<const __nv_bfloat16*>(comm_sym_local(L.comm) + g.site(site) + g.result_off);
}
// Owner-side reduce + all-gather of a site on the network stream: ~2 CTAs per SM of the
// plan's network budget (they are light: 128 threads, no shared memory)
nf_status run_peer_reduce(const LayerCtx& L, int site, int M) {
  comm_fused_site_barrier(L.comm);
  // (an emulated group runs every rank's reduce on the same GPU: 2 CTAs each, so the ranks' spinning
  // reduce CTAs never crowd out the GEMM CTAs they wait for)
  // (SEQUENTIAL / NANO_ONLY: the reduce follows the GEMM on the compute stream and has the GPU)
  const int ctas = comm_host_sync(L.comm) ? 2
                   : L.ns == L.cs       ? 2 * num_sms()
                                        : std::max(4, std::min(64, 4 * std::max(1, L.p->green_net_sms)));
  ProfScope ps(NF_OP_NET, L.ns);
  NF_CUDA(launch_peer_reduce(comm_peer_bases(L.comm), comm_peer_geom(L.comm), site, M, ctas,
                             comm_peer_timeout_ns(L.comm), L.ns));
  comm_count_fused(L.comm);
  return NF_OK;
}

int gemm_aslots_env() {  // read per launch (tests switch it at run time)
  const char* e = getenv("NF_GEMM_ASLOTS");
  return !(e && e[0] == '0');
}

// Front of a group: KQV of each of its attention nano-batches, decode attention on
// the memory stream as soon as that KQV lands, prefill attention on the compute stream.
nf_status tp_front(nf_plan* p, const LayerCtx& L, int gi, const Group& G, const __nv_bfloat16* x, const float* part,
                   int nparts, const nf_packed_layer* wt, void* pool) {
  for (int k = G.k0; k < G.k1; ++k) {
    const NanoRange& nr = L.m->nanos[k];
    NF_TRY(run_kqv(L, nr, x, part, nparts, wt, pool));
    if (L.ms != L.cs) {
      NF_TRY(edge(p->ev_kqv[k], L.cs, L.ms));
      NF_TRY(run_decode(L, nr, L.ms, 1));
      NF_CUDA(cudaEventRecord(p->ev_att[k], L.ms));
      NF_TRY(run_prefill(L, nr, L.cs));
      NF_TRY(run_decode(L, nr, L.cs, 2));
    } else {
      NF_TRY(run_attn(L, nr, L.cs));
    }
  }
  if (L.ns != L.cs) NF_CUDA(cudaEventRecord(p->ev_pre[gi], L.cs));
  return NF_OK;
}

// Make `st` wait for the decode attention of the group's nano-batches (memory stream).
nf_status wait_attention(nf_plan* p, const LayerCtx& L, const Group& G, cudaStream_t st) {
  if (L.ms == st) return NF_OK;
  for (int k = G.k0; k < G.k1; ++k) NF_CUDA(cudaStreamWaitEvent(st, p->ev_att[k], 0));
  return NF_OK;
}

// Stage A (column group): AllGather of the group's attention output rows (rank-major).
nf_status tp_stage_a(nf_plan* p, const LayerCtx& L, int gi, const Group& G) {
  if (!G.col) return NF_OK;
  const int M = G.nr.t1 - G.nr.t0;
  if (M <= 0) return NF_OK;
  const int64_t qd = (int64_t)L.c->n_q_heads / L.c->tp_size * L.c->head_dim;
  NF_TRY(wait_attention(p, L, G, L.ns));
  if (L.ns != L.cs) NF_CUDA(cudaStreamWaitEvent(L.ns, p->ev_pre[gi], 0));
  {
    ProfScope ps(NF_OP_NET, L.ns);
    NF_TRY(comm_all_gather(L.comm, L.w->o + G.nr.t0 * qd, L.w->ag, (size_t)M * qd, L.ns));
  }
  if (L.ns != L.cs) NF_CUDA(cudaEventRecord(p->ev_agattn, L.ns));
  return NF_OK;
}

// Stage B: O projection and its collective.
nf_status tp_stage_b(nf_plan* p, const LayerCtx& L, int gi, const Group& G, const __nv_bfloat16* x,
                     const nf_packed_layer* wt) {
  const nf_model_cfg* c = L.c;
  const int M = G.nr.t1 - G.nr.t0;
  if (M <= 0) return NF_OK;
  const int N = c->tp_size, rank = c->tp_rank;
  const int64_t D = c->d_model, qd = (int64_t)c->n_q_heads / N * c->head_dim, qd_full = qd * N, Dl = D / N;
  const int stages = L.p->spec.colocate ? 3 : 4;
  __nv_bfloat16* h1 = L.w->h1 + G.nr.t0 * D;
  if (G.col) {
    if (L.ns != L.cs) NF_CUDA(cudaStreamWaitEvent(L.cs, p->ev_agattn, 0));
    // the gathered attention output [N][M][qd] is the GEMM's A in slot layout (a 3-D TMA box per
    // k-block); NF_GEMM_ASLOTS=0 restores the interleave pass into [M][N qd] (A/B runs)
    const bool aslots = gemm_aslots_env() && qd % 64 == 0;
    if (!aslots) NF_CUDA(launch_interleave(L.w->ag, N, M, (int)qd, L.w->ocat, nullptr, L.cs));
    GemmArgs a{};
    if (aslots) {
      a.a_slots = N;
      a.a_slot_w = (int)qd;
    }
    a.epi = EPI_RESID;
    a.stages = stages;
    a.sk_part = L.w->sk_part;
    a.sk_slots = L.w->sk_slots;
    a.sk_flag = L.w->sk_flag;
    a.M = M;
    a.N = (int)Dl;
    a.K = (int)qd_full;
    a.n_valid = (int)Dl;
    a.out = L.w->hcol;
    a.ldo = Dl;
    a.resid = x + G.nr.t0 * D + rank * Dl;
    a.ldr = D;
    const bool fz = fused_ag_ok(L, M);
    if (fz) set_peer_ag_args(&a, L, M);  // all-gather fused into the epilogue (NEXT-3)
    {
      ProfScope ps(NF_OP_O, L.cs);
      NF_CUDA(launch_gemm(aslots ? L.w->ag : L.w->ocat, aslots ? qd : qd_full, (const __nv_bfloat16*)wt->w_o, qd_full,
                          a, clamp_dense(L, L.p->spec.sm[NF_OP_O]), L.cs));
    }
    if (fz) {
      comm_fused_site_barrier(L.comm);
      const PeerGeom& g = comm_peer_geom(L.comm);
      ProfScope ps(NF_OP_NET, L.ns);
      NF_CUDA(launch_peer_wait(comm_peer_bases(L.comm), g, 0, (uint32_t)(g.n * ((M + PEER_BM - 1) / PEER_BM) * (Dl / 64)),
                               comm_peer_timeout_ns(L.comm), L.ns));
      comm_count_fused(L.comm);
    } else {
      NF_TRY(edge(p->ev_o[gi], L.cs, L.ns));
      ProfScope ps(NF_OP_NET, L.ns);
      NF_TRY(comm_all_gather(L.comm, L.w->hcol, L.w->ag2, (size_t)M * Dl, L.ns));
    }
    if (L.ns != L.cs) NF_CUDA(cudaEventRecord(p->ev_ago, L.ns));
  } else {
    NF_TRY(wait_attention(p, L, G, L.cs));
    const bool fz = fused_site_ok(L, M);
    GemmArgs a{};
    a.epi = EPI_STORE;
    a.stages = stages;
    a.sk_part = L.w->sk_part;
    a.sk_slots = L.w->sk_slots;
    a.sk_flag = L.w->sk_flag;
    a.M = M;
    a.N = (int)D;
    a.K = (int)qd;
    a.n_valid = (int)D;
    a.out = h1;
    a.ldo = D;
    if (fz) {  // reduce-scatter in the epilogue; the owner reduce runs on the network stream meanwhile
      set_peer_args(&a, L, site_of(false, gi), M);
      NF_TRY(edge(p->ev_o[gi], L.cs, L.ns));
    }
    {
      ProfScope ps(NF_OP_O, L.cs);
      NF_CUDA(launch_gemm(L.w->o + G.nr.t0 * qd, qd, (const __nv_bfloat16*)wt->w_o_row, qd, a,
                          clamp_dense(L, L.p->spec.sm[NF_OP_O]), L.cs));
    }
    if (fz) {
      NF_TRY(run_peer_reduce(L, site_of(false, gi), M));
    } else {
      NF_TRY(edge(p->ev_o[gi], L.cs, L.ns));
      ProfScope ps(NF_OP_NET, L.ns);
      NF_TRY(comm_all_reduce_bf16(L.comm, h1, (size_t)M * D, L.ns, L.w->red));
    }
    if (L.ns != L.cs) NF_CUDA(cudaEventRecord(p->ev_aro[gi], L.ns));
  }
  return NF_OK;
}

// Stage C: h1 (+ its RMS statistics), Up/Gate + SiLU, row-parallel Down partial, AR.
nf_status tp_stage_c(nf_plan* p, const LayerCtx& L, int gi, const Group& G, const __nv_bfloat16* x,
                     const nf_packed_layer* wt, __nv_bfloat16* x_out) {
  const nf_model_cfg* c = L.c;
  const int M = G.nr.t1 - G.nr.t0;
  if (M <= 0) return NF_OK;
  const int N = c->tp_size;
  const int64_t D = c->d_model, Fl = c->d_ffn / N, Dl = D / N;
  const int T = L.m->T;
  const int stages = L.p->spec.colocate ? 3 : 4;
  __nv_bfloat16* h1 = L.w->h1 + G.nr.t0 * D;
  if (G.col) {
    if (L.ns != L.cs) NF_CUDA(cudaStreamWaitEvent(L.cs, p->ev_ago, 0));
    if (fused_ag_ok(L, M))
      NF_CUDA(launch_interleave_from_peers(peer_result(L, 0), N, M, (int)Dl, h1, L.w->part_h1 + G.nr.t0, L.cs));
    else
      NF_CUDA(launch_interleave(L.w->ag2, N, M, (int)Dl, h1, L.w->part_h1 + G.nr.t0, L.cs));
  } else {
    if (L.ns != L.cs) NF_CUDA(cudaStreamWaitEvent(L.cs, p->ev_aro[gi], 0));
    if (fused_site_ok(L, M))
      NF_CUDA(launch_resid_add_rows_from(h1, peer_result(L, site_of(false, gi)), x + G.nr.t0 * D, M, (int)D,
                                         L.w->part_h1 + G.nr.t0, L.cs));
    else
      NF_CUDA(launch_resid_add_rows(h1, x + G.nr.t0 * D, M, (int)D, L.w->part_h1 + G.nr.t0, L.cs));
  }
  if (c->n_experts > 0) {
    // MoE: every expert's F columns are split across ranks; this rank's weighted partial sum
    NF_TRY(run_moe_ffn(L, G.nr, L.w->h1, wt, nullptr, x_out, nullptr));
  } else {
    GemmArgs u{};
    u.epi = EPI_SILU;
    u.stages = stages;
    u.sk_part = L.w->sk_part;
    u.sk_slots = L.w->sk_slots;
    u.sk_flag = L.w->sk_flag;
    u.M = M;
    u.N = (int)(((Fl + 127) / 128) * 256);
    u.K = (int)D;
    u.n_valid = (int)Fl;
    u.out = L.w->m + G.nr.t0 * Fl;
    u.ldo = Fl;
    u.norm_part = L.w->part_h1 + G.nr.t0;
    u.norm_nparts = 1;
    u.norm_stride = T;
    u.inv_d = 1.f / D;
    u.eps = c->rms_eps;
    {
      ProfScope ps(NF_OP_UG, L.cs);
      NF_CUDA(launch_gemm(h1, D, (const __nv_bfloat16*)wt->w_gate_up, D, u, clamp_dense(L, L.p->spec.sm[NF_OP_UG]), L.cs));
    }
    GemmArgs d{};
    d.epi = EPI_STORE;
    d.stages = stages;
    d.sk_part = L.w->sk_part;
    d.sk_slots = L.w->sk_slots;
    d.sk_flag = L.w->sk_flag;
    d.M = M;
    d.N = (int)D;
    d.K = (int)Fl;
    d.n_valid = (int)D;
    d.out = x_out + G.nr.t0 * D;
    d.ldo = D;
    if (fused_site_ok(L, M)) {
      set_peer_args(&d, L, site_of(true, gi), M);
      NF_TRY(edge(p->ev_d[gi], L.cs, L.ns));
    }
    {
      ProfScope ps(NF_OP_DOWN, L.cs);
      NF_CUDA(launch_gemm(L.w->m + G.nr.t0 * Fl, Fl, (const __nv_bfloat16*)wt->w_down, Fl, d,
                          clamp_dense(L, L.p->spec.sm[NF_OP_DOWN]), L.cs));
    }
  }
  if (c->n_experts == 0 && fused_site_ok(L, M)) {
    NF_TRY(run_peer_reduce(L, site_of(true, gi), M));
  } else {
    NF_TRY(edge(p->ev_d[gi], L.cs, L.ns));
    ProfScope ps(NF_OP_NET, L.ns);
    NF_TRY(comm_all_reduce_bf16(L.comm, x_out + G.nr.t0 * D, (size_t)M * D, L.ns, L.w->red));
  }
  if (L.ns != L.cs) NF_CUDA(cudaEventRecord(p->ev_ard[gi], L.ns));
  return NF_OK;
}

// Stage D: x_out = h1 + AR(Down partials), RMS statistics of x_out for the next layer.
nf_status tp_stage_d(nf_plan* p, const LayerCtx& L, int gi, const Group& G, __nv_bfloat16* x_out, float* part_out) {
  const int M = G.nr.t1 - G.nr.t0;
  if (M <= 0) return NF_OK;
  const int64_t D = L.c->d_model;
  if (L.ns != L.cs) NF_CUDA(cudaStreamWaitEvent(L.cs, p->ev_ard[gi], 0));
  if (L.c->n_experts == 0 && fused_site_ok(L, M))
    NF_CUDA(launch_resid_add_rows_from(x_out + G.nr.t0 * D, peer_result(L, site_of(true, gi)), L.w->h1 + G.nr.t0 * D,
                                       M, (int)D, part_out ? part_out + G.nr.t0 : nullptr, L.cs));
  else
    NF_CUDA(launch_resid_add_rows(x_out + G.nr.t0 * D, L.w->h1 + G.nr.t0 * D, M, (int)D,
                                  part_out ? part_out + G.nr.t0 : nullptr, L.cs));
  return NF_OK;
}

// Optional inspection copy (nf_model_step_ex hidden taps): rows [t0, t1) of an internal-order
// buffer to their caller rows.
nf_status tap_rows(const LayerCtx& L, void* dst, const __nv_bfloat16* src, int t0, int t1) {
  if (!dst || t1 <= t0) return NF_OK;
  const int D = L.c->d_model;
  NF_CUDA(launch_scatter_rows(src + (int64_t)t0 * D, L.meta_dev + L.m->off_tok_src + t0, t1 - t0, D,
                              (__nv_bfloat16*)dst, L.cs));
  return NF_OK;
}

int tp_dec_side_env() {  // (dev) NF_TP_DEC_SIDE=1: decode side streams when there is no memory partition
  const char* e = getenv("NF_TP_DEC_SIDE");
  return e && e[0] == '1';
}

// OVERLAP plans run on green-context partitions when available: fork the
// caller stream into the compute / memory (/ network) partition streams, join at the end.
nf_status enter_partitions(nf_plan* p, LayerCtx* L, cudaStream_t caller) {
  if (p->spec.mode != NF_OVERLAP || p->spec.colocate) return NF_OK;
  // TP: a network partition only for collectives whose CTA count is known to fit it
  // (an emulated group, or NCCL capped to <= the partition); otherwise NCCL stays on
  // an ordinary stream (it could otherwise wait for SMs held by a co-partitioned kernel).
  int net = 0;
  if (p->cfg.tp_size > 1 && L->comm) {
    const int want = p->spec.sm[NF_OP_NET];
    const int cap = comm_max_ctas(L->comm);
    if (comm_emulated(L->comm) || (cap > 0 && cap <= (want + 7) / 8 * 8)) net = want;
  }
  const bool two = p->cfg.tp_size > 1 && L->comm && !p->spec.colocate;  // per-group compute streams
  const bool no_mem = p->spec.sm[NF_OP_DECODE_ATTN] >= num_sms();  // plan without a memory partition
  if (!green_setup(p, p->spec.sm[NF_OP_DECODE_ATTN], net)) {
    if (no_mem) {
      L->ms = L->cs;
      L->dec_on_cs = true;
    }
    if (two) {
      NF_CUDA(cudaEventRecord(p->ev_fork2, caller));
      NF_CUDA(cudaStreamWaitEvent(p->cs2, p->ev_fork2, 0));
      L->cs2 = p->cs2;
    }
    return NF_OK;
  }
  NF_CUDA(cudaEventRecord(p->ev_fork, caller));
  if (two) {
    NF_CUDA(cudaStreamWaitEvent(p->green_cs2, p->ev_fork, 0));
    L->cs2 = p->green_cs2;
  }
  NF_CUDA(cudaStreamWaitEvent(p->green_cs, p->ev_fork, 0));
  L->cs = p->green_cs;
  if (p->green_ms) {
    NF_CUDA(cudaStreamWaitEvent(p->green_ms, p->ev_fork, 0));
    L->ms = p->green_ms;
  } else if (tp_dec_side_env() && p->green_ds1 && p->green_ds2) {
    NF_CUDA(cudaStreamWaitEvent(p->green_ds1, p->ev_fork, 0));
    L->ms = p->green_ds1;
    if (two) {
      NF_CUDA(cudaStreamWaitEvent(p->green_ds2, p->ev_fork, 0));
      L->ms2 = p->green_ds2;
    }
    L->dec_side = true;
  } else {
    L->ms = L->cs;
    L->dec_on_cs = true;
  }
  L->cap_dense = p->green_dense_sms;
  L->cap_dec = p->green_dec_sms;
  if (p->green_ns && L->ns != caller) {
    NF_CUDA(cudaStreamWaitEvent(p->green_ns, p->ev_fork, 0));
    L->ns = p->green_ns;
  }
  return NF_OK;
}
nf_status leave_partitions(nf_plan* p, const LayerCtx& L, cudaStream_t caller) {
  if (L.cs2) {
    NF_CUDA(cudaEventRecord(p->ev_join_c2, L.cs2));
    NF_CUDA(cudaStreamWaitEvent(caller, p->ev_join_c2, 0));
  }
  if (L.cs != caller) {
    NF_CUDA(cudaEventRecord(p->ev_join_c, L.cs));
    NF_CUDA(cudaStreamWaitEvent(caller, p->ev_join_c, 0));
  }
  if (L.ms2) {
    NF_CUDA(cudaEventRecord(p->ev_join_m2, L.ms2));
    NF_CUDA(cudaStreamWaitEvent(caller, p->ev_join_m2, 0));
  }
  if (L.ms != caller && L.ms != L.cs) {
    NF_CUDA(cudaEventRecord(p->ev_join_m, L.ms));
    NF_CUDA(cudaStreamWaitEvent(caller, p->ev_join_m, 0));
  }
  if (L.ns != caller && L.ns != L.cs) {
    NF_CUDA(cudaEventRecord(p->ev_join_n, L.ns));
    NF_CUDA(cudaStreamWaitEvent(caller, p->ev_join_n, 0));
  }
  return NF_OK;
}

}  // namespace

// One layer with the plan's pipeline.  x/part: input + its RMS partials (nparts),
// x_out/part_out: output + partials for the next layer.
nf_status run_layer(nf_plan* p, const LayerCtx& L, const nf_packed_layer* wt, void* pool, const __nv_bfloat16* x,
                    const float* part, int nparts, __nv_bfloat16* x_out, float* part_out, void* tap) {
  const auto& nanos = L.m->nanos;
  const int mode = p->spec.mode;
  if (L.c->tp_size > 1) {
    const auto groups = dense_groups(p, *L.m);
    if (mode != NF_OVERLAP) {
      for (size_t g = 0; g < groups.size(); ++g) {
        NF_TRY(tp_front(p, L, (int)g, groups[g], x, part, nparts, wt, pool));
        NF_TRY(tp_stage_a(p, L, (int)g, groups[g]));
        NF_TRY(tp_stage_b(p, L, (int)g, groups[g], x, wt));
        NF_TRY(tp_stage_c(p, L, (int)g, groups[g], x, wt, x_out));
        NF_TRY(tp_stage_d(p, L, (int)g, groups[g], x_out, part_out));
        NF_TRY(tap_rows(L, tap, x_out, groups[g].nr.t0, groups[g].nr.t1));
      }
      return NF_OK;
    }
    Workspace wg[NF_MAX_NANO];
    std::vector<LayerCtx> Lg;
    for (size_t g = 0; g < groups.size(); ++g) Lg.push_back(group_ctx(L, (int)g, &wg[g]));
    for (size_t g = 0; g < groups.size(); ++g) NF_TRY(tp_front(p, Lg[g], (int)g, groups[g], x, part, nparts, wt, pool));
    NF_TRY(tp_stage_a(p, Lg[0], 0, groups[0]));
    for (size_t g = 0; g < groups.size(); ++g) NF_TRY(tp_stage_b(p, Lg[g], (int)g, groups[g], x, wt));
    for (size_t g = 0; g < groups.size(); ++g) NF_TRY(tp_stage_c(p, Lg[g], (int)g, groups[g], x, wt, x_out));
    for (size_t g = 0; g < groups.size(); ++g) {
      NF_TRY(tp_stage_d(p, Lg[g], (int)g, groups[g], x_out, part_out));
      NF_TRY(tap_rows(Lg[g], tap, x_out, groups[g].nr.t0, groups[g].nr.t1));
    }
    return NF_OK;
  }
  if (mode != NF_OVERLAP) {
    for (size_t k = 0; k < nanos.size(); ++k) {
      NF_TRY(run_kqv(L, nanos[k], x, part, nparts, wt, pool));
      NF_TRY(run_attn(L, nanos[k], L.cs));
      NF_TRY(run_dense_tail(L, nanos[k], x, wt, x_out, part_out));
      NF_TRY(tap_rows(L, tap, x_out, nanos[k].t0, nanos[k].t1));
    }
    return NF_OK;
  }
  // OVERLAP: KQV of every nano first, attention on the memory stream as soon as
  // its KQV lands, then the dense tail of each nano after its attention.
  for (size_t k = 0; k < nanos.size(); ++k) {
    NF_TRY(run_kqv(L, nanos[k], x, part, nparts, wt, pool));
    NF_TRY(edge(p->ev_kqv[k], L.cs, L.ms));
    NF_TRY(run_decode(L, nanos[k], L.ms, 1));
    NF_CUDA(cudaEventRecord(p->ev_att[k], L.ms));
    NF_TRY(run_prefill(L, nanos[k], L.cs));
    NF_TRY(run_decode(L, nanos[k], L.cs, 2));
  }
  for (size_t k = 0; k < nanos.size(); ++k) {
    NF_CUDA(cudaStreamWaitEvent(L.cs, p->ev_att[k], 0));
    NF_TRY(run_dense_tail(L, nanos[k], x, wt, x_out, part_out));
    NF_TRY(tap_rows(L, tap, x_out, nanos[k].t0, nanos[k].t1));
  }
  return NF_OK;
}

namespace {

nf_status check_comm(const nf_model_cfg* c, nf_comm* comm) {
  if (c->tp_size == 1) return NF_OK;
  if (!comm) return set_error(NF_EINVAL, "tp_size > 1 needs a communicator");
  if (comm_size(comm) != c->tp_size || comm_rank(comm) != c->tp_rank)
    return set_error(NF_EINVAL, "communicator size/rank %d/%d != cfg %d/%d", comm_size(comm), comm_rank(comm),
                     c->tp_size, c->tp_rank);
  return NF_OK;
}

// The launches of one model step after the metadata upload (captured into a CUDA
// graph when the plan asks for it).
nf_status model_step_launches(nf_plan* p, nf_comm* comm, const nf_model_weights* w, void* const* kv_pools,
                              const nf_batch* b, const int32_t* token_ids, const nf_step_outputs* out,
                              const StepMeta& m, const Workspace& wsp, cudaStream_t cs) {
  const nf_model_cfg* c = &p->cfg;
  NF_CUDA(cudaMemsetAsync(wsp.sk_flag, 0, (size_t)wsp.sk_flag_total * 4, cs));
  const int D = c->d_model;
  const int NP = D / GEMM_NORM_COLS;
  void* const* taps = out->hidden;
  // token ids in internal row order: the embedding gather reads token_ids[tok_src[row]]
  // (+ RMS partials, one part); ids outside [0, V) are clamped (documented in nf.h)
  NF_CUDA(launch_gather_ids_embed((const __nv_bfloat16*)w->embed, token_ids, wsp.meta + m.off_tok_src, m.T, D,
                                  c->vocab, wsp.xa, wsp.part_a, cs));
  LayerCtx L{};
  L.p = p;
  L.c = c;
  L.m = &m;
  L.w = &wsp;
  L.meta_dev = wsp.meta;
  L.cs = cs;
  L.ms = p->spec.mode == NF_OVERLAP ? p->mem_stream : cs;
  L.ns = (p->spec.mode == NF_OVERLAP && c->tp_size > 1) ? p->net_stream : cs;
  L.comm = comm;
  if (taps && taps[0]) NF_TRY(tap_rows(L, taps[0], wsp.xa, 0, m.T));
  const int NPn = c->tp_size > 1 ? 1 : NP;  // RMS partials per row of layer outputs
  __nv_bfloat16 *x = wsp.xa, *y = wsp.xb;
  float *px = wsp.part_a, *py = wsp.part_b;
  std::vector<CUtensorMap> maps(c->n_layers), pmaps(c->n_layers);
  for (int l = 0; l < c->n_layers; ++l) {
    NF_CUDA(make_pool_tmap(&maps[l], kv_pools[l], b->n_pages_pool, c->n_kv_heads / c->tp_size, c->head_dim,
                           c->page_size));
    NF_CUDA(make_page_tmap(&pmaps[l], kv_pools[l], b->n_pages_pool, c->n_kv_heads / c->tp_size, c->head_dim,
                           c->page_size));
  }
  NF_TRY(enter_partitions(p, &L, cs));
  comm_fused_step_barrier(comm);
  auto tap_of = [&](int l) -> void* { return taps ? taps[l + 1] : nullptr; };
  if (p->spec.mode != NF_OVERLAP) {
    int nparts = 1;
    for (int l = 0; l < c->n_layers; ++l) {
      L.pool_map = maps[l];
      L.page_map = pmaps[l];
      NF_TRY(run_layer(p, L, &w->layers[l], kv_pools[l], x, px, nparts, y, py, tap_of(l)));
      std::swap(x, y);
      std::swap(px, py);
      nparts = NPn;
    }
  } else if (c->tp_size > 1) {
    // TP operation-level pipeline across layers: layer l+1's
    // KQV of a group is issued right after that group's layer-l output is complete.
    const auto groups = dense_groups(p, m);
    const int G = (int)groups.size();
    Workspace wg[NF_MAX_NANO];
    std::vector<LayerCtx> Lg;
    L.pool_map = maps[0];
    L.page_map = pmaps[0];
    for (int g = 0; g < G; ++g) Lg.push_back(group_ctx(L, g, &wg[g]));
    for (int g = 0; g < G; ++g) NF_TRY(tp_front(p, Lg[g], g, groups[g], x, px, 1, &w->layers[0], kv_pools[0]));
    for (int l = 0; l < c->n_layers; ++l) {
      const nf_packed_layer* wt = &w->layers[l];
      NF_TRY(tp_stage_a(p, Lg[0], 0, groups[0]));
      for (int g = 0; g < G; ++g) NF_TRY(tp_stage_b(p, Lg[g], g, groups[g], x, wt));
      for (int g = 0; g < G; ++g) NF_TRY(tp_stage_c(p, Lg[g], g, groups[g], x, wt, y));
      for (int g = 0; g < G; ++g) {
        NF_TRY(tp_stage_d(p, Lg[g], g, groups[g], y, py));
        NF_TRY(tap_rows(Lg[g], tap_of(l), y, groups[g].nr.t0, groups[g].nr.t1));
        if (l + 1 < c->n_layers) {
          Lg[g].pool_map = maps[l + 1];
          Lg[g].page_map = pmaps[l + 1];
          NF_TRY(tp_front(p, Lg[g], g, groups[g], y, py, 1, &w->layers[l + 1], kv_pools[l + 1]));
        }
      }
      std::swap(x, y);
      std::swap(px, py);
    }
  } else {
    // Operation-level pipeline across layers (single-GPU variant
    // PAPER.md:691): the compute stream runs, per nano-batch k, O_k UG_k D_k of
    // layer l then KQV_k of layer l+1; the memory stream runs ATT_k(l+1) as
    // soon as KQV_k(l+1) lands, overlapping the other nano-batches' dense ops.
    const auto& nanos = m.nanos;
    L.pool_map = maps[0];
    L.page_map = pmaps[0];
    for (size_t k = 0; k < nanos.size(); ++k) {
      NF_TRY(run_kqv(L, nanos[k], x, px, 1, &w->layers[0], kv_pools[0]));
      NF_TRY(edge(p->ev_kqv[k], L.cs, L.ms));
      NF_TRY(run_decode(L, nanos[k], L.ms, 1));
      NF_CUDA(cudaEventRecord(p->ev_att[k], L.ms));
      NF_TRY(run_prefill(L, nanos[k], L.cs));
      NF_TRY(run_decode(L, nanos[k], L.cs, 2));
    }
    for (int l = 0; l < c->n_layers; ++l) {
      for (size_t k = 0; k < nanos.size(); ++k) {
        NF_CUDA(cudaStreamWaitEvent(L.cs, p->ev_att[k], 0));
        NF_TRY(run_dense_tail(L, nanos[k], x, &w->layers[l], y, py));
        NF_TRY(tap_rows(L, tap_of(l), y, nanos[k].t0, nanos[k].t1));
        if (l + 1 < c->n_layers) {
          L.pool_map = maps[l + 1];
          L.page_map = pmaps[l + 1];
          NF_TRY(run_kqv(L, nanos[k], y, py, NPn, &w->layers[l + 1], kv_pools[l + 1]));
          NF_TRY(edge(p->ev_kqv[k], L.cs, L.ms));
          NF_TRY(run_decode(L, nanos[k], L.ms, 1));
          NF_CUDA(cudaEventRecord(p->ev_att[k], L.ms));
          NF_TRY(run_prefill(L, nanos[k], L.cs));
          NF_TRY(run_decode(L, nanos[k], L.cs, 2));
        }
      }
      std::swap(x, y);
      std::swap(px, py);
    }
  }
  NF_TRY(leave_partitions(p, L, cs));
  // final RMSNorm (gamma folded into lm_head_packed) + LM head over this rank's vocab
  // shard + argmax; at TP > 1 the per-rank (max, global index) pairs are AllGathered and
  // merged
  int32_t* next_ids = out->next_ids;
  NF_CUDA(launch_fill_i32(next_ids, b->n_req, -1, cs));
  const int Vl = c->vocab / c->tp_size;
  if (m.n_emit > 0) {
    const int* erow = wsp.meta + m.off_emit_row;
    NF_CUDA(launch_gather_rows(x, erow, m.n_emit, D, wsp.lm_rows, wsp.lm_part, cs));
    GemmArgs a{};
    a.epi = EPI_ARGMAX;
    a.sk_part = wsp.sk_part;
    a.sk_slots = wsp.sk_slots;
    a.sk_flag = wsp.sk_flag;
    a.M = m.n_emit;
    a.N = Vl;
    a.K = D;
    a.n_valid = Vl;
    a.am_val = wsp.am_val;
    a.am_idx = wsp.am_idx;
    a.am_stride = m.n_emit;
    {
      ProfScope ps(NF_PROF_LMHEAD, cs);
      NF_CUDA(launch_gemm(wsp.lm_rows, D, (const __nv_bfloat16*)w->lm_head_packed, D, a, num_sms(), cs));
    }
    const int vt = (Vl + GEMM_BN - 1) / GEMM_BN;
    if (c->tp_size == 1) {
      NF_CUDA(launch_argmax_reduce(wsp.am_val, wsp.am_idx, vt, m.n_emit, m.n_emit, wsp.meta + m.off_emit_req, next_ids,
                                   cs));
    } else {
      NF_CUDA(launch_argmax_pairs(wsp.am_val, wsp.am_idx, vt, m.n_emit, m.n_emit, c->tp_rank * Vl, wsp.am_pair, cs));
      {
        ProfScope ps(NF_OP_NET, cs);
        NF_TRY(comm_all_gather(comm, wsp.am_pair, wsp.am_pair_all, (size_t)m.n_emit * 4, cs));
      }
      NF_CUDA(launch_argmax_merge(wsp.am_pair_all, c->tp_size, m.n_emit, wsp.meta + m.off_emit_req, next_ids, cs));
    }
    if (out->logits) {
      // inspection: logits of the emitting rows in caller request order (plain store epilogue)
      // (the argmax above skips the final RMSNorm's positive row scale 1/rms, which cannot
      // change a row's argmax; the logits apply it)
      NF_CUDA(launch_gather_rows(x, wsp.meta + m.off_emit_sorted, m.n_emit, D, wsp.lm_rows, wsp.lm_part, cs));
      GemmArgs s{};
      s.epi = EPI_STORE;
      s.M = m.n_emit;
      s.N = Vl;
      s.K = D;
      s.n_valid = Vl;
      s.norm_part = wsp.lm_part;
      s.norm_nparts = 1;
      s.norm_stride = m.n_emit;
      s.inv_d = 1.f / D;
      s.eps = c->rms_eps;
      s.out = (__nv_bfloat16*)out->logits;
      s.ldo = Vl;
      NF_CUDA(launch_gemm(wsp.lm_rows, D, (const __nv_bfloat16*)w->lm_head_packed, D, s, num_sms(), cs));
    }
  }
  // join the memory and network streams when the plan forked onto them
  if (L.ms != cs && L.ms == p->mem_stream) {
    NF_CUDA(cudaEventRecord(p->ev_join, p->mem_stream));
    NF_CUDA(cudaStreamWaitEvent(cs, p->ev_join, 0));
  }
  if (L.ns != cs && L.ns == p->net_stream) {
    NF_CUDA(cudaEventRecord(p->ev_join_n, p->net_stream));
    NF_CUDA(cudaStreamWaitEvent(cs, p->ev_join_n, 0));
  }
  return NF_OK;
}

// Launch-structure key of a model step: everything the captured kernels' parameters
// depend on besides the uploaded metadata contents.
std::vector<int64_t> graph_key(const nf_plan* p, nf_comm* comm, const nf_model_weights* w, void* const* kv_pools,
                               const nf_batch* b, const int32_t* token_ids, const nf_step_outputs* out,
                               const StepMeta& m, void* ws, cudaStream_t cs) {
  (void)cs;
  std::vector<int64_t> k{(int64_t)(uintptr_t)comm, (int64_t)(uintptr_t)w->embed, (int64_t)(uintptr_t)w->lm_head_packed,
                         (int64_t)(uintptr_t)token_ids, (int64_t)(uintptr_t)out->next_ids, (int64_t)(uintptr_t)ws,
                         b->n_req, b->n_pages_pool, m.T, m.n_emit,
                         (int64_t)m.off_pos, (int64_t)m.off_slot, (int64_t)m.off_pages, (int64_t)m.off_dec,
                         (int64_t)m.off_pf, (int64_t)m.off_emit_row, (int64_t)m.off_emit_req,
                         (int64_t)m.off_tok_src, (int64_t)m.off_emit_sorted};
  for (const auto& nr : m.nanos)
    for (int v : {nr.r0, nr.r1, nr.t0, nr.t1, nr.dec_off, nr.dec_n, nr.dec_cs_n, nr.pf_off, nr.pf_n}) k.push_back(v);
  for (int l = 0; l < p->cfg.n_layers; ++l) {
    k.push_back((int64_t)(uintptr_t)kv_pools[l]);
    const nf_packed_layer& q = w->layers[l];
    for (const void* ptr : {q.w_qkv, q.w_o, q.w_o_row, q.w_gate_up, q.w_down, q.w_router})
      k.push_back((int64_t)(uintptr_t)ptr);
  }
  return k;
}

nf_status model_step_impl(const nf_plan* plan, nf_comm* comm, const nf_model_weights* w, void* const* kv_pools,
                          const nf_batch* b, const int32_t* token_ids, const nf_step_outputs* out, void* ws,
                          size_t ws_bytes, void* stream) {
  if (!plan) return set_error(NF_EINVAL, "plan is NULL");
  nf_plan* p = const_cast<nf_plan*>(plan);
  const nf_model_cfg* c = &p->cfg;
  NF_TRY(validate_batch(c, b));
  NF_TRY(check_comm(c, comm));
  if (!w || !w->embed || !w->layers || !w->lm_head_packed || !kv_pools || !token_ids || !out || !out->next_ids || !ws)
    return set_error(NF_EINVAL, "NULL pointer argument");
  for (int l = 0; l < c->n_layers; ++l)
    if (!kv_pools[l]) return set_error(NF_EINVAL, "kv_pools[%d] is NULL", l);
  for (int l = 0; l < c->n_layers; ++l) NF_TRY(validate_packed(c, &w->layers[l], l));
  Workspace wsp = carve_workspace(c, b, ws);
  if (ws_bytes < wsp.total) return set_error(NF_EINVAL, "workspace %zu bytes < required %zu", ws_bytes, wsp.total);
  NF_TRY(ensure_runtime(p));
  std::vector<int> order, cuts;
  BatchView view;
  bool use_view = false;
  plan_order(p, b, true, &order, &cuts, &view, &use_view);
  StepMeta m;
  if (use_view)
    build_meta(c, &view.b, order, cuts, &m, &view.caller_row0, &view.caller_req);
  else
    build_meta(c, b, order, cuts, &m);
  cudaStream_t cs = (cudaStream_t)stream;
  NF_TRY(upload_meta(p, m, wsp.meta, cs));
  // CUDA graph (plan spec.graph): not with an emulated group (host barriers inside the
  // collectives), inspection outputs or per-launch profiling
  const bool want_graph = p->spec.graph && !comm_host_sync(comm) && !out->logits && !out->hidden && !profile_active();
  if (!want_graph) return model_step_launches(p, comm, w, kv_pools, b, token_ids, out, m, wsp, cs);
  std::vector<int64_t> key = graph_key(p, comm, w, kv_pools, b, token_ids, out, m, ws, cs);
  for (auto& g : p->graphs)
    if (g.key == key) {
      NF_CUDA(cudaGraphLaunch(g.exec, cs));
      count_launch(1);
      return NF_OK;
    }
  // capture on the plan's own stream (the caller's may be the legacy default stream,
  // which cannot be captured); the graph is then launched on the caller's stream,
  // after the metadata upload
  if (!p->cap_stream) NF_CUDA(cudaStreamCreateWithFlags(&p->cap_stream, cudaStreamNonBlocking));
  NF_CUDA(cudaStreamBeginCapture(p->cap_stream, cudaStreamCaptureModeThreadLocal));
  const nf_status st = model_step_launches(p, comm, w, kv_pools, b, token_ids, out, m, wsp, p->cap_stream);
  cudaGraph_t graph = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(p->cap_stream, &graph);
  if (st != NF_OK) {
    if (graph) cudaGraphDestroy(graph);
    return st;
  }
  if (ce != cudaSuccess) return set_error(NF_ECUDA, "cudaStreamEndCapture: %s", cudaGetErrorString(ce));
  cudaGraphExec_t exec = nullptr;
  const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ie != cudaSuccess) return set_error(NF_ECUDA, "cudaGraphInstantiate: %s", cudaGetErrorString(ie));
  if (p->graphs.size() >= 4) {
    cudaGraphExecDestroy(p->graphs.front().exec);
    p->graphs.erase(p->graphs.begin());
  }
  p->graphs.push_back(NfGraph{std::move(key), exec});
  p->graph_note = "captured " + std::to_string(p->graphs.size()) + " graph(s)";
  NF_CUDA(cudaGraphLaunch(exec, cs));
  count_launch(1);
  return NF_OK;
}

}  // namespace

}  // namespace nf

extern "C" {

nf_status nf_layer_forward(const nf_plan* plan, nf_comm* comm, const nf_packed_layer* w, void* kv_pool, const nf_batch* b,
                           const void* x_in, void* x_out, void* ws, size_t ws_bytes, void* stream) {
  if (!plan) return set_error(NF_EINVAL, "plan is NULL");
  nf_plan* p = const_cast<nf_plan*>(plan);
  const nf_model_cfg* c = &p->cfg;
  NF_TRY(validate_batch(c, b));
  NF_TRY(check_comm(c, comm));
  if (!w || !kv_pool || !x_in || !x_out || !ws) return set_error(NF_EINVAL, "NULL pointer argument");
  NF_TRY(validate_packed(c, w, 0));
  Workspace wsp = carve_workspace(c, b, ws);
  if (ws_bytes < wsp.total) return set_error(NF_EINVAL, "workspace %zu bytes < required %zu", ws_bytes, wsp.total);
  NF_TRY(ensure_runtime(p));
  std::vector<int> order, cuts;
  plan_order(p, b, false, &order, &cuts);
  StepMeta m;
  build_meta(c, b, order, cuts, &m);
  cudaStream_t cs = (cudaStream_t)stream;
  NF_TRY(upload_meta(p, m, wsp.meta, cs));
  NF_CUDA(cudaMemsetAsync(wsp.sk_flag, 0, (size_t)wsp.sk_flag_total * 4, cs));
  LayerCtx L{};
  L.p = p;
  L.c = c;
  L.m = &m;
  L.w = &wsp;
  L.meta_dev = wsp.meta;
  L.cs = cs;
  L.ms = p->spec.mode == NF_OVERLAP ? p->mem_stream : cs;
  L.ns = (p->spec.mode == NF_OVERLAP && c->tp_size > 1) ? p->net_stream : cs;
  L.comm = comm;
  NF_CUDA(make_pool_tmap(&L.pool_map, kv_pool, b->n_pages_pool, c->n_kv_heads / c->tp_size, c->head_dim, c->page_size));
  NF_CUDA(make_page_tmap(&L.page_map, kv_pool, b->n_pages_pool, c->n_kv_heads / c->tp_size, c->head_dim, c->page_size));
  // RMS partials of x_in (one part per row)
  NF_CUDA(launch_gather_rows((const __nv_bfloat16*)x_in, nullptr, m.T, c->d_model, nullptr, wsp.part_a, cs));
  NF_TRY(enter_partitions(p, &L, cs));
  comm_fused_step_barrier(comm);
  NF_TRY(run_layer(p, L, w, kv_pool, (const __nv_bfloat16*)x_in, wsp.part_a, 1, (__nv_bfloat16*)x_out, nullptr, nullptr));
  NF_TRY(leave_partitions(p, L, cs));
  if (L.ms != cs && L.ms == p->mem_stream) {
    NF_CUDA(cudaEventRecord(p->ev_join, p->mem_stream));
    NF_CUDA(cudaStreamWaitEvent(cs, p->ev_join, 0));
  }
  if (L.ns != cs && L.ns == p->net_stream) {
    NF_CUDA(cudaEventRecord(p->ev_join_n, p->net_stream));
    NF_CUDA(cudaStreamWaitEvent(cs, p->ev_join_n, 0));
  }
  return NF_OK;
}

nf_status nf_model_step(const nf_plan* plan, nf_comm* comm, const nf_model_weights* w, void* const* kv_pools,
                        const nf_batch* b, const int32_t* token_ids, int32_t* next_ids, void* ws, size_t ws_bytes,
                        void* stream) {
  nf_step_outputs out{next_ids, nullptr, nullptr};
  return model_step_impl(plan, comm, w, kv_pools, b, token_ids, &out, ws, ws_bytes, stream);
}

nf_status nf_model_step_ex(const nf_plan* plan, nf_comm* comm, const nf_model_weights* w, void* const* kv_pools,
                           const nf_batch* b, const int32_t* token_ids, const nf_step_outputs* out, void* ws,
                           size_t ws_bytes, void* stream) {
  return model_step_impl(plan, comm, w, kv_pools, b, token_ids, out, ws, ws_bytes, stream);
}

// ------------------------------------------------------------------ MoE op-level entries
int64_t nf_moe_rows_cap(const nf_model_cfg* c, int32_t T) {
  if (!c || c->n_experts <= 0 || T < 0) return 0;
  return moe_rows_cap(c, T);
}

size_t nf_moe_route_ws_bytes(const nf_model_cfg* c, int32_t T) {
  if (!c || c->n_experts <= 0 || T < 0) return 0;
  return ((size_t)T + c->n_experts + 2 * (size_t)moe_rows_cap(c, T) + moe_group_ints(T, c->n_experts) + 1) * 4 + 1024;
}

nf_status nf_moe_route(const nf_model_cfg* c, const void* h1, const void* router_packed, int32_t T, int32_t* ids,
                       float* wts, int32_t* grp_off, int32_t* dst, int32_t* row_tok, void* ws, size_t ws_bytes,
                       void* stream) {
  NF_TRY(validate_cfg(c));
  if (c->n_experts <= 0) return set_error(NF_EINVAL, "nf_moe_route needs n_experts > 0");
  if (T < 1) return set_error(NF_EINVAL, "T = %d < 1", T);
  if (!h1 || !router_packed || !ids || !wts || !grp_off || !dst || !row_tok || !ws)
    return set_error(NF_EINVAL, "NULL pointer argument");
  if (ws_bytes < nf_moe_route_ws_bytes(c, T))
    return set_error(NF_EINVAL, "workspace %zu bytes < required %zu", ws_bytes, nf_moe_route_ws_bytes(c, T));
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t cap = moe_rows_cap(c, T);
  float* inv = (float*)ws;
  int* grp_end = (int*)(inv + T);
  float* row_w = (float*)(grp_end + c->n_experts);
  float* row_inv = row_w + cap;
  int* cta = (int*)(row_inv + cap);
  MoeGroupArgs g{};
  g.cta_cnt = cta;
  g.cta_base = cta + moe_group_ints(T, c->n_experts) / 2;
  g.counter = cta + moe_group_ints(T, c->n_experts);
  g.grp_off = grp_off;
  g.grp_end = grp_end;
  g.row_tok = row_tok;
  g.row_w = row_w;
  g.row_inv = row_inv;
  g.tile = GEMM_BM;
  NF_CUDA(cudaMemsetAsync(g.counter, 0, 4, st));
  NF_CUDA(launch_moe_route((const __nv_bfloat16*)h1, T, c->d_model, (const float*)router_packed, c->n_experts,
                           c->top_k, c->rms_eps, ids, wts, inv, g, st));
  NF_CUDA(launch_moe_scatter((const __nv_bfloat16*)h1, T, c->d_model, c->top_k, c->n_experts, ids, wts, inv, g, dst,
                             nullptr, st));
  return NF_OK;
}

nf_status nf_plan_probe_partitions(nf_plan* p, nf_comm* comm, int32_t* smids_out, int32_t n_sm, void* stream) {
  if (!p || !smids_out) return set_error(NF_EINVAL, "NULL plan/output");
  if (p->spec.mode != NF_OVERLAP) return set_error(NF_EINVAL, "not an OVERLAP plan");
  if (n_sm != num_sms()) return set_error(NF_EINVAL, "n_sm %d != device SMs %d", n_sm, num_sms());
  NF_TRY(ensure_runtime(p));
  cudaStream_t cs = (cudaStream_t)stream;
  LayerCtx L{};
  L.p = p;
  L.c = &p->cfg;
  L.cs = cs;
  L.ms = p->mem_stream;
  L.ns = p->cfg.tp_size > 1 ? p->net_stream : cs;
  L.comm = comm;
  NF_TRY(enter_partitions(p, &L, cs));
  comm_fused_step_barrier(comm);
  int* d = nullptr;
  NF_CUDA(cudaMalloc(&d, (size_t)3 * n_sm * sizeof(int)));  // (probe only; not on the forward path)
  NF_CUDA(cudaMemsetAsync(d, 0, (size_t)3 * n_sm * sizeof(int), cs));
  NF_CUDA(cudaStreamSynchronize(cs));
  const cudaStream_t parts[3] = {L.dec_on_cs ? nullptr : L.ms, L.cs, (L.ns != L.cs) ? L.ns : nullptr};
  for (int i = 0; i < 3; ++i)
    if (parts[i]) NF_CUDA(launch_smid_probe(d + i * n_sm, 4 * n_sm, parts[i]));
  NF_TRY(leave_partitions(p, L, cs));
  for (int i = 0; i < 3; ++i)
    if (parts[i]) NF_CUDA(cudaStreamSynchronize(parts[i]));
  NF_CUDA(cudaStreamSynchronize(cs));
  NF_CUDA(cudaMemcpy(smids_out, d, (size_t)3 * n_sm * sizeof(int), cudaMemcpyDeviceToHost));
  NF_CUDA(cudaFree(d));
  return NF_OK;
}

nf_status nf_moe_last_ids(const nf_model_cfg* c, const nf_batch* b, const void* ws, size_t ws_bytes,
                          const int32_t** ids_out) {
  NF_TRY(validate_cfg(c));
  NF_TRY(validate_batch(c, b));
  if (c->n_experts <= 0) return set_error(NF_EINVAL, "not a MoE model");
  if (!ws || !ids_out) return set_error(NF_EINVAL, "NULL pointer");
  Workspace w = carve_workspace(c, b, const_cast<void*>(ws));
  if (ws_bytes < w.total) return set_error(NF_EINVAL, "workspace %zu bytes < required %zu", ws_bytes, w.total);
  *ids_out = w.mo_ids;
  return NF_OK;
}

nf_status nf_assemble_tokens(const int32_t* tok_src, const int32_t* prev_next_ids, int32_t* token_ids, int32_t T,
                             void* stream) {
  if (T < 0 || (T > 0 && (!tok_src || !token_ids))) return set_error(NF_EINVAL, "bad arguments");
  NF_CUDA(launch_assemble_tokens(tok_src, prev_next_ids, token_ids, T, (cudaStream_t)stream));
  return NF_OK;
}

// ------------------------------------------------------------------ op-level entry points
nf_status nf_gemm_bf16(const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc, int32_t M,
                       int32_t N, int32_t K, int32_t sm_budget, void* ws, size_t ws_bytes, void* stream) {
  if (!A || !B || !C) return set_error(NF_EINVAL, "NULL pointer");
  if (M < 0 || N <= 0 || K <= 0) return set_error(NF_EINVAL, "bad shape M=%d N=%d K=%d", M, N, K);
  if (N % 32) return set_error(NF_EINVAL, "N must be a multiple of 32");
  if (lda % 8 || ldb % 8 || ldc % 8 || lda < K || ldb < K || ldc < N) return set_error(NF_EINVAL, "bad leading dimension");
  if (((uintptr_t)A | (uintptr_t)B | (uintptr_t)C) & 15) return set_error(NF_EINVAL, "pointers must be 16-byte aligned");
  GemmArgs a{};
  a.epi = EPI_STORE;
  a.M = M;
  a.N = N;
  a.K = K;
  a.n_valid = N;
  a.out = (__nv_bfloat16*)C;
  a.ldo = ldc;
  {
    // (dev) NF_GEMM_EPI=resid times the residual epilogue: C = C + A.B^T, in place
    static int epi_env = -1;
    if (epi_env < 0) {
      const char* e = getenv("NF_GEMM_EPI");
      epi_env = (e && std::string(e) == "resid") ? 1 : 0;
    }
    if (epi_env == 1) {
      a.epi = EPI_RESID;
      a.resid = (const __nv_bfloat16*)C;
      a.ldr = ldc;
    }
  }
  const int grid_max = std::max(1, std::min<int>(sm_budget, num_sms()));
  const int tiles = ((M + GEMM_BM - 1) / GEMM_BM) * ((N + 127) / 128);
  const int slots = std::max(148, ((M + GEMM_BM - 1) / GEMM_BM) * ((N + 255) / 256));
  if (ws) {
    if (ws_bytes < gemm_sk_bytes(slots, tiles)) return set_error(NF_EINVAL, "gemm workspace too small");
    if ((uintptr_t)ws & 255) return set_error(NF_EINVAL, "gemm workspace must be 256-byte aligned");
    a.sk_part = (float*)ws;
    a.sk_slots = slots;
    a.sk_flag = (int*)((char*)ws + (size_t)slots * GEMM_BM * GEMM_SK_LD * 4);
    // (dev) NF_GEMM_NOZERO=1: the caller zeroed the workspace once (the kernel leaves its arrival
    // flags zeroed), so no memset node sits between back-to-back launches in a graph -- GEMM to
    // GEMM as in the model step, whose flags are cleared once per step (tools/gemm_phases.py)
    static int nozero_env = -1;
    if (nozero_env < 0) {
      const char* e = getenv("NF_GEMM_NOZERO");
      nozero_env = e ? atoi(e) : 0;
    }
    if (!nozero_env) NF_CUDA(cudaMemsetAsync(a.sk_flag, 0, (size_t)tiles * 4, (cudaStream_t)stream));
  }
  NF_CUDA(launch_gemm((const __nv_bfloat16*)A, lda, (const __nv_bfloat16*)B, ldb, a, grid_max, (cudaStream_t)stream));
  return NF_OK;
}

size_t nf_gemm_workspace_bytes(int32_t M, int32_t N) {
  const int tiles = ((M + GEMM_BM - 1) / GEMM_BM) * ((N + 127) / 128);
  const int slots = std::max(148, ((M + GEMM_BM - 1) / GEMM_BM) * ((N + 255) / 256));
  return gemm_sk_bytes(slots, tiles);
}

nf_status nf_attention(const nf_model_cfg* cfg, const nf_batch* b, const void* q, const void* kv_pool, void* o, void* ws,
                       size_t ws_bytes, int32_t sm_decode, int32_t sm_prefill, void* stream) {
  NF_TRY(validate_cfg(cfg));
  NF_TRY(validate_batch(cfg, b));
  if (!q || !kv_pool || !o || !ws) return set_error(NF_EINVAL, "NULL pointer");
  Workspace wsp = carve_workspace(cfg, b, ws);
  if (ws_bytes < wsp.total) return set_error(NF_EINVAL, "workspace %zu bytes < required %zu", ws_bytes, wsp.total);
  static thread_local nf_plan* tmp = nullptr;
  if (!tmp) {
    tmp = new nf_plan();
    tmp->spec.n_nano = 1;
    tmp->spec.share[0] = 1;
  }
  tmp->cfg = *cfg;
  for (int k = 0; k < NF_OP_COUNT; ++k) tmp->spec.sm[k] = num_sms();
  tmp->spec.sm[NF_OP_DECODE_ATTN] = std::max(1, sm_decode);
  tmp->spec.sm[NF_OP_PREFILL_ATTN] = std::max(1, sm_prefill);
  NF_TRY(ensure_runtime(tmp));
  std::vector<int> order(b->n_req);
  std::iota(order.begin(), order.end(), 0);
  StepMeta m;
  build_meta(cfg, b, order, {0, b->n_req}, &m);
  cudaStream_t st = (cudaStream_t)stream;
  NF_TRY(upload_meta(tmp, m, wsp.meta, st));
  Workspace w2 = wsp;
  w2.q = (__nv_bfloat16*)q;
  w2.o = (__nv_bfloat16*)o;
  LayerCtx L{};
  L.p = tmp;
  L.c = cfg;
  L.m = &m;
  L.w = &w2;
  L.meta_dev = wsp.meta;
  NF_CUDA(make_pool_tmap(&L.pool_map, kv_pool, b->n_pages_pool, cfg->n_kv_heads / cfg->tp_size, cfg->head_dim,
                         cfg->page_size));
  NF_CUDA(make_page_tmap(&L.page_map, kv_pool, b->n_pages_pool, cfg->n_kv_heads / cfg->tp_size, cfg->head_dim,
                         cfg->page_size));
  NF_TRY(run_attn(L, m.nanos[0], st));
  return NF_OK;
}

}  // extern "C"
