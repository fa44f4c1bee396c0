// Global batch scheduler + KV-cache manager of the serving loop (SURVEY.md §8f
// NEXT-4): continuous batching with chunked prefill, discrete
// dense batch sizes, peak-memory admission with eviction on
// exhaustion, asynchronous EOS detection one step late
// (PAPER.md:652-657).  Readings A-25..A-29; the bit-exact contract
// is oracle/serving.py.  Host-only: it runs while the GPU executes the
// previous step, so its cost is hidden behind the step.
#include <algorithm>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <set>
#include <unordered_map>
#include <vector>

#include "host.h"

namespace nf {
namespace {

struct Req {
  int64_t id;
  std::vector<int32_t> prompt;
  int32_t out_len;
  int64_t order;
  int32_t prefilled = 0, generated = 0;
  std::vector<int32_t> pages;
  int32_t last_tok = -1;
  bool has_last_tok = false;
  int64_t last_step = -1;
  int32_t last_row = -1;
  bool finished = false;
  int64_t admit_seq = -1;
  void reset() {
    prefilled = generated = 0;
    pages.clear();
    has_last_tok = false;
    last_tok = -1;
    last_step = -1;
    last_row = -1;
    finished = false;
    admit_seq = -1;
  }
};

struct Item {
  Req* r;
  int32_t q, kv, emit;
};

}  // namespace
}  // namespace nf

struct nf_sched {
  nf_sched_cfg cfg{};
  std::vector<int32_t> bdense;  // descending, unique
  std::set<int32_t> free_pages;
  std::deque<nf::Req*> queue;
  std::vector<nf::Req*> running;  // admission order
  std::unordered_map<int64_t, std::unique_ptr<nf::Req>> by_id;
  int64_t n_submitted = 0, admit_counter = 0, step_no = 0;
  std::map<int64_t, std::vector<std::pair<nf::Req*, int32_t>>> pending;  // step -> (req, generated after)
  nf_sched_stats st{};
  // storage of the last formed step
  std::vector<int64_t> o_ids;
  std::vector<int32_t> o_q, o_kv, o_emit, o_indptr, o_pages, o_src;
};

namespace nf {
namespace {

int64_t peak_pages(const nf_sched* s, const std::vector<Req*>& reqs, const Req* extra) {
  // max_j floor(sum_{r: tau_r >= tau_j} (L_r + tau_j + page - 1) / page)   (reading A-27)
  std::vector<std::pair<int64_t, int64_t>> it;  // (tau, L)
  it.reserve(reqs.size() + 1);
  auto add = [&](const Req* r) {
    it.push_back({std::max<int64_t>((int64_t)s->cfg.avg_decode - r->generated, 1),
                  (int64_t)r->prompt.size() + r->generated});
  };
  for (const Req* r : reqs) add(r);
  if (extra) add(extra);
  std::sort(it.begin(), it.end(), [](auto& a, auto& b) { return a.first > b.first; });
  const int64_t P = s->cfg.page_size;
  int64_t best = 0, cnt = 0, sumL = 0;
  size_t i = 0;
  while (i < it.size()) {
    const int64_t tau = it[i].first;
    while (i < it.size() && it[i].first == tau) {
      sumL += it[i].second;
      ++cnt;
      ++i;
    }
    best = std::max(best, (sumL + cnt * (tau + P - 1)) / P);
  }
  return best;
}

std::vector<Item> compose(nf_sched* s) {
  std::vector<Req*> dec;
  int64_t avail = 0;
  for (Req* r : s->running) {
    if (r->prefilled == (int32_t)r->prompt.size()) dec.push_back(r);
    avail += (int64_t)r->prompt.size() - r->prefilled;
  }
  avail += (int64_t)dec.size();
  int64_t B = avail;
  for (int32_t b : s->bdense)
    if (b <= avail) {
      B = b;
      break;
    }
  if (B < (int64_t)dec.size()) B = std::min<int64_t>((int64_t)dec.size(), s->bdense.front());  // decodes never wait
  std::vector<Item> comp;
  const int64_t nd = std::min<int64_t>((int64_t)dec.size(), B);
  for (int64_t i = 0; i < nd; ++i) {
    Req* r = dec[i];
    comp.push_back({r, 1, (int32_t)r->prompt.size() + r->generated - 1, 1});
  }
  int64_t budget = B - nd;
  for (Req* r : s->running) {
    if (budget == 0) break;
    const int64_t rem = (int64_t)r->prompt.size() - r->prefilled;
    if (rem > 0) {
      const int64_t c = std::min(rem, budget);
      comp.push_back({r, (int32_t)c, r->prefilled, c == rem ? 1 : 0});
      budget -= c;
    }
  }
  return comp;
}

void release(nf_sched* s, Req* r) {
  for (int32_t p : r->pages) s->free_pages.insert(p);
  r->pages.clear();
}

// Allocates the step's new pages (lowest free id first); on exhaustion returns the
// most recently admitted running request (nothing allocated).
Req* allocate(nf_sched* s, const std::vector<Item>& comp) {
  const int64_t P = s->cfg.page_size;
  int64_t need_total = 0;
  for (const Item& it : comp)
    need_total += std::max<int64_t>(0, ((int64_t)it.kv + it.q + P - 1) / P - (int64_t)it.r->pages.size());
  if (need_total <= (int64_t)s->free_pages.size()) {
    for (const Item& it : comp) {
      const int64_t need = ((int64_t)it.kv + it.q + P - 1) / P - (int64_t)it.r->pages.size();
      for (int64_t j = 0; j < need; ++j) {
        auto b = s->free_pages.begin();
        it.r->pages.push_back(*b);
        s->free_pages.erase(b);
      }
    }
    const int32_t used = s->cfg.n_pages - (int32_t)s->free_pages.size();
    s->st.peak_pages_used = std::max(s->st.peak_pages_used, used);
    return nullptr;
  }
  Req* v = nullptr;
  for (Req* r : s->running)
    if (!v || r->admit_seq > v->admit_seq) v = r;
  return v;
}

void evict(nf_sched* s, Req* r) {
  release(s, r);
  s->running.erase(std::find(s->running.begin(), s->running.end(), r));
  for (auto& kv : s->pending)
    for (auto& e : kv.second)
      if (e.first == r) e = {nullptr, 0};
  r->reset();
  s->queue.push_front(r);
  s->st.evictions++;
}

}  // namespace
}  // namespace nf

using namespace nf;

extern "C" {

nf_status nf_sched_create(const nf_sched_cfg* cfg, nf_sched** out) {
  if (!cfg || !out) return set_error(NF_EINVAL, "NULL argument");
  if (cfg->n_pages < 1 || cfg->page_size < 1 || cfg->avg_decode < 1 || cfg->n_bdense < 1 || cfg->n_bdense > 16 ||
      !cfg->bdense)
    return set_error(NF_EINVAL, "bad scheduler config");
  auto s = std::make_unique<nf_sched>();
  s->cfg = *cfg;
  for (int i = 0; i < cfg->n_bdense; ++i) {
    if (cfg->bdense[i] < 1) return set_error(NF_EINVAL, "bdense[%d] = %d < 1", i, cfg->bdense[i]);
    s->bdense.push_back(cfg->bdense[i]);
  }
  std::sort(s->bdense.begin(), s->bdense.end(), std::greater<int32_t>());
  s->bdense.erase(std::unique(s->bdense.begin(), s->bdense.end()), s->bdense.end());
  s->cfg.bdense = nullptr;
  for (int32_t p = 0; p < cfg->n_pages; ++p) s->free_pages.insert(s->free_pages.end(), p);
  *out = s.release();
  return NF_OK;
}

void nf_sched_destroy(nf_sched* s) { delete s; }

nf_status nf_sched_submit(nf_sched* s, int64_t req_id, const int32_t* prompt, int32_t prompt_len, int32_t out_len) {
  if (!s || !prompt) return set_error(NF_EINVAL, "NULL argument");
  if (prompt_len < 1 || out_len < 1) return set_error(NF_EINVAL, "prompt_len %d / out_len %d < 1", prompt_len, out_len);
  if (s->by_id.count(req_id)) return set_error(NF_EINVAL, "duplicate request id %lld", (long long)req_id);
  auto r = std::make_unique<Req>();
  r->id = req_id;
  r->prompt.assign(prompt, prompt + prompt_len);
  r->out_len = out_len;
  r->order = s->n_submitted++;
  s->queue.push_back(r.get());
  s->by_id[req_id] = std::move(r);
  return NF_OK;
}

nf_status nf_sched_next(nf_sched* s, nf_sched_step* out) {
  if (!s || !out) return set_error(NF_EINVAL, "NULL argument");
  // 1. retire requests whose EOS was read back
  for (size_t i = 0; i < s->running.size();) {
    Req* r = s->running[i];
    if (r->finished) {
      release(s, r);
      s->running.erase(s->running.begin() + i);
    } else {
      ++i;
    }
  }
  // 2. FCFS admission under the peak-memory estimate
  while (!s->queue.empty()) {
    Req* c = s->queue.front();
    if (peak_pages(s, s->running, c) > s->cfg.n_pages) break;
    s->queue.pop_front();
    c->admit_seq = s->admit_counter++;
    s->running.push_back(c);
  }
  // 3-4. compose, allocate pages, evict on exhaustion
  std::vector<Item> comp;
  for (;;) {
    comp = compose(s);
    Req* v = allocate(s, comp);
    if (!v) break;
    evict(s, v);
  }
  // 5. emit the step (bookkeeping as if it runs)
  s->o_ids.clear();
  s->o_q.clear();
  s->o_kv.clear();
  s->o_emit.clear();
  s->o_indptr.assign(1, 0);
  s->o_pages.clear();
  s->o_src.clear();
  const int64_t step = s->step_no, prev = step - 1;
  std::vector<std::pair<Req*, int32_t>> rows;
  for (size_t row = 0; row < comp.size(); ++row) {
    const Item& it = comp[row];
    Req* r = it.r;
    const int32_t plen = (int32_t)r->prompt.size();
    s->o_ids.push_back(r->id);
    s->o_q.push_back(it.q);
    s->o_kv.push_back(it.kv);
    s->o_pages.insert(s->o_pages.end(), r->pages.begin(), r->pages.end());
    s->o_indptr.push_back((int32_t)s->o_pages.size());
    s->o_emit.push_back(it.emit);
    const bool decode = it.q == 1 && it.kv >= plen;
    if (decode) {
      if (r->last_step >= 0 && s->pending.count(r->last_step)) {
        if (r->last_step != prev)
          return set_error(NF_EINVAL, "step %lld not completed before forming step %lld", (long long)r->last_step,
                           (long long)step + 1);
        s->o_src.push_back(-(1 + r->last_row));
      } else {
        s->o_src.push_back(r->last_tok);
      }
      s->st.decode_tokens++;
    } else {
      s->o_src.insert(s->o_src.end(), r->prompt.begin() + it.kv, r->prompt.begin() + it.kv + it.q);
      r->prefilled += it.q;
      s->st.prefill_tokens += it.q;
    }
    if (it.emit) {
      r->generated++;
      r->last_step = step;
      r->last_row = (int32_t)row;
      s->st.generated++;
      if (r->generated > r->out_len) s->st.useless++;
      rows.push_back({r, r->generated});
    } else {
      rows.push_back({nullptr, 0});
    }
  }
  s->pending[step] = std::move(rows);
  s->st.steps++;
  int64_t ntok = 0;
  for (int32_t q : s->o_q) ntok += q;
  s->st.tokens += ntok;
  s->step_no++;
  out->step = step;
  out->n_req = (int32_t)s->o_ids.size();
  out->n_tokens = (int32_t)ntok;
  out->req_ids = s->o_ids.data();
  out->q_len = s->o_q.data();
  out->kv_prefix = s->o_kv.data();
  out->emit = s->o_emit.data();
  out->page_indptr = s->o_indptr.data();
  out->page_ids = s->o_pages.data();
  out->tok_src = s->o_src.data();
  return NF_OK;
}

nf_status nf_sched_complete(nf_sched* s, int64_t step, const int32_t* next_ids) {
  if (!s) return set_error(NF_EINVAL, "NULL scheduler");
  auto itp = s->pending.find(step);
  if (itp == s->pending.end()) return set_error(NF_EINVAL, "step %lld is not pending", (long long)step);
  if (!next_ids && !itp->second.empty()) return set_error(NF_EINVAL, "next_ids is NULL");
  const auto rows = std::move(itp->second);
  s->pending.erase(itp);
  for (size_t row = 0; row < rows.size(); ++row) {
    Req* r = rows[row].first;
    if (!r) continue;
    const int32_t tok = next_ids[row];
    if (r->last_step == step) {
      r->last_tok = tok;
      r->has_last_tok = true;
    }
    if (!r->finished && (rows[row].second == r->out_len || (s->cfg.eos_id >= 0 && tok == s->cfg.eos_id))) {
      r->finished = true;
      s->st.finished++;
    }
  }
  return NF_OK;
}

nf_status nf_sched_get_stats(const nf_sched* s, nf_sched_stats* out) {
  if (!s || !out) return set_error(NF_EINVAL, "NULL argument");
  *out = s->st;
  out->running = (int32_t)s->running.size();
  out->queued = (int32_t)s->queue.size();
  return NF_OK;
}

}  // extern "C"
