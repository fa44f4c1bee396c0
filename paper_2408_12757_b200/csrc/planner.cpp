// Automatic parameter search: critical-path greedy SM
// assignment per candidate nano-batch split over measured kernel curves,
// keeping the split with the shortest pipeline makespan.  Host-only,
// deterministic.  Readings P-1..P-7 of DESIGN.md ("Planner").
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <map>
#include <set>
#include <string>
#include <vector>

#include "host.h"

namespace nf {
namespace {

struct PNode {
  int kind, nano;
  double work;
  std::vector<int> deps;
};

// latency(kind, units, work) from measured samples (reading P-2)
class CurveSet {
 public:
  std::map<int, std::map<double, std::vector<std::pair<int, double>>>> by;
  void add(int kind, int units, double work, double lat) { by[kind][work].push_back({units, lat}); }
  void finish() {
    for (auto& k : by)
      for (auto& w : k.second) std::sort(w.second.begin(), w.second.end());
  }
  bool has(int kind) const { return by.count(kind) > 0; }
  double at_work(const std::vector<std::pair<int, double>>& pts, int u) const {
    if (u <= pts.front().first) return pts.front().second * pts.front().first / u;
    if (u >= pts.back().first) return pts.back().second;
    for (size_t i = 0; i + 1 < pts.size(); ++i) {
      const int u0 = pts[i].first, u1 = pts[i + 1].first;
      if (u0 <= u && u <= u1) {
        const double l0 = pts[i].second, l1 = pts[i + 1].second;
        return l0 + (l1 - l0) * (u - u0) / (u1 - u0);
      }
    }
    return pts.back().second;
  }
  double latency(int kind, int u, double work) const {
    if (work <= 0) return 0.0;
    const auto& ws = by.at(kind);
    const double w_lo = ws.begin()->first, w_hi = ws.rbegin()->first;
    if (work <= w_lo) return at_work(ws.begin()->second, u) * work / w_lo;
    if (work >= w_hi) return at_work(ws.rbegin()->second, u) * work / w_hi;
    auto it1 = ws.lower_bound(work);
    if (it1->first == work) return at_work(it1->second, u);
    auto it0 = std::prev(it1);
    const double l0 = at_work(it0->second, u), l1 = at_work(it1->second, u);
    return l0 + (l1 - l0) * (work - it0->first) / (it1->first - it0->first);
  }
};

struct Sched {
  double makespan;
  std::vector<double> start, end;
};

// list scheduling (reading P-3): at each event time, start every ready node
// whose units fit the free capacity in (rank, id) order
Sched simulate(const std::vector<PNode>& g, const std::vector<int>& rank_order, const int* units, const CurveSet& cv,
               int budget) {
  const int n = (int)g.size();
  Sched s;
  s.start.assign(n, -1.0);
  s.end.assign(n, -1.0);
  std::vector<double> dur(n);
  for (int i = 0; i < n; ++i) dur[i] = cv.latency(g[i].kind, units[g[i].kind], g[i].work);
  std::vector<char> done(n, 0);
  std::vector<int> running;
  int free_units = budget, n_done = 0;
  double t = 0.0;
  while (n_done < n) {
    for (int i : rank_order) {
      if (s.start[i] >= 0) continue;
      bool ready = true;
      for (int d : g[i].deps)
        if (!done[d]) { ready = false; break; }
      if (!ready) continue;
      const int need = units[g[i].kind];
      if (need <= free_units) {
        s.start[i] = t;
        s.end[i] = t + dur[i];
        free_units -= need;
        running.push_back(i);
      }
    }
    if (running.empty()) {
      s.makespan = INFINITY;
      return s;
    }
    double tn = INFINITY;
    for (int i : running) tn = std::min(tn, s.end[i]);
    t = tn;
    std::sort(running.begin(), running.end());
    std::vector<int> keep;
    for (int i : running) {
      if (s.end[i] <= t) {
        done[i] = 1;
        free_units += units[g[i].kind];
        ++n_done;
      } else {
        keep.push_back(i);
      }
    }
    running.swap(keep);
  }
  s.makespan = *std::max_element(s.end.begin(), s.end.end());
  return s;
}

// longest duration-weighted chain ending at the node that ends last (reading P-4)
std::vector<int> critical_path(const std::vector<PNode>& g, const Sched& s) {
  const int n = (int)g.size();
  std::vector<double> best(n, 0.0);
  std::vector<int> pred(n, -1);
  for (int i = 0; i < n; ++i) {
    double b = 0.0;
    int p = -1;
    std::vector<int> deps = g[i].deps;
    std::sort(deps.begin(), deps.end());
    for (int d : deps)
      if (best[d] > b) { b = best[d]; p = d; }
    best[i] = b + (s.end[i] - s.start[i]);
    pred[i] = p;
  }
  int last = 0;
  for (int i = 1; i < n; ++i)
    if (s.end[i] > s.end[last]) last = i;
  std::vector<int> path;
  for (int v = last; v >= 0; v = pred[v]) path.push_back(v);
  std::reverse(path.begin(), path.end());
  return path;
}

struct Result {
  std::vector<int> units;
  Sched sched;
};

Result local_search(const std::vector<PNode>& g, const std::vector<int>& order, const CurveSet& cv, int budget, int q,
                    std::vector<int> units, int max_iters) {
  std::set<int> used_set;
  for (const auto& nd : g) used_set.insert(nd.kind);
  const std::vector<int> used(used_set.begin(), used_set.end());
  Sched cur = simulate(g, order, units.data(), cv, budget);
  for (int it = 0; it < max_iters; ++it) {
    std::set<int> crit;
    for (int v : critical_path(g, cur)) crit.insert(g[v].kind);
    bool found = false;
    double cand_m = 0.0;
    std::vector<int> cand_u;
    Sched cand_s;
    for (int c : crit) {
      std::vector<int> donors{-1};
      for (int k : used)
        if (k != c) donors.push_back(k);
      for (int d : donors) {
        std::vector<int> u = units;
        if (d < 0) {
          if (u[c] + q > budget) continue;
          u[c] += q;
        } else {
          if (u[d] - q < q || u[c] + q > budget) continue;
          u[d] -= q;
          u[c] += q;
        }
        Sched s = simulate(g, order, u.data(), cv, budget);
        if (s.makespan < cur.makespan - 1e-15 && (!found || s.makespan < cand_m - 1e-15)) {
          found = true;
          cand_m = s.makespan;
          cand_u = u;
          cand_s = s;
        }
      }
    }
    if (!found) break;
    units = cand_u;
    cur = cand_s;
  }
  return Result{units, cur};
}

// the executor's OVERLAP schedule (api.cu nf_model_step) as a DAG over n_layers layers:
// decode attention on the memory stream, prefill attention on the compute stream (A-11)
std::vector<PNode> build_pipeline(const std::vector<std::array<double, 3>>& work, int n_layers) {
  std::vector<PNode> g;
  auto add = [&](int kind, int nano, double w, std::vector<int> deps) {
    PNode nd;
    nd.kind = kind;
    nd.nano = nano;
    nd.work = w;
    for (int d : deps)
      if (d >= 0) nd.deps.push_back(d);
    g.push_back(nd);
    return (int)g.size() - 1;
  };
  const int K = (int)work.size();
  int last_c = -1, last_m = -1;
  std::vector<int> dec(K, -1);
  for (int k = 0; k < K; ++k) {
    const int kq = add(NF_OP_KQV, k, work[k][0], {last_c});
    dec[k] = add(NF_OP_DECODE_ATTN, k, work[k][1], {kq, last_m});
    last_m = dec[k];
    last_c = add(NF_OP_PREFILL_ATTN, k, work[k][2], {kq});
  }
  for (int l = 0; l < n_layers; ++l) {
    for (int k = 0; k < K; ++k) {
      const int o = add(NF_OP_O, k, work[k][0], {dec[k], last_c});
      const int ug = add(NF_OP_UG, k, work[k][0], {o});
      const int dn = add(NF_OP_DOWN, k, work[k][0], {ug});
      last_c = dn;
      if (l + 1 < n_layers) {
        const int kq = add(NF_OP_KQV, k, work[k][0], {dn});
        dec[k] = add(NF_OP_DECODE_ATTN, k, work[k][1], {kq, last_m});
        last_m = dec[k];
        last_c = add(NF_OP_PREFILL_ATTN, k, work[k][2], {kq});
      }
    }
  }
  return g;
}

// The tensor-parallel pipeline (reading P-8): quarters Q1..Q4 for
// KQV / attention, H1 = Q1+Q2 (column O + AllGathers), H2 = Q3+Q4 (row O + AllReduce);
// NET work = AllGather-equivalent tokens (an AllReduce counts twice its tokens).
std::vector<PNode> build_pipeline_tp(const std::vector<std::array<double, 3>>& work, int n_layers) {
  std::vector<PNode> g;
  auto add = [&](int kind, int nano, double w, std::vector<int> deps) {
    PNode nd;
    nd.kind = kind;
    nd.nano = nano;
    nd.work = w;
    for (int d : deps)
      if (d >= 0) nd.deps.push_back(d);
    g.push_back(nd);
    return (int)g.size() - 1;
  };
  int last_c = -1, last_m = -1, last_n = -1;
  int dec[4] = {-1, -1, -1, -1}, pf[4] = {-1, -1, -1, -1}, ready[2] = {-1, -1};
  const double tok[2] = {work[0][0] + work[1][0], work[2][0] + work[3][0]};
  auto front = [&](int gi) {
    for (int q = 2 * gi; q < 2 * gi + 2; ++q) {
      const int kq = add(NF_OP_KQV, q, work[q][0], {last_c, ready[gi]});
      dec[q] = add(NF_OP_DECODE_ATTN, q, work[q][1], {kq, last_m});
      last_m = dec[q];
      pf[q] = add(NF_OP_PREFILL_ATTN, q, work[q][2], {kq});
      last_c = pf[q];
    }
  };
  front(0);
  front(1);
  for (int l = 0; l < n_layers; ++l) {
    const int ag_a = add(NF_OP_NET, 0, tok[0], {dec[0], dec[1], pf[1], last_n});
    last_n = ag_a;
    const int o1 = add(NF_OP_O, 0, tok[0], {ag_a, last_c});
    last_c = o1;
    const int ag_o = add(NF_OP_NET, 0, tok[0], {o1, last_n});
    last_n = ag_o;
    const int o2 = add(NF_OP_O, 1, tok[1], {dec[2], dec[3], last_c});
    last_c = o2;
    const int ar_o = add(NF_OP_NET, 1, 2 * tok[1], {o2, last_n});
    last_n = ar_o;
    const int ug1 = add(NF_OP_UG, 0, tok[0], {ag_o, last_c});
    const int d1 = add(NF_OP_DOWN, 0, tok[0], {ug1});
    last_c = d1;
    const int ar_d1 = add(NF_OP_NET, 0, 2 * tok[0], {d1, last_n});
    last_n = ar_d1;
    const int ug2 = add(NF_OP_UG, 1, tok[1], {ar_o, last_c});
    const int d2 = add(NF_OP_DOWN, 1, tok[1], {ug2});
    last_c = d2;
    const int ar_d2 = add(NF_OP_NET, 1, 2 * tok[1], {d2, last_n});
    last_n = ar_d2;
    ready[0] = ar_d1;
    ready[1] = ar_d2;
    if (l + 1 < n_layers) {
      front(0);
      front(1);
    }
  }
  return g;
}

std::vector<int> rank_order(const std::vector<PNode>& g) {
  const int n = (int)g.size();
  std::vector<int> rank(n, 0), order(n);
  for (int i = 0; i < n; ++i)
    for (int d : g[i].deps) rank[i] = std::max(rank[i], rank[d] + 1);
  for (int i = 0; i < n; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return rank[a] < rank[b]; });
  return order;
}

std::vector<int> initial_units(const std::vector<PNode>& g, const CurveSet& cv, int budget, int q) {
  double tot[NF_OP_COUNT] = {0};
  for (const auto& nd : g) tot[nd.kind] += cv.latency(nd.kind, budget, nd.work);
  double s = 0;
  for (double v : tot) s += v;
  std::vector<int> u(NF_OP_COUNT);
  for (int k = 0; k < NF_OP_COUNT; ++k) {
    int v = s > 0 ? (int)(budget * tot[k] / s) / q * q : budget;
    u[k] = std::max(q, v);
  }
  return u;
}

const char* kind_name(int k) {
  static const char* n[] = {"KQV", "DecodeAttn", "PrefillAttn", "O", "UGD_up_gate", "Down", "Net"};
  return k >= 0 && k < NF_OP_COUNT ? n[k] : "?";
}

}  // namespace
}  // namespace nf

using namespace nf;

extern "C" nf_status nf_plan_create(const nf_model_cfg* cfg, const nf_batch* shape, const nf_curve_point* pts,
                                    int32_t n_pts, const nf_plan_opts* opts, nf_plan** out) {
  NF_TRY(validate_cfg(cfg));
  NF_TRY(validate_batch(cfg, shape));
  if (!opts || !out) return set_error(NF_EINVAL, "NULL opts/out");
  if (opts->sm_budget < 1 || opts->sm_quantum < 1 || opts->sm_quantum > opts->sm_budget)
    return set_error(NF_EINVAL, "bad sm_budget/sm_quantum");
  if (opts->mode < NF_SEQUENTIAL || opts->mode > NF_OVERLAP) return set_error(NF_EINVAL, "bad mode");
  const bool tp = cfg->tp_size > 1;
  const int budget = opts->sm_budget, q = opts->sm_quantum, iters = std::max(0, opts->max_iters);
  nf_plan_spec spec{};
  spec.mode = opts->mode;
  spec.n_nano = 1;
  spec.share[0] = 1;
  for (int k = 0; k < NF_OP_COUNT; ++k) spec.sm[k] = budget;
  spec.balance = 1;
  std::string csv = "node_id,kind,nano_index,units,start_s,end_s\n";
  if (opts->mode != NF_SEQUENTIAL) {
    if (!pts || n_pts < 1) return set_error(NF_EINVAL, "no curve points");
    CurveSet cv;
    for (int i = 0; i < n_pts; ++i) {
      if (pts[i].op_kind < 0 || pts[i].op_kind >= NF_OP_COUNT) return set_error(NF_EINVAL, "curve op_kind out of range");
      if (pts[i].units < 1 || !(pts[i].work > 0) || !(pts[i].latency_s >= 0))
        return set_error(NF_EINVAL, "curve point %d out of range", i);
      cv.add(pts[i].op_kind, pts[i].units, pts[i].work, pts[i].latency_s);
    }
    cv.finish();
    // single-GPU pipeline: two nano-batches; TP: four attention quarters
    // grouped into two dense halves (reading P-8)
    const int nn = tp ? 4 : 2;
    bool have = false;
    double best_m = 0.0;
    int best_s = 0;
    std::vector<int> best_u;
    std::vector<PNode> best_g;
    Sched best_sched;
    for (int s8 = 1; s8 <= 7; ++s8) {
      const int32_t sh[4] = {s8, tp ? s8 : 8 - s8, 8 - s8, 8 - s8};
      std::vector<std::vector<int>> grp;
      balance_requests(shape, nn, sh, &grp);
      std::vector<std::array<double, 3>> work;
      for (const auto& gr : grp) {
        double tok = 0, dk = 0, pk = 0;
        for (int r : gr) {
          tok += shape->q_len[r];
          if (shape->q_len[r] == 1) {
            dk += shape->kv_prefix[r] + 1;
          } else {
            for (int i = 0; i < shape->q_len[r]; ++i) pk += shape->kv_prefix[r] + i + 1;
          }
        }
        work.push_back({tok, dk, pk});
      }
      std::vector<PNode> g = tp ? build_pipeline_tp(work, 3) : build_pipeline(work, 3);
      for (const auto& nd : g)
        if (nd.work > 0 && !cv.has(nd.kind))
          return set_error(NF_EINVAL, "no curve for op kind %d (%s)", nd.kind, kind_name(nd.kind));
      const std::vector<int> order = rank_order(g);
      Result r1 = local_search(g, order, cv, budget, q, initial_units(g, cv, budget, q), iters);
      Result r2 = local_search(g, order, cv, budget, q, std::vector<int>(NF_OP_COUNT, budget), iters);
      Result& r = r2.sched.makespan < r1.sched.makespan - 1e-15 ? r2 : r1;
      if (!std::isfinite(r.sched.makespan)) continue;
      if (!have || r.sched.makespan < best_m - 1e-15) {
        have = true;
        best_m = r.sched.makespan;
        best_s = s8;
        best_u = r.units;
        best_g = g;
        best_sched = r.sched;
      }
    }
    if (!have) return set_error(NF_EINFEASIBLE, "no candidate split fits the SM budget");
    spec.n_nano = nn;
    if (tp) {
      spec.n_dense = 2;
      spec.share[0] = spec.share[1] = best_s;
      spec.share[2] = spec.share[3] = 8 - best_s;
      spec.balance = 2;
    } else {
      spec.share[0] = best_s;
      spec.share[1] = 8 - best_s;
    }
    for (int k = 0; k < NF_OP_COUNT; ++k) spec.sm[k] = std::max(1, best_u[k]);
    char line[160];
    for (size_t i = 0; i < best_g.size(); ++i) {
      snprintf(line, sizeof(line), "%zu,%s,%d,%d,%.9g,%.9g\n", i, kind_name(best_g[i].kind), best_g[i].nano,
               best_u[best_g[i].kind], best_sched.start[i], best_sched.end[i]);
      csv += line;
    }
  }
  nf_status st = nf_plan_create_explicit(cfg, &spec, out);
  if (st != NF_OK) return st;
  (*out)->csv = csv;
  return NF_OK;
}
