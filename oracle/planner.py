"""Automatic parameter search (§5.6) — test infrastructure only.

Step by step, in the paper's order:
  "autosearch uses topological sorting to find the critical path (the chain
   of dependent operations that takes the longest execution time) and assign
   more SMs to the operators on the critical path ... limits total execution
   unit usage according to the number of SMs ... iteratively identifies new
   critical paths ... After applying the above critical path optimization
   algorithm to all possible combinations of nano-batch sizes, we choose the
   scheduling with the shortest critical path.  The autosearch estimates the
   kernel performance based on offline profiling."

Where the paper is silent we follow SPEC S:369-445 (list scheduling, greedy
moves, deterministic ties) with the readings listed in DESIGN.md
("Planner readings" P-1..P-7):
  P-1 units are assigned per op KIND (the executor applies one SM budget per kind);
  P-2 curve evaluation: piecewise linear in units at fixed work (clamped to the
      sampled range, 1/u scaling below it), linear in work between sampled
      works, proportional to work outside them;
  P-3 list scheduling: at each event time start every ready node whose units
      fit the free capacity, in (topological rank, node id) order;
  P-4 critical path: longest duration-weighted path ending at the node that
      ends last (ties: smallest id), predecessor ties -> smallest id;
  P-5 greedy move set: +q units to a critical kind, or move q units from any
      other kind to a critical kind; best strict makespan improvement wins,
      ties by (receiver, donor) order, "no donor" first;
  P-6 initial units: proportional to each kind's full-budget latency share,
      rounded down to the quantum, at least one quantum; a second greedy run
      starts from the whole budget for every kind (the sequential schedule) and
      the shorter result wins, so the search never returns worse than
      sequential (SPEC S:423 upper bound);
  P-7 candidate splits: nano-batch-0 token share s/8, s = 1..7 (2 nano-batches).
  P-8 tensor parallelism: four KQV/attention nano-batches
      (quarters Q1..Q4) and two dense nano-batches H1 = Q1+Q2 (column O +
      AllGathers) and H2 = Q3+Q4 (row O + AllReduce); candidate splits give H1
      the token share s/8 (s = 1..7), split evenly into its two quarters
      (shares s, s, 8-s, 8-s).  Collectives are NET nodes whose work is the
      AllGather-equivalent token count: an AllGather of the group's rows counts
      its tokens, an AllReduce twice its tokens (a ring AllReduce moves twice
      the bytes of an AllGather of the same buffer, D = Hq*hd rows here).  The
      three streams of the executor add order edges: compute (KQV, prefill,
      O, Up/Gate, Down), memory (decode attention) and network (collectives in
      the fixed issue order AG_attn(H1), AG_o(H1), AR_o(H2), AR_d(H1),
      AR_d(H2) per layer, identical on every rank).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

# op kinds (same numbering as include/nf.h NF_OP_*)
KQV, DECODE, PREFILL, O, UG, DOWN, NET = range(7)
N_KINDS = 7


@dataclass
class Node:
    id: int
    kind: int
    nano: int
    work: float
    deps: List[int] = field(default_factory=list)


class Curves:
    """Measured latency samples per kind: (units, work, latency_s)."""

    def __init__(self, points: Sequence[Tuple[int, int, float, float]]):
        self.by: Dict[int, Dict[float, List[Tuple[int, float]]]] = {}
        for kind, units, work, lat in points:
            self.by.setdefault(int(kind), {}).setdefault(float(work), []).append((int(units), float(lat)))
        for k in self.by:
            for w in self.by[k]:
                self.by[k][w].sort()

    def _at_work(self, kind: int, w: float, u: int) -> float:
        pts = self.by[kind][w]
        if u <= pts[0][0]:
            return pts[0][1] * pts[0][0] / u
        if u >= pts[-1][0]:
            return pts[-1][1]
        for (u0, l0), (u1, l1) in zip(pts, pts[1:]):
            if u0 <= u <= u1:
                return l0 + (l1 - l0) * (u - u0) / (u1 - u0)
        raise AssertionError

    def latency(self, kind: int, units: int, work: float) -> float:
        """Reading P-2."""
        if work <= 0:
            return 0.0
        if kind not in self.by:
            raise KeyError(f"no curve for op kind {kind}")
        ws = sorted(self.by[kind])
        if work in self.by[kind]:
            return self._at_work(kind, work, units)
        if work <= ws[0]:
            return self._at_work(kind, ws[0], units) * work / ws[0]
        if work >= ws[-1]:
            return self._at_work(kind, ws[-1], units) * work / ws[-1]
        for w0, w1 in zip(ws, ws[1:]):
            if w0 <= work <= w1:
                l0, l1 = self._at_work(kind, w0, units), self._at_work(kind, w1, units)
                return l0 + (l1 - l0) * (work - w0) / (w1 - w0)
        raise AssertionError


def topo_rank(nodes: List[Node]) -> List[int]:
    """Longest-chain depth of every node (topological rank)."""
    rank = [0] * len(nodes)
    for n in nodes:  # nodes are created in a topological order (deps have smaller ids)
        for d in n.deps:
            assert d < n.id
            rank[n.id] = max(rank[n.id], rank[d] + 1)
    return rank


def simulate(nodes: List[Node], units: Sequence[int], curves: Curves, budget: int):
    """List scheduling (reading P-3).  Returns (makespan, start, end)."""
    n = len(nodes)
    rank = topo_rank(nodes)
    dur = [curves.latency(nd.kind, units[nd.kind], nd.work) for nd in nodes]
    start = [None] * n
    end = [None] * n
    done = [False] * n
    running: List[int] = []
    free = budget
    t = 0.0
    order = sorted(range(n), key=lambda i: (rank[i], i))
    n_done = 0
    while n_done < n:
        for i in order:
            if start[i] is None and all(done[d] for d in nodes[i].deps):
                need = units[nodes[i].kind]
                if need > budget:
                    raise ValueError("op demands more units than the budget")
                if need <= free:
                    start[i] = t
                    end[i] = t + dur[i]
                    free -= need
                    running.append(i)
        if not running:
            raise RuntimeError("deadlock")
        t = min(end[i] for i in running)
        for i in sorted(running):
            if end[i] <= t:
                running.remove(i)
                done[i] = True
                free += units[nodes[i].kind]
                n_done += 1
    return max(end), start, end


def critical_path(nodes: List[Node], start, end) -> List[int]:
    """Reading P-4: longest duration-weighted dependency chain ending at the
    node that ends last."""
    n = len(nodes)
    dur = [end[i] - start[i] for i in range(n)]
    best = [0.0] * n
    pred = [-1] * n
    for nd in nodes:
        b, p = 0.0, -1
        for d in sorted(nd.deps):
            if best[d] > b:
                b, p = best[d], d
        best[nd.id] = b + dur[nd.id]
        pred[nd.id] = p
    last = max(range(n), key=lambda i: (end[i], -i))
    path = []
    while last >= 0:
        path.append(last)
        last = pred[last]
    return path[::-1]


def initial_units(nodes: List[Node], curves: Curves, budget: int, q: int) -> List[int]:
    """Reading P-6."""
    tot = [0.0] * N_KINDS
    for nd in nodes:
        tot[nd.kind] += curves.latency(nd.kind, budget, nd.work)
    s = sum(tot)
    units = []
    for k in range(N_KINDS):
        u = int(budget * tot[k] / s) // q * q if s > 0 else budget
        units.append(max(q, u))
    return units


def local_search(nodes: List[Node], curves: Curves, budget: int, q: int, units: List[int], max_iters: int):
    """Critical-path greedy moves from a start assignment (reading P-5)."""
    used = sorted({nd.kind for nd in nodes})
    best, st, en = simulate(nodes, units, curves, budget)
    for _ in range(max_iters):
        crit_kinds = sorted({nodes[i].kind for i in critical_path(nodes, st, en)})
        cand = None
        for c in crit_kinds:
            for d in [None] + [k for k in used if k != c]:
                u = list(units)
                if d is None:
                    if u[c] + q > budget:
                        continue
                    u[c] += q
                else:
                    if u[d] - q < q or u[c] + q > budget:
                        continue
                    u[d] -= q
                    u[c] += q
                m, s2, e2 = simulate(nodes, u, curves, budget)
                if m < best - 1e-15 and (cand is None or m < cand[0] - 1e-15):
                    cand = (m, u, s2, e2)
        if cand is None:
            break
        best, units, st, en = cand
    return units, best, st, en


def greedy(nodes: List[Node], curves: Curves, budget: int, q: int, max_iters: int = 200):
    """Greedy search from the two starts of reading P-6 (proportional, then the
    whole budget per kind); the shorter result wins, ties to the first."""
    r1 = local_search(nodes, curves, budget, q, initial_units(nodes, curves, budget, q), max_iters)
    r2 = local_search(nodes, curves, budget, q, [budget] * N_KINDS, max_iters)
    return r2 if r2[1] < r1[1] - 1e-15 else r1


# ------------------------------------------------------------------ the single-GPU NanoFlow pipeline
def balanced_groups(q_len, kv_prefix, shares) -> List[List[int]]:
    """Request -> nano-batch assignment of the executor's `balance` mode
    (reading A-10b): prefill requests (q_len > 1), largest first,
    go to the nano-batch with the most remaining token share; then decode
    requests, longest context first, to the nano-batch with the least
    accumulated attention work (prefill work counted as
    q_len * (prefix + q_len/2) / 64)."""
    T = sum(q_len)
    tot = sum(shares)
    cap = [T * s / tot for s in shares]
    kv = [0.0] * len(shares)
    grp = [[] for _ in shares]
    pre = sorted([r for r in range(len(q_len)) if q_len[r] > 1], key=lambda r: (-q_len[r], r))
    dec = sorted([r for r in range(len(q_len)) if q_len[r] == 1], key=lambda r: (-kv_prefix[r], r))
    for r in pre:
        k = max(range(len(shares)), key=lambda i: (cap[i], -i))
        grp[k].append(r)
        cap[k] -= q_len[r]
        kv[k] += q_len[r] * (kv_prefix[r] + q_len[r] / 2.0) / 64.0
    for r in dec:
        k = min(range(len(shares)), key=lambda i: (kv[i], i))
        grp[k].append(r)
        cap[k] -= 1
        kv[k] += kv_prefix[r] + 1
    return [sorted(g) for g in grp]


def nano_work(q_len, kv_prefix, groups):
    """Per nano-batch: (tokens, decode keys, prefill keys)."""
    out = []
    for g in groups:
        tok = sum(q_len[r] for r in g)
        dk = sum(kv_prefix[r] + 1 for r in g if q_len[r] == 1)
        pk = sum(sum(kv_prefix[r] + i + 1 for i in range(q_len[r])) for r in g if q_len[r] > 1)
        out.append((tok, dk, pk))
    return out


def build_pipeline(work: List[Tuple[int, int, int]], n_layers: int = 3) -> List[Node]:
    """The executor's OVERLAP schedule as a DAG (PAPER.md:691 single-GPU
    pipeline; api.cu nf_model_step): per nano k, KQV_k(l) -> DECODE_k(l)
    (memory stream) and KQV_k(l) -> PREFILL_k(l) (compute stream, reading
    A-11); O_k(l) waits for both, then UG_k(l) -> DOWN_k(l) -> KQV_k(l+1).
    Stream order adds edges: the compute stream runs
    [O UG DOWN KQV(next) PREFILL(next)] nano by nano, the memory stream the
    decode attention of nano 0, 1, ... in issue order."""
    nodes: List[Node] = []

    def add(kind, nano, w, deps):
        nodes.append(Node(len(nodes), kind, nano, float(w), [d for d in deps if d is not None]))
        return nodes[-1].id

    K = len(work)
    last_compute = None
    last_memory = None
    dec = [None] * K
    for k in range(K):  # prologue: KQV (+ prefill) of layer 0 for every nano
        kq = add(KQV, k, work[k][0], [last_compute])
        dec[k] = add(DECODE, k, work[k][1], [kq, last_memory])
        last_memory = dec[k]
        last_compute = add(PREFILL, k, work[k][2], [kq])
    for l in range(n_layers):
        for k in range(K):
            o = add(O, k, work[k][0], [dec[k], last_compute])
            ug = add(UG, k, work[k][0], [o])
            dn = add(DOWN, k, work[k][0], [ug])
            last_compute = dn
            if l + 1 < n_layers:
                kq = add(KQV, k, work[k][0], [dn])
                dec[k] = add(DECODE, k, work[k][1], [kq, last_memory])
                last_memory = dec[k]
                last_compute = add(PREFILL, k, work[k][2], [kq])
    return nodes


def search(q_len, kv_prefix, curves: Curves, budget=148, q=8, max_iters=200, n_layers=3):
    """All candidate splits (reading P-7); keep the shortest makespan
    ("choose the scheduling with the shortest critical path")."""
    best = None
    table = []
    for s in range(1, 8):
        shares = [s, 8 - s]
        groups = balanced_groups(q_len, kv_prefix, shares)
        nodes = build_pipeline(nano_work(q_len, kv_prefix, groups), n_layers)
        units, mk, st, en = greedy(nodes, curves, budget, q, max_iters)
        table.append((shares, units, mk))
        if best is None or mk < best[2] - 1e-15:
            best = (shares, units, mk, nodes, st, en)
    return best, table


# ------------------------------------------------------------------ the tensor-parallel pipeline (reading P-8)
def build_pipeline_tp(work: List[Tuple[int, int, int]], n_layers: int = 3) -> List[Node]:
    """PAPER.md:547-548 DAG over four quarters (work[q] = (tokens, decode keys,
    prefill keys)); H1 = quarters 0, 1 (column O + AG), H2 = quarters 2, 3 (row O + AR)."""
    assert len(work) == 4
    nodes: List[Node] = []

    def add(kind, nano, w, deps):
        nodes.append(Node(len(nodes), kind, nano, float(w), [d for d in deps if d is not None]))
        return nodes[-1].id

    last_c = last_m = last_n = None
    dec = [None] * 4
    pf = [None] * 4
    ready = [None, None]  # per group: the node its next-layer KQV waits for (its AR_d)
    tok = [work[0][0] + work[1][0], work[2][0] + work[3][0]]

    def front(g):
        nonlocal last_c, last_m
        for q in (2 * g, 2 * g + 1):
            kq = add(KQV, q, work[q][0], [last_c, ready[g]])
            dec[q] = add(DECODE, q, work[q][1], [kq, last_m])
            last_m = dec[q]
            pf[q] = add(PREFILL, q, work[q][2], [kq])
            last_c = pf[q]

    front(0)
    front(1)
    for l in range(n_layers):
        ag_a = add(NET, 0, tok[0], [dec[0], dec[1], pf[1], last_n])
        last_n = ag_a
        o1 = add(O, 0, tok[0], [ag_a, last_c])
        last_c = o1
        ag_o = add(NET, 0, tok[0], [o1, last_n])
        last_n = ag_o
        o2 = add(O, 1, tok[1], [dec[2], dec[3], last_c])
        last_c = o2
        ar_o = add(NET, 1, 2 * tok[1], [o2, last_n])
        last_n = ar_o
        ug1 = add(UG, 0, tok[0], [ag_o, last_c])
        d1 = add(DOWN, 0, tok[0], [ug1])
        last_c = d1
        ar_d1 = add(NET, 0, 2 * tok[0], [d1, last_n])
        last_n = ar_d1
        ug2 = add(UG, 1, tok[1], [ar_o, last_c])
        d2 = add(DOWN, 1, tok[1], [ug2])
        last_c = d2
        ar_d2 = add(NET, 1, 2 * tok[1], [d2, last_n])
        last_n = ar_d2
        ready = [ar_d1, ar_d2]
        if l + 1 < n_layers:
            front(0)
            front(1)
    return nodes


def search_tp(q_len, kv_prefix, curves: Curves, budget=148, q=8, max_iters=200, n_layers=3):
    """Reading P-8 candidates (H1 share s/8, quarters even); shortest makespan wins."""
    best = None
    table = []
    for s in range(1, 8):
        shares = [s, s, 8 - s, 8 - s]
        groups = balanced_groups(q_len, kv_prefix, shares)
        nodes = build_pipeline_tp(nano_work(q_len, kv_prefix, groups), n_layers)
        units, mk, st, en = greedy(nodes, curves, budget, q, max_iters)
        table.append((shares, units, mk))
        if best is None or mk < best[2] - 1e-15:
            best = (shares, units, mk, nodes, st, en)
    return best, table
