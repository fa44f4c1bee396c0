"""Global batch scheduler and KV-cache manager of NanoFlow's serving loop
 -- TEST INFRASTRUCTURE ONLY: the plain, step-by-step
statement of the policy that the native scheduler (csrc/sched.cpp,
nf_sched_*) must reproduce bit-exactly (integer work).

Passages followed (readings A-25..A-29 in DESIGN.md):

* P:504 continuous batching with chunked prefill: every step refills the
  global batch; decode requests contribute one token, prompt chunks fill the
  rest of the dense batch (A-25: decodes first, then prompt chunks of the
  admitted requests in admission order).
* P:504-505 discrete batching: B_dense is chosen among a few
  high-performance sizes -- the largest allowed size not above the tokens
  available, or everything when fewer tokens than the smallest size are
  available; decode requests are never deferred to reach a smaller size
  (if that size is below the decode count, every decode runs, up to the
  largest allowed size, and no prefill) (A-26).
* P:573-575 peak-memory admission: the manager predicts each running
  request's completion assuming its total decode length equals the average
  decode length, computes the highest future memory use and admits new
  requests (first come, first served) only if that peak fits; when the pool
  still runs out, it discards a request (A-27: the most recently admitted one
  is evicted, its pages freed, and it is re-queued at the front with its
  progress reset).  Estimate (integer, A-27): request r with L_r = prompt +
  generated tokens is predicted to live tau_r = max(avg_decode - generated, 1)
  more steps, holding L_r + tau tokens at future step tau <= tau_r; the peak
  in pages is max_j floor(sum_{r: tau_r >= tau_j} (L_r + tau_j + page - 1) / page).
* P:652-657 asynchronous scheduling: step i+1 is formed and launched before
  step i's tokens are read; EOS of step i is detected after launching i+1 and
  the request is removed by the formation of step i+2, generating one
  useless token (A-28).  A decode's input token is therefore a device
  reference into the previous step's next_ids when it was produced by that
  step (tok_src = -(1 + row)), else the host-known token id.
* A-29 pages: a request holds ceil(tokens / page) pages of the pool,
  allocated lowest free page id first when its length crosses a page
  boundary, released when it finishes or is evicted.
* A synthetic request's EOS is its output length (the trace's "output
  length": EOS is detected when the token generated at that count is read
  back), or a token equal to eos_id (>= 0).
"""
from __future__ import annotations

import heapq
from typing import Dict, List, Optional, Sequence


class _Req:
    def __init__(self, rid: int, prompt: Sequence[int], out_len: int, order: int):
        self.rid = rid
        self.prompt = list(int(t) for t in prompt)
        self.out_len = int(out_len)
        self.order = order          # submission order (FCFS)
        self.reset()

    def reset(self):
        self.prefilled = 0          # prompt tokens cached
        self.generated = 0          # tokens emitted
        self.pages: List[int] = []
        self.last_tok: Optional[int] = None
        self.last_step = -1         # step whose next_ids hold the last emitted token
        self.last_row = -1
        self.finished = False
        self.admit_seq = -1


class Step:
    """One formed step: the nf_batch arrays plus token sources."""

    def __init__(self):
        self.step = -1
        self.req_ids: List[int] = []
        self.q_len: List[int] = []
        self.kv_prefix: List[int] = []
        self.page_indptr: List[int] = [0]
        self.page_ids: List[int] = []
        self.emit: List[int] = []
        self.tok_src: List[int] = []

    @property
    def n_tokens(self) -> int:
        return sum(self.q_len)


class Scheduler:
    def __init__(self, n_pages: int, page_size: int, bdense: Sequence[int], avg_decode: int, eos_id: int = -1):
        if n_pages < 1 or page_size < 1 or not bdense or avg_decode < 1:
            raise ValueError("bad scheduler config")
        self.n_pages = n_pages
        self.page = page_size
        self.bdense = sorted(set(int(b) for b in bdense), reverse=True)
        self.avg = int(avg_decode)
        self.eos = int(eos_id)
        self.free = list(range(n_pages))          # min-heap of free page ids
        heapq.heapify(self.free)
        self.queue: List[_Req] = []                 # waiting, FCFS
        self.running: List[_Req] = []               # admission order
        self.by_id: Dict[int, _Req] = {}
        self.n_submitted = 0
        self.admit_counter = 0
        self.step_no = 0
        self.pending: Dict[int, List] = {}          # step -> [(req, generated count after the step)]
        self.stats = {"steps": 0, "tokens": 0, "prefill_tokens": 0, "decode_tokens": 0, "finished": 0,
                      "generated": 0, "useless": 0, "evictions": 0, "peak_pages_used": 0}

    # ------------------------------------------------------------ API
    def submit(self, rid: int, prompt: Sequence[int], out_len: int):
        if rid in self.by_id or len(prompt) < 1 or out_len < 1:
            raise ValueError("bad request")
        r = _Req(rid, prompt, out_len, self.n_submitted)
        self.n_submitted += 1
        self.by_id[rid] = r
        self.queue.append(r)

    def idle(self) -> bool:
        return not self.queue and not self.running

    def next(self) -> Step:
        """Form the next step (A-25..A-29)."""
        # 1. retire requests whose EOS has been read back
        for r in [r for r in self.running if r.finished]:
            self._release(r)
            self.running.remove(r)
        # 2. FCFS admission under the peak-memory estimate
        while self.queue:
            c = self.queue[0]
            if self._peak_pages(self.running + [c]) > self.n_pages:
                break
            self.queue.pop(0)
            c.admit_seq = self.admit_counter
            self.admit_counter += 1
            self.running.append(c)
        # 3-4. compose and allocate pages, evicting on exhaustion
        while True:
            comp = self._compose()
            victim = self._allocate(comp)
            if victim is None:
                break
            self._evict(victim)
        return self._emit_step(comp)

    def complete(self, step: int, next_ids: Sequence[int]):
        """Tokens of `step` read back: remember them, detect EOS (A-28)."""
        if step not in self.pending:
            raise ValueError(f"step {step} not pending")
        for row, (r, gen_after) in enumerate(self.pending.pop(step)):
            if r is None:
                continue
            tok = int(next_ids[row])
            if r.last_step == step:
                r.last_tok = tok
            if not r.finished and (gen_after == r.out_len or (self.eos >= 0 and tok == self.eos)):
                r.finished = True
                self.stats["finished"] += 1

    # ------------------------------------------------------------ policy
    def _peak_pages(self, reqs: List[_Req]) -> int:
        items = []
        for r in reqs:
            L = len(r.prompt) + r.generated
            tau = max(self.avg - r.generated, 1)
            items.append((tau, L))
        best = 0
        for tau_j, _ in items:
            tot = sum(L + tau_j + self.page - 1 for tau, L in items if tau >= tau_j)
            best = max(best, tot // self.page)
        return best

    def _compose(self):
        dec = [r for r in self.running if r.prefilled == len(r.prompt)]
        avail = len(dec) + sum(len(r.prompt) - r.prefilled for r in self.running)
        fits = [b for b in self.bdense if b <= avail]
        B = fits[0] if fits else avail
        if B < len(dec):                            # decodes never wait for a smaller size (A-26)
            B = min(len(dec), self.bdense[0])
        comp = []                                   # (req, q_len, kv_prefix, emit)
        for r in dec[:B]:
            comp.append((r, 1, len(r.prompt) + r.generated - 1, 1))
        budget = B - min(len(dec), B)
        for r in self.running:
            if budget == 0:
                break
            rem = len(r.prompt) - r.prefilled
            if rem > 0:
                c = min(rem, budget)
                comp.append((r, c, r.prefilled, 1 if c == rem else 0))
                budget -= c
        return comp

    def _allocate(self, comp) -> Optional[_Req]:
        """Allocate pages for the composed step; returns the request to evict if
        the pool runs out (nothing allocated then)."""
        need_total = 0
        for r, q, kv, _ in comp:
            need_total += max(0, -(-(kv + q) // self.page) - len(r.pages))
        if need_total <= len(self.free):
            for r, q, kv, _ in comp:
                need = -(-(kv + q) // self.page) - len(r.pages)
                for _ in range(max(0, need)):
                    r.pages.append(heapq.heappop(self.free))
            used = self.n_pages - len(self.free)
            self.stats["peak_pages_used"] = max(self.stats["peak_pages_used"], used)
            return None
        return max(self.running, key=lambda r: r.admit_seq)

    def _release(self, r: _Req):
        for p in r.pages:
            heapq.heappush(self.free, p)
        r.pages = []

    def _evict(self, r: _Req):
        self._release(r)
        self.running.remove(r)
        for lst in self.pending.values():             # its in-flight outputs are dropped
            for i, (q, g) in enumerate(lst):
                if q is r:
                    lst[i] = (None, 0)
        r.reset()
        self.queue.insert(0, r)
        self.stats["evictions"] += 1

    def _emit_step(self, comp) -> Step:
        s = Step()
        s.step = self.step_no
        prev = self.step_no - 1
        rows = []
        for row, (r, q, kv, em) in enumerate(comp):
            s.req_ids.append(r.rid)
            s.q_len.append(q)
            s.kv_prefix.append(kv)
            s.page_ids += r.pages
            s.page_indptr.append(len(s.page_ids))
            s.emit.append(em)
            if q == 1 and kv >= len(r.prompt):       # decode: last generated token
                if r.last_step >= 0 and r.last_step in self.pending:
                    if r.last_step != prev:
                        raise RuntimeError("decode input from a step older than the previous one is not read back")
                    s.tok_src.append(-(1 + r.last_row))
                else:
                    s.tok_src.append(r.last_tok)
            else:
                s.tok_src += r.prompt[kv:kv + q]
            # bookkeeping as if the step runs
            if q > 1 or kv < len(r.prompt):
                r.prefilled += q
                self.stats["prefill_tokens"] += q
            else:
                self.stats["decode_tokens"] += 1
            if em:
                r.generated += 1
                r.last_step = s.step
                r.last_row = row
                self.stats["generated"] += 1
                if r.generated > r.out_len:
                    self.stats["useless"] += 1
                rows.append((r, r.generated))
            else:
                rows.append((None, 0))
        self.pending[s.step] = rows
        self.stats["steps"] += 1
        self.stats["tokens"] += s.n_tokens
        self.step_no += 1
        return s
