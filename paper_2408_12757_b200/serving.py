"""Offline serving loop: the asynchronous top-level
schedule of PAPER.md:652-657 around nf_model_step.

Per iteration i (all decisions in the native scheduler, nf_sched_*):

  1. nf_sched_next forms step i (continuous batching + chunked prefill,
     discrete B_dense, peak-memory admission, page allocation) while the GPU
     still runs step i-1;
  2. the step's token sources go to the device (pinned, async) and
     nf_assemble_tokens resolves decode inputs that exist only in step i-1's
     device next_ids; nf_model_step i is launched behind step i-1 on the stream;
  3. only then is step i-1's next_ids read back (event sync) and passed to
     nf_sched_complete, which detects EOS -- a request finishing at step i-1
     has already been launched in step i (one useless token) and is
     removed by the formation of step i+1.

This module is orchestration only: no arithmetic, no scheduling policy.
"""
from __future__ import annotations

import time
from typing import Dict, List, Optional, Sequence

import numpy as np
import torch

from . import nf


class OfflineServer:
    def __init__(self, model, plan: nf.Plan, pools: Sequence[torch.Tensor], sched: nf.Scheduler, n_pages_pool: int,
                 max_tokens: int, max_reqs: int, comm: Optional[int] = None):
        self.model, self.plan, self.pools, self.sched = model, plan, list(pools), sched
        self.n_pages_pool = n_pages_pool
        self.comm = comm
        dev = pools[0].device
        i32 = torch.int32
        self.next_ids = [torch.zeros(max_reqs, dtype=i32, device=dev) for _ in range(2)]
        self.host_ids = [torch.zeros(max_reqs, dtype=i32).pin_memory() for _ in range(2)]
        self.src_host = [torch.zeros(max_tokens, dtype=i32).pin_memory() for _ in range(2)]
        self.src_dev = [torch.zeros(max_tokens, dtype=i32, device=dev) for _ in range(2)]
        self.tok_dev = torch.zeros(max_tokens, dtype=i32, device=dev)
        self.done = [torch.cuda.Event() for _ in range(2)]
        self.ws: Optional[torch.Tensor] = None
        self.max_tokens, self.max_reqs = max_tokens, max_reqs

    def _workspace(self, b: nf.Batch) -> torch.Tensor:
        n = nf.workspace_size(self.model.cfg, b)
        if self.ws is None or self.ws.numel() < n:
            self.ws = torch.empty(int(n * 1.25) + 4096, dtype=torch.uint8, device=self.pools[0].device)
        return self.ws

    def run(self, max_steps: int = 1 << 30, on_step=None) -> Dict:
        """Serve until every submitted request finished (or max_steps).  on_step(st, ids):
        optional callback per completed step with its formed batch (nf.Scheduler.next dict)
        and its next_ids read back from the device."""
        stream = torch.cuda.current_stream()
        prev = None
        self.timeline = []          # per launched step: (wall s since start, tokens, requests still queued)
        host_sched_s = 0.0
        steps = tokens = 0
        t0 = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(max_steps):
            h0 = time.perf_counter()
            st = self.sched.next()
            host_sched_s += time.perf_counter() - h0
            n, T = len(st["req_ids"]), int(st["q_len"].sum()) if len(st["q_len"]) else 0
            launched = None
            if n > 0:
                if T > self.max_tokens or n > self.max_reqs:
                    raise RuntimeError(f"step of {T} tokens / {n} requests exceeds the server's buffers")
                slot = st["step"] % 2
                b = nf.Batch(st["q_len"], st["kv_prefix"], st["page_indptr"], st["page_ids"], self.n_pages_pool,
                             emit=st["emit"])
                self.src_host[slot][:T].copy_(torch.from_numpy(st["tok_src"]))
                self.src_dev[slot][:T].copy_(self.src_host[slot][:T], non_blocking=True)
                nf.assemble_tokens(self.src_dev[slot].data_ptr(), self.next_ids[1 - slot].data_ptr(),
                                   self.tok_dev.data_ptr(), T, int(stream.cuda_stream))
                ws = self._workspace(b)
                self.model.step(self.plan, self.pools, b, self.tok_dev[:T], ws, self.next_ids[slot][:n], comm=self.comm)
                self.host_ids[slot][:n].copy_(self.next_ids[slot][:n], non_blocking=True)
                self.done[slot].record(stream)
                launched = (st, slot, n, T)
                steps += 1
                tokens += T
                self.timeline.append((time.perf_counter() - t0, T, self.sched.stats()["queued"]))
            if prev is not None:
                pst, pslot, pn, pT = prev
                self.done[pslot].synchronize()
                ids = self.host_ids[pslot][:pn].numpy().copy()
                h0 = time.perf_counter()
                self.sched.complete(pst["step"], ids)
                host_sched_s += time.perf_counter() - h0
                if on_step is not None:
                    on_step(pst, ids)
            elif launched is None:
                self.sched.complete(st["step"], np.zeros(0, np.int32))
                break                                  # idle: nothing running, nothing queued
            if launched is None and prev is not None:
                self.sched.complete(st["step"], np.zeros(0, np.int32))
            prev = launched
        e1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        out = self.sched.stats()
        out.update({"gpu_steps": steps, "step_tokens": tokens, "wall_s": wall,
                    "device_s": e0.elapsed_time(e1) / 1e3, "host_sched_s": host_sched_s})
        # steady state: the steps launched while requests were still waiting for admission
        # (the system is at capacity; the drain of the last long requests is excluded)
        busy = [i for i, (_, _, q) in enumerate(self.timeline) if q > 0]
        if len(busy) >= 2:
            i0, i1 = busy[0], busy[-1]
            t_end = self.timeline[i1 + 1][0] if i1 + 1 < len(self.timeline) else wall
            out["steady_steps"] = i1 - i0 + 1
            out["steady_tokens"] = sum(T for _, T, _ in self.timeline[i0:i1 + 1])
            out["steady_s"] = t_end - self.timeline[i0][0]
        return out
