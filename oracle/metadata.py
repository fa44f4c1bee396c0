"""Batch metadata of step a1 — test infrastructure only.

Integer-exact definitions the CUDA path's host metadata must reproduce
bit-for-bit:

* token rows are request-major (PAPER.md:155, :504 — prefill chunks and
  decode tokens co-batched into one dense batch);
* token i of request r sits at absolute position kv_prefix[r] + i
  (reading A-4: position = absolute index in the request);
* its K/V goes to logical page (pos // page) of the request, slot pos % page,
  through the PagedAttention-style page table (reading A-7);
* nano-batch cuts snap to request boundaries, nearest boundary to the target
  offset, ties to the lower (reading A-10; "split a batch of
  user requests into smaller nano-batches").
"""
from __future__ import annotations

from fractions import Fraction
from typing import List, Sequence

import numpy as np


def qo_indptr(q_len: np.ndarray) -> np.ndarray:
    out = np.zeros(len(q_len) + 1, dtype=np.int64)
    for r, n in enumerate(q_len):
        out[r + 1] = out[r] + int(n)
    return out


def token_request(q_len: np.ndarray) -> np.ndarray:
    return np.array([r for r, n in enumerate(q_len) for _ in range(int(n))], dtype=np.int64)


def positions(q_len: np.ndarray, kv_prefix: np.ndarray) -> np.ndarray:
    """pos[t] = kv_prefix[r] + i for the i-th new token of request r (A-4)."""
    return np.array([int(kv_prefix[r]) + i for r, n in enumerate(q_len) for i in range(int(n))],
                    dtype=np.int64)


def kv_len(q_len: np.ndarray, kv_prefix: np.ndarray) -> np.ndarray:
    """Keys visible to the last token of request r after the append (A-6)."""
    return np.asarray(kv_prefix, dtype=np.int64) + np.asarray(q_len, dtype=np.int64)


def write_slots(q_len, kv_prefix, page_indptr, page_ids, page_size: int = 16):
    """(physical page, in-page slot) of every new token, request-major."""
    pages, offs = [], []
    for r, n in enumerate(q_len):
        for i in range(int(n)):
            p = int(kv_prefix[r]) + i
            pages.append(int(page_ids[int(page_indptr[r]) + p // page_size]))
            offs.append(p % page_size)
    return np.array(pages, dtype=np.int64), np.array(offs, dtype=np.int64)


def snap_cuts(q_len: Sequence[int], fractions: Sequence[Fraction]) -> List[int]:
    """Request-index boundaries of nano-batches (reading A-10).

    ``fractions`` are the nano-batch token shares (sum 1).  Target token
    offset k = T * (f_0 + .. + f_{j}); the cut is the request boundary whose
    token offset is nearest to the target, ties to the lower boundary.
    Returns request indices [0, c_1, ..., n_req] (non-decreasing; empty
    nano-batches allowed).
    """
    ind = qo_indptr(np.asarray(q_len))
    T = int(ind[-1])
    n_req = len(q_len)
    cuts = [0]
    acc = Fraction(0)
    for f in list(fractions)[:-1]:
        acc += Fraction(f)
        target = acc * T
        best = None
        for b in range(n_req + 1):
            d = abs(Fraction(int(ind[b])) - target)
            if best is None or d < best[0]:
                best = (d, b)
        cuts.append(max(best[1], cuts[-1]))
    cuts.append(n_req)
    return cuts
