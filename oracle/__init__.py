"""CPU oracle of NanoFlow's hot path (arXiv 2408.12757) — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import anything under
``oracle/``.  The product package ``paper_2408_12757_b200`` never imports it
and has no CPU fallback.

What it computes: NanoFlow reaches exactly the same result as
running the decoder layer unsplit, unsharded and sequentially
("within a given nano-batch, all of the operations follow
sequential dependencies"; TP is an algebraic decomposition).
So the oracle is the plain definition of a LLaMA-style decoder layer over a
mixed prefill/decode batch with a paged KV cache, written in float64 numpy:

* ``metadata``  — positions, KV write slots, nano-batch cut snapping (a1).
* ``layer``     — RMSNorm, RoPE, KV append, paged causal GQA attention,
                  the decoder layer, per-nano-batch execution, the TP-sharded
                  algebra and the model step (embedding .. argmax).
* ``moe``       — the Mixtral-shape MoE FFN (readings A-20..A-23):
                  router top-k, expert SwiGLU, weighted combine, TP-sharded
                  form, and the integer token grouping of the grouped GEMMs.
* ``costmodel`` — the paper's analytic model (Eq. 2-10, Table 2), pinned by the
                  golden values the paper prints (tests/golden/).
* ``serving``   — the global batch scheduler / KV-cache manager policy (NEXT-4).
* ``planner``   — the §5.6 autosearch step by step (critical path + greedy).

Every function cites the PAPER.md line (``P:n``) or SURVEY.md reading
(``A-k``) it follows.  Parity status: all functions are pinned by
``tests/test_oracle_*.py`` (closed forms, invariants, brute force, paper
values); none is "parity unpinned".
"""
