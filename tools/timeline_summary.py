#!/usr/bin/env python
"""Summarise a bench --timeline CSV: per-stream busy time, idle gaps, overlap."""
import sys
from collections import defaultdict

rows = [l.strip().split(",") for l in open(sys.argv[1]).read().splitlines()[1:]]
spans = [(op, int(s), float(a), float(b)) for op, s, a, b in rows]
t0 = min(a for _, _, a, _ in spans)
t1 = max(b for _, _, _, b in spans)
print(f"step span {t1 - t0:.2f} ms, {len(spans)} kernels")
by = defaultdict(list)
for op, s, a, b in spans:
    by[s].append((a, b, op))
for s, lst in sorted(by.items()):
    lst.sort()
    busy = sum(b - a for a, b, _ in lst)
    ops = defaultdict(float)
    for a, b, op in lst:
        ops[op] += b - a
    print(f"stream {s}: busy {busy:.2f} ms ({100 * busy / (t1 - t0):.0f}%)", {k: round(v, 2) for k, v in ops.items()})
if len(sys.argv) > 2:
    for op, s, a, b in sorted(spans, key=lambda x: x[2])[: int(sys.argv[2])]:
        print(f"{s} {op:14s} {a - t0:8.3f} {b - t0:8.3f} {b - a:7.3f}")
