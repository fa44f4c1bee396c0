#!/usr/bin/env python
"""Summarise ncu reports (--set full) and a launch-list CSV into profiles/.
Usage: ncu_summary.py OUT_MD REPORT.ncu-rep... [--launches launches.csv]"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

KEYS = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "dram read"),
        ("dram__bytes_write.sum", "dram write"), ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram %"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe (HMMA) %"),
        ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "tcgen05 pipe %"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
        ("launch__grid_size", "grid"), ("launch__block_size", "block"), ("launch__registers_per_thread", "regs"),
        ("sm__cycles_elapsed.avg.per_second", "SM clock"), ("lts__t_bytes.sum", "L2 bytes")]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return [dict(zip(rows[0], r)) for r in rows[2:]], dict(zip(rows[0], rows[1]))


def to_bytes(v, unit):
    v = float(v)
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main():
    args = sys.argv[1:]
    launches = None
    if "--launches" in args:
        i = args.index("--launches")
        launches = args[i + 1]
        args = args[:i] + args[i + 2:]
    out_md, reps = args[0], args[1:]
    lines = ["# ncu summaries", "", "Captured with `ncu --set full --import-source on --clock-control none` "
             "on one B200 (gpurun); one launch per report.  Durations under ncu are serialised and cold-cache.", ""]
    traffic = {}
    for rep in reps:
        rows, units = raw(rep)
        for r in rows:
            name = r.get("Kernel Name", "?")[:90]
            lines.append(f"## {os.path.basename(rep)} — `{name}`")
            lines.append("")
            lines.append("| metric | value |")
            lines.append("|---|---|")
            for k, label in KEYS:
                if k in r:
                    lines.append(f"| {label} (`{k}`) | {r[k]} {units.get(k, '')} |")
            try:
                rd = to_bytes(r["dram__bytes_read.sum"].replace(",", ""), units["dram__bytes_read.sum"])
                wr = to_bytes(r["dram__bytes_write.sum"].replace(",", ""), units["dram__bytes_write.sum"])
                dur = float(r["gpu__time_duration.sum"].replace(",", "")) * (1e-9 if units["gpu__time_duration.sum"] == "nsecond" else 1e-6)
                lines.append(f"| dram read+write per launch | {(rd + wr) / 1e6:.1f} MB ({(rd + wr) / dur / 1e9:.0f} GB/s) |")
                key = "decode_attn" if "decode" in name else ("prefill_attn" if "prefill" in name else "gemm")
                traffic.setdefault(key, rd + wr)
            except Exception:
                pass
            lines.append("")
    if launches:
        rows = list(csv.reader(open(launches)))
        hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
        hdr = rows[hdr_i]
        ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
        per = defaultdict(lambda: [0, 0.0])
        tot = 0.0
        data = rows[hdr_i + 1:]
        # step kernels only: weight generation (torch RNG) and one-time packing are setup
        setup = ("CUDAGeneratorImpl", "pack_gate_up", "scale_cols", "elementwise", "vectorized", "fill_kernel")
        for r in data:
            if len(r) <= vi or any(k in r[ki] for k in setup):
                continue
            nm = r[ki].split("(")[0].split("::")[-1]
            v = float(r[vi].replace(",", ""))
            per[nm][0] += 1
            per[nm][1] += v
            tot += v
        lines += ["## Launch list (`ncu --metrics gpu__time_duration.sum`, whole bench command)", "",
                  f"{sum(n for n, _ in per.values())} step launches (setup kernels excluded); per-kernel share of summed device time (serialised, cold cache):", "",
                  "| kernel | launches | total ms | share |", "|---|---|---|---|"]
        for nm, (n, t) in sorted(per.items(), key=lambda kv: -kv[1][1]):
            lines.append(f"| `{nm}` | {n} | {t / 1e6:.2f} | {100 * t / tot:.1f} % |")
        lines.append("")
    open(out_md, "w").write("\n".join(lines) + "\n")
    tpath = os.path.join(os.path.dirname(out_md), "traffic.json")
    json.dump(traffic, open(tpath, "w"), indent=1)
    print(open(out_md).read())


if __name__ == "__main__":
    main()
