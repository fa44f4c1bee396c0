timeout 3000 python tools/workload_sweep.py --config c3loop --curves profiles/curves_b200_tp8.csv --steps 3 --rounds 2 > gpurun_out/r2j_workloads_c3loop.jsonl 2> gpurun_out/r2j_workloads_c3loop.err
tail -5 gpurun_out/r2j_workloads_c3loop.err; cat gpurun_out/r2j_workloads_c3loop.jsonl | cut -c1-600
