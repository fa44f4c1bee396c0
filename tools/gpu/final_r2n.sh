# round-2 re-entry validation at HEAD: full GPU suite, smoke (and its launch list under ncu), default bench
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2n_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/r2n_gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2n_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2n_smoke.log
timeout 900 python bench.py > gpurun_out/r2n_bench_default.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r2n_smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2n_smoke_ncu.out 2>&1; echo "rc=$?" >> gpurun_out/r2n_smoke_ncu.out
