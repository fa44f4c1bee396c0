# final validation at the last commit: full GPU suite, smoke, default bench (driver's N=1 line)
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2o_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/r2o_gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2o_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2o_smoke.log
timeout 900 python bench.py > gpurun_out/r2o_bench_default.log 2>&1; echo "rc=$?" >> gpurun_out/r2o_bench_default.log
