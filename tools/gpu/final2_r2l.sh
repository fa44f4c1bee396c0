# round-2 final validation at the last commit: full GPU suite, smoke, default bench, TP8-rank proxy (plain / modeled link)
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2m_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/r2m_gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2m_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2m_smoke.log
timeout 900 python bench.py > gpurun_out/r2m_bench_default.log 2>&1
timeout 900 python bench.py --config c3loop --net-model nvlink --steps 10 > gpurun_out/r2m_bench_c3loop_nvlink.log 2>&1
timeout 900 python bench.py --config c3loop --steps 10 --no-cpu-baseline > gpurun_out/r2m_bench_c3loop.log 2>&1
