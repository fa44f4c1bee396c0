timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2k_gputest.log 2>&1; tail -3 gpurun_out/r2k_gputest.log
timeout 900 python bench.py > gpurun_out/r2k_bench_default.log 2>&1; tail -c 300 gpurun_out/r2k_bench_default.log
timeout 900 python bench.py --config c3loop --steps 10 > gpurun_out/r2k_bench_c3loop.log 2>&1; tail -c 300 gpurun_out/r2k_bench_c3loop.log
