timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2h_gputest.log 2>&1; tail -3 gpurun_out/r2h_gputest.log
timeout 600 python bench.py > gpurun_out/r2h_bench_default.log 2>&1; tail -c 400 gpurun_out/r2h_bench_default.log
NF_GREEN=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2h_launches.csv python bench.py --steps 1 --warmup 3 --ncu > gpurun_out/r2h_ncu_launches.out 2>&1
NF_GREEN=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_stream -s 8 -c 1 -o gpurun_out/r2h_dec_step python bench.py --steps 1 --warmup 3 --ncu > gpurun_out/r2h_ncu_step.out 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_stream -c 1 -o gpurun_out/r2h_dec32 python tools/attn_micro.py 32 1 > gpurun_out/r2h_ncu_micro.out 2>&1
ls -la gpurun_out/
