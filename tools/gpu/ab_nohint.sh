set -x
python tools/gemm_fixed.py 148 > gpurun_out/gemm_fixed_nohint.log 2>&1
MS=1024,2048 python tools/gemm_micro.py 148 116 > gpurun_out/gemm_micro_nohint.log 2>&1
timeout 300 python tools/attn_micro.py 16,32,48,148 5 > gpurun_out/attn_nohint.log 2>&1
SHAPE=c3rank timeout 300 python tools/attn_micro.py 16,32,148 5 >> gpurun_out/attn_nohint.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_nohint.log 2>&1
timeout 900 python bench.py --config c3loop --steps 10 > gpurun_out/bench_c3loop_nohint.log 2>&1
