# 8B step: nano-batch shares aligned to 128-row GEMM tiles at 116 SMs (7:9 -> 896/1152 tokens) and finer SM splits
timeout 1500 python tools/sweep_plans.py --config c2 --steps 6 --shares 1:1,7:9,9:7,5:3 --splits 116/32,112/36,120/28 > gpurun_out/r2n_sweep_c2.log 2>&1
timeout 1500 python tools/sweep_plans.py --config c2 --steps 6 --shares 1:1,7:9,9:7 --splits 116/32,120/28 > gpurun_out/r2n_sweep_c2_b.log 2>&1
