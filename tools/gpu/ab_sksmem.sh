# smem-staged stream-K / split-K fix-up: GEMM parity, phase timings and throughput A/B
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm" > gpurun_out/sksmem_tests.log 2>&1; echo "rc=$?" >> gpurun_out/sksmem_tests.log
NF_LIB=paper_2408_12757_b200/_ts/libnf.so python tools/gemm_phases.py 148 > gpurun_out/sksmem_phases.log 2>&1
NF_GEMM_SKSMEM=0 NF_LIB=paper_2408_12757_b200/_ts/libnf.so python tools/gemm_phases.py 148 > gpurun_out/sksmem_phases_off.log 2>&1
MS=512,1024,2048 python tools/gemm_micro.py 148 132 116 > gpurun_out/sksmem_micro_on.log 2>&1
NF_GEMM_SKSMEM=0 MS=512,1024,2048 python tools/gemm_micro.py 148 132 116 > gpurun_out/sksmem_micro_off.log 2>&1
