# slot-layout A for the O column-parallel GEMM: TP parity tests, then the TP8-rank proxy A/B
timeout 1500 python -m pytest tests/test_gpu_tp.py tests/test_gpu_nccl.py -x -q > gpurun_out/aslots_tests.log 2>&1; echo "rc=$?" >> gpurun_out/aslots_tests.log
run() { tag=$1; shift; echo "== $tag" >> gpurun_out/aslots_ab.log; env "$@" timeout 900 python bench.py --config c3loop --net-model nvlink --steps 10 --no-cpu-baseline >> gpurun_out/aslots_ab.log 2>&1; }
run on
run off NF_GEMM_ASLOTS=0
run on2
run off2 NF_GEMM_ASLOTS=0
