# TP: decode attention on side streams of the compute partition (NF_TP_DEC_SIDE=1) vs on the group's compute stream
NF_TP_DEC_SIDE=1 timeout 1500 python -m pytest tests/test_gpu_tp.py -x -q > gpurun_out/decside_tests.log 2>&1; echo "rc=$?" >> gpurun_out/decside_tests.log
run() { tag=$1; shift; echo "== $tag" >> gpurun_out/decside_ab.log; env "$@" timeout 900 python bench.py --config c3loop --net-model nvlink --steps 10 --no-cpu-baseline >> gpurun_out/decside_ab.log 2>&1; }
run side NF_TP_DEC_SIDE=1
run base
run side2 NF_TP_DEC_SIDE=1
run base2
