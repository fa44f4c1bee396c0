# L1 prefetch of the split-tile fix-up's partial chunks (NF_GEMM_SKPF): parity, phases, micro, TP8-rank step
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm or layer_70b or layer_8b_full" > gpurun_out/skpf_tests.log 2>&1; echo "rc=$?" >> gpurun_out/skpf_tests.log
NF_LIB=paper_2408_12757_b200/_ts/libnf.so python tools/gemm_phases.py 148 > gpurun_out/skpf_phases.log 2>&1
NF_GEMM_SKPF=0 NF_LIB=paper_2408_12757_b200/_ts/libnf.so python tools/gemm_phases.py 148 > gpurun_out/skpf_phases_off.log 2>&1
for i in 1 2; do
ONLY=70r MS=1024,2048 python tools/gemm_micro.py 148 132 >> gpurun_out/skpf_micro_on.log 2>&1
NF_GEMM_SKPF=0 ONLY=70r MS=1024,2048 python tools/gemm_micro.py 148 132 >> gpurun_out/skpf_micro_off.log 2>&1
done
run() { tag=$1; shift; echo "== $tag" >> gpurun_out/skpf_ab.log; env "$@" timeout 900 python bench.py --config c3loop --net-model nvlink --steps 10 --no-cpu-baseline >> gpurun_out/skpf_ab.log 2>&1; }
run on
run off NF_GEMM_SKPF=0
run on2
run off2 NF_GEMM_SKPF=0
