# parity of the changed kernels, then the default 8B step and the TP8-rank proxy with the
# decode variant A/B (NF_DEC_STREAM_VAR=1: four S^T chains)
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/parity.log 2>&1; echo "parity rc=$?" >> gpurun_out/parity.log
run() { tag=$1; shift; echo "== $tag" >> gpurun_out/ab_step.log; env "$@" timeout 600 python bench.py --no-cpu-baseline --no-parity $BARGS >> gpurun_out/ab_step.log 2>&1; }
BARGS=""
run base
run var1 NF_DEC_STREAM_VAR=1
run base2
run var1b NF_DEC_STREAM_VAR=1
BARGS="--config c3loop --steps 10"
run c3base
run c3var1 NF_DEC_STREAM_VAR=1
