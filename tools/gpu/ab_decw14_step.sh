# step-level A/B of the 14-warp decode stream kernel (NF_DEC_STREAM_WARPS=14) on the 8B OVERLAP step and the TP8-rank proxy
run() { tag=$1; shift; echo "== $tag" >> gpurun_out/r2n_ab_decw14_step.log; env "$@" timeout 600 python bench.py --no-cpu-baseline --no-parity $BARGS >> gpurun_out/r2n_ab_decw14_step.log 2>&1; }
BARGS="--steps 20"
run base
run w14 NF_DEC_STREAM_WARPS=14
run base2
run w142 NF_DEC_STREAM_WARPS=14
run base3
run w143 NF_DEC_STREAM_WARPS=14
BARGS="--config c3loop --net-model nvlink --steps 10"
run c3base
run c3w14 NF_DEC_STREAM_WARPS=14
run c3base2
run c3w142 NF_DEC_STREAM_WARPS=14
