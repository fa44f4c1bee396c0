# step-level A/B of the smem-staged split-tile fix-up (NF_GEMM_SKSMEM=1) on the 8B OVERLAP step and the TP8-rank proxy
run() { tag=$1; shift; echo "== $tag" >> gpurun_out/r2n_ab_sksmem_step.log; env "$@" timeout 600 python bench.py --no-cpu-baseline --no-parity $BARGS >> gpurun_out/r2n_ab_sksmem_step.log 2>&1; }
BARGS="--steps 20"
run base
run sks NF_GEMM_SKSMEM=1
run base2
run sks2 NF_GEMM_SKSMEM=1
run base3
run sks3 NF_GEMM_SKSMEM=1
BARGS="--config c3loop --net-model nvlink --steps 10"
run c3base
run c3sks NF_GEMM_SKSMEM=1
run c3base2
run c3sks2 NF_GEMM_SKSMEM=1
