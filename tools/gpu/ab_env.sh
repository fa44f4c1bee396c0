# A/B of launch-level options on the default 8B step and the TP8-rank proxy (bench JSON lines)
run() { tag=$1; shift; echo "== $tag" >> gpurun_out/ab_env.log; env "$@" timeout 600 python bench.py --no-cpu-baseline --no-parity $BARGS >> gpurun_out/ab_env.log 2>&1; }
BARGS=""
run base0
run cg2 NF_GEMM_FORCE=3
run pdl NF_PDL=1
run cg2pdl NF_GEMM_FORCE=3 NF_PDL=1
run base1
BARGS="--config c3loop --steps 10"
run c3base
run c3pdl NF_PDL=1
