# 8B OVERLAP step: CTA pairs on tied schedules (default) vs single-CTA tiles for the narrow-N GEMMs (O, Down, KQV)
run() { tag=$1; shift; echo "== $tag" >> gpurun_out/r2n_ab_pairminn.log; env "$@" timeout 600 python bench.py --no-cpu-baseline --no-parity --steps 20 >> gpurun_out/r2n_ab_pairminn.log 2>&1; }
run base
run minn8192 NF_GEMM_PAIR_MINN=8192
run base2
run minn8192b NF_GEMM_PAIR_MINN=8192
run base3
run minn8192c NF_GEMM_PAIR_MINN=8192
