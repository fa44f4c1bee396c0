# one-step kernel timelines of the TP8-rank proxy (modeled link time): OVERLAP (default plan) and SEQUENTIAL
timeout 900 python bench.py --config c3loop --net-model nvlink --steps 3 --no-cpu-baseline --no-ablation --timeline gpurun_out/tl_overlap.csv > gpurun_out/tl_overlap.log 2>&1
timeout 900 python bench.py --config c3loop --net-model nvlink --steps 3 --no-cpu-baseline --no-ablation --mode sequential --timeline gpurun_out/tl_seq.csv > gpurun_out/tl_seq.log 2>&1
timeout 900 python bench.py --steps 3 --no-cpu-baseline --no-ablation --timeline gpurun_out/tl_8b.csv > gpurun_out/tl_8b.log 2>&1
