# TP8-rank proxy with the modeled NVLink link time (ring bytes / 725 GB/s per collective):
# default TP plan, the refined plan, and the plain loopback for reference
timeout 900 python bench.py --config c3loop --net-model nvlink --steps 10 --no-cpu-baseline > gpurun_out/r2l_c3loop_nvlink.log 2>&1
timeout 1500 python bench.py --config c3loop --net-model nvlink --steps 10 --no-cpu-baseline --plan refine > gpurun_out/r2l_c3loop_nvlink_refine.log 2>&1
timeout 900 python bench.py --config c3loop --net-model nvlink --steps 10 --no-cpu-baseline --shares 1,1,1,1 > gpurun_out/r2l_c3loop_nvlink_4way.log 2>&1
