timeout 600 python tools/tma_probe.py 12:2:0,12:2:3,12:2:4,8:2:3,8:2:4,8:1:4,24:1:0,24:1:4 16,32,48 > gpurun_out/r2f_tma_probe_lsu.log 2>&1
