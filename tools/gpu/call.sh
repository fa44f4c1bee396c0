export NF_PEER_TIMEOUT_MS=5000
for i in 1 2 3; do echo "run $i"; timeout 900 python -m pytest tests/test_gpu_tp.py -x -q -k "fused" 2>&1 | grep -E "timed out|passed|failed|Error:|not taken" | head -3; done > gpurun_out/r2g_fused_final.log 2>&1
timeout 900 python -m pytest tests/test_gpu_nccl.py -x -q 2>&1 | tail -2 >> gpurun_out/r2g_fused_final.log
cat gpurun_out/r2g_fused_final.log
