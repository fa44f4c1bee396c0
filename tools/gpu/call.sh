export NF_PEER_TIMEOUT_MS=5000
for i in 1 2; do timeout 1200 python -m pytest tests/test_gpu_tp.py -x -q -k "fused" 2>&1 | grep -E "timed out|passed|failed|Error|not taken" | head -4; done
timeout 900 python -m pytest tests/test_gpu_nccl.py -x -q 2>&1 | tail -2
for f in "" "--fused-ar"; do timeout 900 python bench.py --config c3loop --no-cpu-baseline --no-ablation --steps 10 $f 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c3loop [$f]', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['plan'].get('collectives'))"; done
