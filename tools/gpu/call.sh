for f in "" "--fused-ar" "" "--fused-ar"; do timeout 900 python bench.py --config c3loop --no-cpu-baseline --no-ablation --steps 10 $f 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('[$f]', round(d['ms_per_step'],2), round(d['value']), d['clocks']['sm_mhz'], (d['plan'].get('collectives') or {}).get('peer_wait_timeouts'), round(d['per_op']['net']['ms_per_step'],2))"; done > gpurun_out/r2g_c3loop_fused_ab2.log 2>&1
timeout 900 python -m pytest tests/test_gpu_tp.py -x -q -k "fused" 2>&1 | tail -1 >> gpurun_out/r2g_c3loop_fused_ab2.log
cat gpurun_out/r2g_c3loop_fused_ab2.log
