# decode S^T look-ahead with one V register set (NF_DEC_STREAM_VAR 4 / 5) vs the default
NF_DEC_STREAM_VAR=4 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "attention or decode or layer_c1 or 8b_full_batch" > gpurun_out/la2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/la2_tests.log
for wv in 12:0 12:4 12:5 8:4 12:0 12:4 12:5; do
  w=${wv%:*}; v=${wv#*:}
  echo "== W=$w VAR=$v" >> gpurun_out/la2_micro.log
  NF_DEC_STREAM_WARPS=$w NF_DEC_STREAM_VAR=$v timeout 300 python tools/attn_micro.py 16,16,32,48,148 5 >> gpurun_out/la2_micro.log 2>&1
  NF_DEC_STREAM_WARPS=$w NF_DEC_STREAM_VAR=$v SHAPE=c3rank timeout 300 python tools/attn_micro.py 16,16,32,148 5 >> gpurun_out/la2_micro.log 2>&1
done
