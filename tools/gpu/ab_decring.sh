# decode stream kernel: warps x ring depth (bytes in flight per SM) A/B, 8B and 70B-TP8-rank decode batches
for w in 12 9 7 8 6 13; do
  echo "== W=$w" >> gpurun_out/decring.log
  NF_DEC_STREAM_WARPS=$w timeout 300 python tools/attn_micro.py 16,32,48,148 5 >> gpurun_out/decring.log 2>&1
  NF_DEC_STREAM_WARPS=$w SHAPE=c3rank timeout 300 python tools/attn_micro.py 16,32,148 5 >> gpurun_out/decring.log 2>&1
done
