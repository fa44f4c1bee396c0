# decode stream kernel variants: warps, four S chains (VAR 1), look-ahead (VAR 2), both (VAR 3);
# the first SM budget of each attn_micro run is a warm-up (first-launch effects)
for wv in 12:0 12:1 8:0 8:1 8:2 8:3 12:2 12:0; do
  w=${wv%:*}; v=${wv#*:}
  echo "== W=$w VAR=$v" >> gpurun_out/decvar.log
  NF_DEC_STREAM_WARPS=$w NF_DEC_STREAM_VAR=$v timeout 300 python tools/attn_micro.py 16,16,32,148 5 >> gpurun_out/decvar.log 2>&1
  NF_DEC_STREAM_WARPS=$w NF_DEC_STREAM_VAR=$v SHAPE=c3rank timeout 300 python tools/attn_micro.py 16,16,32,148 5 >> gpurun_out/decvar.log 2>&1
done
