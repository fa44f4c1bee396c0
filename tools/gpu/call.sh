NF_GREEN=0 timeout 1200 ncu --set full --import-source on --clock-control none -k regex:gemm_tcgen05 -s 407 -c 4 -o gpurun_out/r2k_8b_seq_gemms python bench.py --mode sequential --steps 1 --warmup 3 --ncu > gpurun_out/r2k_ncu_8b_seq.out 2>&1
tail -2 gpurun_out/r2k_ncu_8b_seq.out
