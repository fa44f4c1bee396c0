# functional multi-process TP runs of bench.py on ONE GPU (MPS, NCCL socket transport): not performance
nvidia-cuda-mps-control -d; sleep 2
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --no-python --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2955$n \
    tools/tp_on_one_gpu.sh --gpus $n --layers 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2n_bench_tp${n}_on_one_gpu_functional.log 2>&1
  echo "rc=$?" >> gpurun_out/r2n_bench_tp${n}_on_one_gpu_functional.log
done
timeout 900 python -m torch.distributed.run --no-python --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29560 \
  tools/tp_on_one_gpu.sh --gpus 2 --layers 2 --steps 3 --warmup 3 --no-cpu-baseline --fused-ar > gpurun_out/r2n_bench_tp2_fused_on_one_gpu_functional.log 2>&1
echo "rc=$?" >> gpurun_out/r2n_bench_tp2_fused_on_one_gpu_functional.log
timeout 600 python -m torch.distributed.run --no-python --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 \
  tools/tp_on_one_gpu.sh --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/r2n_bench_ref_tp2.log 2>&1
echo "rc=$?" >> gpurun_out/r2n_bench_ref_tp2.log
echo quit | nvidia-cuda-mps-control
