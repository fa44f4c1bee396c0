#!/bin/bash
# Functional run of bench.py's tensor-parallel path with N ranks sharing ONE GPU
# (not a performance measurement): launch as
#   nvidia-cuda-mps-control -d   # ranks share the GPU concurrently
#   python -m torch.distributed.run --no-python --nproc-per-node 2 --master-addr 127.0.0.1 \
#       --master-port 29555 tools/tp_on_one_gpu.sh --gpus 2 --layers 2 --steps 3 --warmup 3
# Every rank uses device 0; each announces its own NCCL host id so NCCL accepts two
# ranks on one device (they talk through NCCL's socket transport on loopback).
export NCCL_HOSTID="nf-tp1gpu-${RANK}"
export NCCL_SOCKET_IFNAME=lo
export NCCL_IB_DISABLE=1
export LOCAL_RANK=0
cd "$(dirname "$0")/.." && exec python bench.py "$@"
