#!/bin/bash
TAG=${1:-r2k}
mkdir -p gpurun_out
CUDA_LAUNCH_BLOCKING=1 timeout 600 python tools/diag_c5_rt.py 16384 1 > gpurun_out/${TAG}_c5rt_16384.txt 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --model qwen3-1.7b --no-variants \
  --no-cpu-baseline > gpurun_out/${TAG}_bench_17b_n2.json 2> gpurun_out/${TAG}_bench_17b_n2.err
echo "exit $?" >> gpurun_out/${TAG}_bench_17b_n2.err
ls -la gpurun_out | tail -4
