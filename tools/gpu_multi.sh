#!/bin/bash
# multi-worker bench paths on one GPU (logical workers share the device): the
# torchrun launch, the single controller on rank 0, hand-offs, recompute slots
T=${1:-mw}
mkdir -p gpurun_out
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 29533 bench.py --gpus $N --model qwen3-1.7b --steps 4 --warmup 3 --no-cpu-baseline \
    > gpurun_out/${T}_bench17_n$N.json 2> gpurun_out/${T}_bench17_n$N.err
  echo "exit $?" >> gpurun_out/${T}_bench17_n$N.err
done
timeout 600 python bench.py --gpus 1 --model qwen3-1.7b --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench17_n1.json 2> gpurun_out/${T}_bench17_n1.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err
