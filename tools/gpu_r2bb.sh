#!/bin/bash
# pass BB: BASELINE configs[3] at reduced depth (Qwen3-32B shapes, 12 of 64 layers, seq 8K)
TAG=${1:-r2bb}
mkdir -p gpurun_out
free -g > gpurun_out/${TAG}_mem.txt
timeout 1500 python bench.py --model qwen3-32b-l12 --seq 8192 --micro-batches 16 --steps 3 --warmup 3 \
  --no-variants --no-cpu-baseline --report-dir gpurun_out/${TAG}_report > gpurun_out/${TAG}_bench_c4.json 2> gpurun_out/${TAG}_bench_c4.err
echo "bench exit $?" >> gpurun_out/${TAG}_bench_c4.err
ls -la gpurun_out | tail -3
