#!/bin/bash
TAG=${1:-r2m}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py -q -p no:cacheprovider -x > gpurun_out/${TAG}_gemm.txt 2>&1
timeout 1500 python bench.py --model qwen3-235b-a22b-l8 --seq 31744 --micro-batches 4 --lora-rank 32 \
  --lora-alpha 64 --steps 4 --warmup 2 --no-variants --no-cpu-baseline \
  --report-dir gpurun_out/${TAG}_report > gpurun_out/${TAG}_bench_c5.json 2> gpurun_out/${TAG}_bench_c5.err
echo "bench exit $?" >> gpurun_out/${TAG}_bench_c5.err
ls -la gpurun_out | tail -3
