#!/bin/bash
# pass V: C5 reduced depth with the LoRA-exact residency (fused stage, no recompute)
TAG=${1:-r2v}
mkdir -p gpurun_out
timeout 1500 python bench.py --model qwen3-235b-a22b-l8 --seq 31744 --micro-batches 4 --lora-rank 32 \
  --lora-alpha 64 --steps 4 --warmup 2 --no-variants --no-cpu-baseline --host-publish --residency-factor 1.0 \
  --report-dir gpurun_out/${TAG}_report_c5 > gpurun_out/${TAG}_bench_c5.json 2> gpurun_out/${TAG}_bench_c5.err
echo "bench exit $?" >> gpurun_out/${TAG}_bench_c5.err
ls -la gpurun_out | tail -3
