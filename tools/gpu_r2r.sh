#!/bin/bash
# pass R: whole GPU suite + smoke + default bench line + C5 (paper publication path)
TAG=${1:-r2r}
bash tools/gpu_r2d.sh ${TAG}
timeout 1500 python bench.py --model qwen3-235b-a22b-l8 --seq 31744 --micro-batches 4 --lora-rank 32 \
  --lora-alpha 64 --steps 4 --warmup 2 --no-variants --no-cpu-baseline --host-publish \
  --report-dir gpurun_out/${TAG}_report_c5 > gpurun_out/${TAG}_bench_c5.json 2> gpurun_out/${TAG}_bench_c5.err
echo "bench exit $?" >> gpurun_out/${TAG}_bench_c5.err
ls -la gpurun_out | tail -3
