#!/bin/bash
# pass N: runtime suites after the trainable-region AdamW output buffers,
# one profiled 8B step (per-kernel-class breakdown), C5 reduced-depth bench
TAG=${1:-r2n}
mkdir -p gpurun_out
: > gpurun_out/${TAG}_pytest.txt
for f in tests/test_runtime_gpu.py tests/test_runtime_moe_gpu.py tests/test_protocol_gpu.py; do
  timeout 1200 python -m pytest $f -m gpu -q -s -rA -p no:cacheprovider >> gpurun_out/${TAG}_pytest.txt 2>&1
  echo "pytest $f exit $?" >> gpurun_out/${TAG}_pytest.txt
done
timeout 900 python tools/step_profile.py --warmup 3 --out gpurun_out/${TAG}_prof.npz > gpurun_out/${TAG}_step_profile.json 2>&1
timeout 120 python tools/step_breakdown.py gpurun_out/${TAG}_prof.npz 40 > gpurun_out/${TAG}_step_breakdown.txt 2>&1
timeout 1500 python bench.py --model qwen3-235b-a22b-l8 --seq 31744 --micro-batches 4 --lora-rank 32 \
  --lora-alpha 64 --steps 4 --warmup 2 --no-variants --no-cpu-baseline \
  --report-dir gpurun_out/${TAG}_report > gpurun_out/${TAG}_bench_c5.json 2> gpurun_out/${TAG}_bench_c5.err
echo "bench exit $?" >> gpurun_out/${TAG}_bench_c5.err
ls -la gpurun_out | tail -4
