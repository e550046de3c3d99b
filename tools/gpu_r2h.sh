#!/bin/bash
# Round-2 pass H: QK-norm/RoPE A/B (HEAD library vs the batched-load kernels,
# same box, alternating), kernel tests, and the reduced-depth C5 MoE bench.
TAG=${1:-r2h}
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_kernel_tests.txt 2>&1
: > gpurun_out/${TAG}_qk_ab.jsonl
for i in 1 2; do
  RP_LIB=$PWD/ab_libs/lib_head.so timeout 200 python tools/bench_kernels.py | sed 's/^/{"lib": "head", "r": /; s/$/}/' >> gpurun_out/${TAG}_qk_ab.jsonl 2>&1
  timeout 200 python tools/bench_kernels.py | sed 's/^/{"lib": "new", "r": /; s/$/}/' >> gpurun_out/${TAG}_qk_ab.jsonl 2>&1
done
timeout 1500 python bench.py --model qwen3-235b-a22b-l8 --seq 31744 --micro-batches 4 --lora-rank 32 \
  --lora-alpha 64 --steps 4 --warmup 2 --no-variants --no-cpu-baseline \
  --report-dir gpurun_out/${TAG}_report > gpurun_out/${TAG}_bench_c5.json 2> gpurun_out/${TAG}_bench_c5.err
echo "bench exit $?" >> gpurun_out/${TAG}_bench_c5.err
ls -la gpurun_out | tail -6
