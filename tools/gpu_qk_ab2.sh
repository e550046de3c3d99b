#!/bin/bash
T=${T:-qkab5}
mkdir -p gpurun_out
: > gpurun_out/${T}.jsonl
for r in 1 2 3; do
  RP_LIB=ab_libs/qkc2.so timeout 300 python tools/bench_qk.py >> gpurun_out/${T}.jsonl 2>> gpurun_out/${T}.err
  timeout 300 python tools/bench_qk.py >> gpurun_out/${T}.jsonl 2>> gpurun_out/${T}.err
done
timeout 600 python -m pytest tests/test_kernels_gpu.py -m gpu -q -k "qk or rmsnorm" > gpurun_out/${T}_pytest.txt 2>&1
