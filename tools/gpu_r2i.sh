#!/bin/bash
TAG=${1:-r2i}
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -k "flash" -p no:cacheprovider > gpurun_out/${TAG}_attn_tests.txt 2>&1
timeout 300 python tools/diag_c5.py > gpurun_out/${TAG}_diag_c5.txt 2>&1
timeout 300 compute-sanitizer --print-limit 5 python -c "
import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tools')
from diag_c5 import attn
attn(31744, 31744, 64, 4)" > gpurun_out/${TAG}_sanitizer.txt 2>&1
: > gpurun_out/${TAG}_qk_ab.jsonl
for i in 1 2; do
  RP_LIB=$PWD/ab_libs/lib_head.so timeout 200 python tools/bench_kernels.py | sed 's/^/{"lib": "head", "r": /; s/$/}/' >> gpurun_out/${TAG}_qk_ab.jsonl 2>&1
  timeout 200 python tools/bench_kernels.py | sed 's/^/{"lib": "new", "r": /; s/$/}/' >> gpurun_out/${TAG}_qk_ab.jsonl 2>&1
done
ls -la gpurun_out | tail -5
