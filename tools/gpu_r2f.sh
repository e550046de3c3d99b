#!/bin/bash
TAG=${1:-r2f}
mkdir -p gpurun_out
timeout 300 python tools/attn_fwd_ab.py 0 1 2 > gpurun_out/${TAG}_attn_fwd_ab.jsonl 2>&1
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -k "tc" -p no:cacheprovider > gpurun_out/${TAG}_attn_tests.txt 2>&1
timeout 900 python -m pytest tests/test_runtime_8b_gpu.py -q -s -k "n2" -p no:cacheprovider > gpurun_out/${TAG}_n2_a.txt 2>&1
timeout 600 python -m pytest tests/test_runtime_gpu.py -q -s -k "pooled" -p no:cacheprovider > gpurun_out/${TAG}_pooled.txt 2>&1
ls -la gpurun_out | tail -6
