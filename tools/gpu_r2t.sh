#!/bin/bash
TAG=${1:-r2t}
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -k "flash" -p no:cacheprovider > gpurun_out/${TAG}_attn_tests.txt 2>&1
timeout 300 python tools/attn_fwd_variant_ab.py > gpurun_out/${TAG}_fwd_ab.jsonl 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"attn_fwd_pp2" -s 3 -c 1 \
    -o gpurun_out/${TAG}_full_attn_fwd_pp2 -f python tools/bench_kernels.py attn > gpurun_out/${TAG}_ncu.log 2>&1
ls -la gpurun_out | tail -3
