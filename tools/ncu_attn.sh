#!/bin/bash
# attention kernels: tests, CUDA-event bench, per-kernel ncu times, full captures of dkv / dq
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q -k "tc" > gpurun_out/k_test.txt 2>&1
timeout 200 python tools/bench_kernels.py attn > gpurun_out/k_bench.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"attn_bwd_dkv|attn_bwd_dq|[^_]delta_kernel|dkv_cast" -c 12 --csv \
  --log-file gpurun_out/launches_attn.csv python tools/bench_kernels.py attn > gpurun_out/ncu_attn2.log 2>&1
if [ "$1" == "full" ]; then
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"attn_bwd_dq" -s 5 -c 1 \
  -o gpurun_out/prof_attn_dq python tools/bench_kernels.py attn > gpurun_out/ncu_attn3.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"attn_bwd_dkv" -s 5 -c 1 \
  -o gpurun_out/prof_attn_dkv python tools/bench_kernels.py attn > gpurun_out/ncu_attn4.log 2>&1
fi
