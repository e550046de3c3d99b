#!/bin/bash
# ncu evidence for profiles/ (run under gpurun; one GPU). Never a bench number.
set -x
mkdir -p gpurun_out
# 1. launch list of the bench command: skip init + 3 warm-up steps, capture 2500 launches of a timed step
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 47000 -c 2500 --csv \
  --log-file gpurun_out/launches_8b.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
  > gpurun_out/ncu_bench.log 2>&1
# 2. full capture of the top kernel (tcgen05 GEMM, gate_up forward shape) and the attention kernels
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 6 -c 1 \
  -o gpurun_out/prof_gemm_gu_fwd python tools/bench_gemm.py gu_fwd > gpurun_out/ncu_gemm.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 6 -c 1 \
  -o gpurun_out/prof_gemm_gu_wgrad python tools/bench_gemm.py gu_wgrad > gpurun_out/ncu_gemm2.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:attn_ -s 12 -c 4 \
  -o gpurun_out/prof_attn python tools/bench_kernels.py > gpurun_out/ncu_attn.log 2>&1
ls -la gpurun_out
