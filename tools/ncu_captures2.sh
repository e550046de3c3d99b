#!/bin/bash
# launch list of the bench command (application replay keeps host memory flat),
# plus per-kernel times of the attention backward pair
mkdir -p gpurun_out
timeout 1200 ncu --replay-mode application --metrics gpu__time_duration.sum --clock-control none \
  -s 47000 -c 2500 --csv --log-file gpurun_out/launches_8b.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"attn_fwd_tc|attn_bwd_dkv|attn_bwd_dq|delta_kernel" -s 8 -c 8 --csv \
  --log-file gpurun_out/launches_attn.csv python tools/bench_kernels.py > gpurun_out/ncu_attn2.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"attn_bwd_dq" -s 5 -c 1 \
  -o gpurun_out/prof_attn_dq python tools/bench_kernels.py > gpurun_out/ncu_attn3.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"attn_bwd_dkv" -s 5 -c 1 \
  -o gpurun_out/prof_attn_dkv python tools/bench_kernels.py > gpurun_out/ncu_attn4.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"gemm_pair_kernel" -s 6 -c 1 \
  -o gpurun_out/prof_gemm_pair_gu_fwd python tools/bench_gemm.py gu_fwd > gpurun_out/ncu_gemm3.log 2>&1
ls -la gpurun_out | tail -20
