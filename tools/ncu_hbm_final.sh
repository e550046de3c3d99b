#!/bin/bash
# ncu --set full of the final HBM kernels (Qwen3-8B shapes, tools/bench_qk.py)
T=${T:-r2z9}
mkdir -p gpurun_out
for k in qk_norm_rope_fwd qk_norm_rope_bwd rmsnorm_bwd_staged rmsnorm_fwd; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:${k}_kernel -s 3 -c 1 \
    -o gpurun_out/${T}_ncu_$k -f python tools/bench_qk.py > gpurun_out/${T}_ncu_$k.log 2>&1
done
