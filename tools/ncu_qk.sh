#!/bin/bash
# ncu full captures of the QK-norm/RoPE kernels (Qwen3-8B shapes, tools/bench_qk.py)
T=${T:-ncuqk}
mkdir -p gpurun_out
for k in qk_norm_rope_fwd qk_norm_rope_bwd rmsnorm_fwd; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:${k}_kernel -s 3 -c 1 \
    -o gpurun_out/${T}_head_$k -f python tools/bench_qk.py > gpurun_out/${T}_head_$k.log 2>&1
done
for k in qk_norm_rope_fwd qk_norm_rope_bwd; do
  RP_LIB=ab_libs/lib_before_qk.so timeout 300 ncu --set full --clock-control none --import-source on -k regex:${k}_kernel -s 3 -c 1 \
    -o gpurun_out/${T}_old_$k -f python tools/bench_qk.py > gpurun_out/${T}_old_$k.log 2>&1
done
