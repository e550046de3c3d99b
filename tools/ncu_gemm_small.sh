#!/bin/bash
# ncu --set full of the K=4096 GEMMs that run below the gate/up GEMM's rate in step (o, qkv fwd)
T=${T:-r2z10}
mkdir -p gpurun_out
for g in o_fwd qkv_fwd; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_pair -s 6 -c 1 \
    -o gpurun_out/${T}_ncu_$g -f python tools/bench_gemm.py $g > gpurun_out/${T}_ncu_$g.log 2>&1
done
