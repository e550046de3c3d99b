#!/bin/bash
TAG=${1:-r2dd}
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_pair -s 6 -c 1 \
  -o gpurun_out/${TAG}_full_gu_wgrad -f python tools/bench_gemm.py gu_wgrad > gpurun_out/${TAG}_ncu_wgrad.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_pair -s 6 -c 1 \
  -o gpurun_out/${TAG}_full_down_wgrad -f python tools/bench_gemm.py down_wgrad > gpurun_out/${TAG}_ncu_dwgrad.log 2>&1
ls -la gpurun_out | tail -3
