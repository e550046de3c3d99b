#!/bin/bash
TAG=${1:-r2l}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py -q -p no:cacheprovider -k "long_k" -rA > gpurun_out/${TAG}_gemm_longk.txt 2>&1
CUDA_LAUNCH_BLOCKING=1 timeout 600 python tools/diag_c5_rt.py 16384 1 > gpurun_out/${TAG}_c5rt_16384.txt 2>&1
ls -la gpurun_out | tail -3
