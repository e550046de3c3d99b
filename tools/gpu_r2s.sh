#!/bin/bash
TAG=${1:-r2s}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_runtime_235b_gpu.py -m gpu -q -s -rA -p no:cacheprovider > gpurun_out/${TAG}_pytest_235b.txt 2>&1
echo "exit $?" >> gpurun_out/${TAG}_pytest_235b.txt
ls -la gpurun_out | tail -2
