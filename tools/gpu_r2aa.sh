#!/bin/bash
TAG=${1:-r2aa}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_runtime_8b_gpu.py -m gpu -q -s -rA -k "lora" -p no:cacheprovider > gpurun_out/${TAG}_pytest.txt 2>&1
echo "exit $?" >> gpurun_out/${TAG}_pytest.txt
timeout 300 python -m pytest tests/test_kernels_gpu.py -m gpu -q -k "adamw" -p no:cacheprovider >> gpurun_out/${TAG}_pytest.txt 2>&1
ls -la gpurun_out | tail -2
