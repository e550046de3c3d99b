#!/bin/bash
T=${1:-it}
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gemm_gpu.py -q -x > gpurun_out/${T}_pytest_g.txt 2>&1; echo "exit $?" >> gpurun_out/${T}_pytest_g.txt
RP_GEMM_TILE_N=128 timeout 300 python -m pytest tests/test_gemm_gpu.py -q -x > gpurun_out/${T}_pytest_g128.txt 2>&1; echo "exit $?" >> gpurun_out/${T}_pytest_g128.txt
timeout 200 python tools/bench_gemm.py > gpurun_out/${T}_gemm.jsonl 2>&1
RP_GEMM_TILE_N=256 timeout 200 python tools/bench_gemm.py > gpurun_out/${T}_gemm256.jsonl 2>&1
RP_GEMM_TILE_N=128 timeout 200 python tools/bench_gemm.py > gpurun_out/${T}_gemm128.jsonl 2>&1
if [ "$2" == "bench" ]; then
  timeout 300 python -m pytest tests/test_runtime_gpu.py -q > gpurun_out/${T}_pytest_r.txt 2>&1; echo "exit $?" >> gpurun_out/${T}_pytest_r.txt
  timeout 900 python bench.py --report-dir gpurun_out > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
fi
