#!/bin/bash
T=${1:-it}
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gemm_gpu.py -q -x > gpurun_out/${T}_pytest_g.txt 2>&1; echo "exit $?" >> gpurun_out/${T}_pytest_g.txt
timeout 200 python tools/bench_gemm.py > gpurun_out/${T}_gemm.jsonl 2>&1
RP_GEMM_NO_TMA_EPI=1 timeout 200 python tools/bench_gemm.py gu_wgrad down_wgrad > gpurun_out/${T}_gemm_old.jsonl 2>&1
timeout 300 python -m pytest tests/test_runtime_gpu.py -q > gpurun_out/${T}_pytest_r.txt 2>&1; echo "exit $?" >> gpurun_out/${T}_pytest_r.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"gemm" -s 6 -c 1 \
  -o gpurun_out/${T}_full_gemm_gu_wgrad -f python tools/bench_gemm.py gu_wgrad > gpurun_out/${T}_ncu_wg.log 2>&1
if [ "$2" == "bench" ]; then
  timeout 900 python bench.py --report-dir gpurun_out > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
fi
