#!/bin/bash
# GEMM tests + same-box A/B of a GEMM knob (arg: ENV=VAL)
KNOB=${1:-RP_GEMM_NO_SPLITK=1}
T=${2:-gab}
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gemm_gpu.py -q -x > gpurun_out/${T}_pytest_g.txt 2>&1; echo "exit $?" >> gpurun_out/${T}_pytest_g.txt
for r in 1 2; do
timeout 200 python tools/bench_gemm.py > gpurun_out/${T}_gemm_new_$r.jsonl 2>&1
env $KNOB timeout 200 python tools/bench_gemm.py > gpurun_out/${T}_gemm_old_$r.jsonl 2>&1
done
