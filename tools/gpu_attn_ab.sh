#!/bin/bash
# attention kernel tests + same-box A/B of an attention knob (arg: ENV=VAL)
KNOB=${1:-RP_ATTN_DQ_PP=1}
T=${2:-ab}
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -k "attention" > gpurun_out/${T}_pytest_k.txt 2>&1; echo "exit $?" >> gpurun_out/${T}_pytest_k.txt
for r in 1 2; do
timeout 200 python tools/bench_kernels.py attn > gpurun_out/${T}_attn_new_$r.jsonl 2>&1
env $KNOB timeout 200 python tools/bench_kernels.py attn > gpurun_out/${T}_attn_old_$r.jsonl 2>&1
done
