#!/bin/bash
# QK-norm/RoPE same-box A/B over ab_libs variants (two passes, interleaved)
T=${T:-qkab}
mkdir -p gpurun_out
: > gpurun_out/${T}.jsonl
for r in 1 2; do
  for lib in ab_libs/lib_before_qk.so ab_libs/qk*.so head; do
    if [ "$lib" = head ]; then timeout 300 python tools/bench_qk.py >> gpurun_out/${T}.jsonl 2>> gpurun_out/${T}.err
    else RP_LIB=$lib timeout 300 python tools/bench_qk.py >> gpurun_out/${T}.jsonl 2>> gpurun_out/${T}.err; fi
  done
done
timeout 600 python -m pytest tests/test_kernels_gpu.py -m gpu -q -k "qk" > gpurun_out/${T}_pytest.txt 2>&1
for k in qk_norm_rope_fwd qk_norm_rope_bwd; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:${k}_kernel -s 3 -c 1 \
    -o gpurun_out/${T}_ncu_$k -f python tools/bench_qk.py > gpurun_out/${T}_ncu_$k.log 2>&1
done
