#!/bin/bash
# QK-norm/RoPE + staged RMSNorm backward: micro A/B (new vs before), ncu of
# the new kernels, the parity suites touching them (in one process, as the
# driver runs them), and the C3 bench line A/B.
T=${T:-qkfin}
mkdir -p gpurun_out
: > gpurun_out/${T}.jsonl
for r in 1 2; do
  RP_LIB=ab_libs/lib_before_qk.so timeout 300 python tools/bench_qk.py >> gpurun_out/${T}.jsonl 2>> gpurun_out/${T}.err
  RP_LIB=ab_libs/rnreg.so timeout 300 python tools/bench_qk.py >> gpurun_out/${T}.jsonl 2>> gpurun_out/${T}.err
  timeout 300 python tools/bench_qk.py >> gpurun_out/${T}.jsonl 2>> gpurun_out/${T}.err
done
for k in qk_norm_rope_fwd qk_norm_rope_bwd rmsnorm_bwd_staged; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:${k}_kernel -s 3 -c 1 \
    -o gpurun_out/${T}_ncu_$k -f python tools/bench_qk.py > gpurun_out/${T}_ncu_$k.log 2>&1
done
timeout 1500 python -m pytest tests/test_kernels_gpu.py tests/test_runtime_8b_gpu.py tests/test_runtime_gpu.py -m gpu -q -s -rA -p no:cacheprovider > gpurun_out/${T}_pytest.txt 2>&1
echo "pytest exit $?" >> gpurun_out/${T}_pytest.txt
for r in 1 2; do
  timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-variants > gpurun_out/${T}_bench_new_$r.json 2> gpurun_out/${T}_bench_new_$r.err
  RP_LIB=ab_libs/lib_before_qk.so timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-variants > gpurun_out/${T}_bench_old_$r.json 2> gpurun_out/${T}_bench_old_$r.err
done
