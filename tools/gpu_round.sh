#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, kernel micro-benches, ncu launch list
# of the bench command and full captures of the top kernels. Outputs in gpurun_out/.
# Usage: tools/gpu_round.sh [tag] [skip-tests] [skip-ncu]
TAG=${1:-r}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
if [ "$2" != "skip-tests" ]; then
  : > gpurun_out/${TAG}_pytest_gpu.txt
  for f in tests/test_kernels_gpu.py tests/test_gemm_gpu.py tests/test_runtime_gpu.py; do
    timeout 420 python -m pytest $f -m gpu -q >> gpurun_out/${TAG}_pytest_gpu.txt 2>&1
    echo "pytest $f exit $?" >> gpurun_out/${TAG}_pytest_gpu.txt
  done
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
  echo "smoke exit $?" >> gpurun_out/${TAG}_smoke.txt
fi
timeout 900 python bench.py --report-dir gpurun_out > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench exit $?" >> gpurun_out/${TAG}_bench.err
timeout 300 python tools/bench_gemm.py > gpurun_out/${TAG}_gemm.jsonl 2>&1
timeout 300 python tools/bench_kernels.py > gpurun_out/${TAG}_kernels.jsonl 2>&1
timeout 300 python tools/bench_kernels.py attn > gpurun_out/${TAG}_attn.jsonl 2>&1
if [ "$3" != "skip-ncu" ]; then
  timeout 1500 ncu --replay-mode application --metrics gpu__time_duration.sum --clock-control none \
    -s 47000 -c 3000 --csv --log-file gpurun_out/${TAG}_launches_8b.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu_bench.log 2>&1
  echo "ncu launch list exit $?" >> gpurun_out/${TAG}_ncu_bench.log
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"gemm_pair_kernel" -s 6 -c 1 \
    -o gpurun_out/${TAG}_full_gemm_gu_fwd -f python tools/bench_gemm.py gu_fwd > gpurun_out/${TAG}_ncu_g1.log 2>&1
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"attn_fwd_tc" -s 3 -c 1 \
    -o gpurun_out/${TAG}_full_attn_fwd -f python tools/bench_kernels.py attn > gpurun_out/${TAG}_ncu_a1.log 2>&1
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"attn_bwd_dkv" -s 3 -c 1 \
    -o gpurun_out/${TAG}_full_attn_dkv -f python tools/bench_kernels.py attn > gpurun_out/${TAG}_ncu_a2.log 2>&1
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"adamw" -s 3 -c 1 \
    -o gpurun_out/${TAG}_full_adamw -f python tools/bench_kernels.py > gpurun_out/${TAG}_ncu_k1.log 2>&1
fi
ls -la gpurun_out | tail -30
