#!/bin/bash
# Round-2 GPU pass: all -m gpu suites with printed margins (-s), smoke, a
# short 8B bench, then the 8B-width step parity suite. Outputs in gpurun_out/.
TAG=${1:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
nproc > gpurun_out/${TAG}_nproc.txt
: > gpurun_out/${TAG}_pytest_gpu.txt
for f in tests/test_kernels_gpu.py tests/test_gemm_gpu.py tests/test_runtime_gpu.py; do
  timeout 900 python -m pytest $f -m gpu -q -s -rA -p no:cacheprovider >> gpurun_out/${TAG}_pytest_gpu.txt 2>&1
  echo "pytest $f exit $?" >> gpurun_out/${TAG}_pytest_gpu.txt
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
echo "smoke exit $?" >> gpurun_out/${TAG}_smoke.txt
timeout 900 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench exit $?" >> gpurun_out/${TAG}_bench.err
timeout 900 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --host-optimizer > gpurun_out/${TAG}_bench_host.json 2> gpurun_out/${TAG}_bench_host.err
echo "bench exit $?" >> gpurun_out/${TAG}_bench_host.err
if [ "$2" != "skip-8b" ]; then
  timeout 2700 python -m pytest tests/test_runtime_8b_gpu.py -m gpu -q -s -rA -p no:cacheprovider > gpurun_out/${TAG}_pytest_8b.txt 2>&1
  echo "pytest 8b exit $?" >> gpurun_out/${TAG}_pytest_8b.txt
fi
ls -la gpurun_out | tail -20
