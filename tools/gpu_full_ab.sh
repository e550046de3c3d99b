mkdir -p gpurun_out
T=r01s25
: > gpurun_out/${T}_pytest_gpu.txt
for f in tests/test_kernels_gpu.py tests/test_gemm_gpu.py tests/test_runtime_gpu.py; do
  timeout 600 python -m pytest $f -m gpu -q >> gpurun_out/${T}_pytest_gpu.txt 2>&1
  echo "pytest $f exit $?" >> gpurun_out/${T}_pytest_gpu.txt
done
T=r01s25 bash tools/gpu_bench_ab.sh RP_GEMM_NO_SPLITK=1
