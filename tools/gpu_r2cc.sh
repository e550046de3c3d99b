#!/bin/bash
# pass CC: qkv GEMM with fused QK-norm/RoPE — bit-exactness + parity tests, same-box A/B
TAG=${1:-r2cc}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_gemm_gpu.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_kernel_tests.txt 2>&1
timeout 900 python -m pytest tests/test_runtime_gpu.py -m gpu -q -x -p no:cacheprovider > gpurun_out/${TAG}_runtime_tests.txt 2>&1
timeout 1200 python -m pytest tests/test_runtime_8b_gpu.py -m gpu -q -s -x -k "host_offloaded" -p no:cacheprovider > gpurun_out/${TAG}_8b_tests.txt 2>&1
: > gpurun_out/${TAG}_ab.jsonl
run() {
  if [ -n "$2" ]; then export RP_LIB=$PWD/ab_libs/$2; else unset RP_LIB; fi
  timeout 900 python bench.py --steps 12 --warmup 3 --no-variants --no-cpu-baseline 2>> gpurun_out/${TAG}_$1.err \
    | sed "s/^/{\"lib\": \"$1\", \"r\": /; s/\$/}/" >> gpurun_out/${TAG}_ab.jsonl
}
for i in 1 2; do
  run head lib_gemmpdl.so
  run qkfused ""
done
ls -la gpurun_out | tail -3
