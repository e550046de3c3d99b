#!/bin/bash
# pass Z: streamed-chunk AdamW on 64 blocks — tests, same-box A/B vs HEAD
TAG=${1:-r2z}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_runtime_gpu.py -m gpu -q -x -k "adamw or parity" -p no:cacheprovider > gpurun_out/${TAG}_tests.txt 2>&1
: > gpurun_out/${TAG}_ab.jsonl
run() {
  if [ -n "$2" ]; then export RP_LIB=$PWD/ab_libs/$2; else unset RP_LIB; fi
  timeout 900 python bench.py --steps 12 --warmup 3 --no-variants --no-cpu-baseline 2>> gpurun_out/${TAG}_$1.err \
    | sed "s/^/{\"lib\": \"$1\", \"r\": /; s/\$/}/" >> gpurun_out/${TAG}_ab.jsonl
}
for i in 1 2; do
  run head lib_gemmpdl.so
  run cap64 ""
done
ls -la gpurun_out | tail -3
