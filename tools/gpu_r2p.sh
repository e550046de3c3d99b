#!/bin/bash
# pass P: same-box A/B of the C3 headline: HEAD (2-slot ring), 3-slot ring,
# 3-slot ring + in-place publication at N=1 (current tree); 12 steps each
TAG=${1:-r2p}
mkdir -p gpurun_out
: > gpurun_out/${TAG}_ab.jsonl
run() {  # $1 label, $2 lib or ""
  if [ -n "$2" ]; then export RP_LIB=$PWD/ab_libs/$2; else unset RP_LIB; fi
  timeout 900 python bench.py --steps 12 --warmup 3 --no-variants --no-cpu-baseline 2>> gpurun_out/${TAG}_$1.err \
    | sed "s/^/{\"lib\": \"$1\", \"r\": /; s/\$/}/" >> gpurun_out/${TAG}_ab.jsonl
}
for i in 1 2; do
  run ring2 lib_ring2.so
  run ring3 lib_ring3.so
  run direct ""
done
timeout 600 python -m pytest tests/test_protocol_gpu.py tests/test_runtime_gpu.py -m gpu -q -x -p no:cacheprovider > gpurun_out/${TAG}_pytest.txt 2>&1
ls -la gpurun_out | tail -3
