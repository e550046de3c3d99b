#!/bin/bash
# pass O: same-box A/B of the 3-slot optimizer ring (C3 headline, host-offloaded)
TAG=${1:-r2o}
mkdir -p gpurun_out
: > gpurun_out/${TAG}_ab.jsonl
for i in 1 2; do
  RP_LIB=$PWD/ab_libs/lib_ring2.so timeout 900 python bench.py --steps 8 --warmup 3 --no-variants --no-cpu-baseline 2>/dev/null | sed 's/^/{"lib": "ring2", "r": /; s/$/}/' >> gpurun_out/${TAG}_ab.jsonl
  timeout 900 python bench.py --steps 8 --warmup 3 --no-variants --no-cpu-baseline 2>/dev/null | sed 's/^/{"lib": "ring3", "r": /; s/$/}/' >> gpurun_out/${TAG}_ab.jsonl
done
ls -la gpurun_out | tail -2
