#!/bin/bash
# same-box bench comparison of several knob sets, interleaved:
#   T=tag bash tools/gpu_bench_abc.sh "" "ENV=VAL" "ENV2=VAL ENV3=VAL"
T=${T:-babc}
mkdir -p gpurun_out
for r in 1 2; do
  i=0
  for arm in "$@"; do
    env $arm timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_arm${i}_$r.json 2> gpurun_out/${T}_arm${i}_$r.err
    i=$((i+1))
  done
done
