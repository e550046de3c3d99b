#!/bin/bash
# same-box bench A/B: default vs the knobs given as arguments (ENV=VAL ...)
T=${T:-bab}
mkdir -p gpurun_out
for r in 1 2; do
  timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_new_$r.json 2> gpurun_out/${T}_new_$r.err
  env "$@" timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_old_$r.json 2> gpurun_out/${T}_old_$r.err
done
