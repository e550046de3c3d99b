#!/bin/bash
# same-box A/B of runtime knobs: alternating bench runs (short: steps 6)
T=${1:-ab}
mkdir -p gpurun_out
for rep in 1 2; do
  for v in "RP_LOGITS_ROWS=1024" "RP_LOGITS_ROWS=2048" "RP_LOGITS_ROWS=4096"; do
    env $v timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_${v}_$rep.json 2> gpurun_out/${T}_${v}_$rep.err
  done
done
