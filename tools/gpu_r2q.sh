#!/bin/bash
# pass Q: same-box A/B of the C3 headline (12 steps each, alternating):
# HEAD (2-slot ring), 3-slot ring, + in-place publication at N=1, + explicit
# shared accesses in the attention backward (current tree); attention kernel A/B
TAG=${1:-r2q}
mkdir -p gpurun_out
: > gpurun_out/${TAG}_ab.jsonl
run() {  # $1 label, $2 lib or ""
  if [ -n "$2" ]; then export RP_LIB=$PWD/ab_libs/$2; else unset RP_LIB; fi
  timeout 900 python bench.py --steps 12 --warmup 3 --no-variants --no-cpu-baseline 2>> gpurun_out/${TAG}_$1.err \
    | sed "s/^/{\"lib\": \"$1\", \"r\": /; s/\$/}/" >> gpurun_out/${TAG}_ab.jsonl
}
: > gpurun_out/${TAG}_attn_ab.jsonl
for i in 1 2; do
  RP_LIB=$PWD/ab_libs/lib_direct.so timeout 200 python tools/bench_kernels.py attn | sed 's/^/{"lib": "direct", "r": /; s/$/}/' >> gpurun_out/${TAG}_attn_ab.jsonl
  timeout 200 python tools/bench_kernels.py attn | sed 's/^/{"lib": "cur", "r": /; s/$/}/' >> gpurun_out/${TAG}_attn_ab.jsonl
done
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -k flash -p no:cacheprovider > gpurun_out/${TAG}_attn_tests.txt 2>&1
for i in 1 2; do
  run ring2 lib_ring2.so
  run ring3 lib_ring3.so
  run direct lib_direct.so
  run cur ""
done
ls -la gpurun_out | tail -3
