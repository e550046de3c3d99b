#!/bin/bash
# attention iteration: kernel tests (fwd/bwd vs torch fp32), CUDA-event bench,
# optional full ncu capture of the fused backward / forward
TAG=${1:-attn}
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q -k "flash_attention" > gpurun_out/${TAG}_test.txt 2>&1
echo "test exit $?" >> gpurun_out/${TAG}_test.txt
timeout 200 python tools/bench_kernels.py attn > gpurun_out/${TAG}_bench.jsonl 2>&1
if [ -n "$2" ]; then
  for k in $2; do
    timeout 300 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 3 -c 1 \
      -o gpurun_out/${TAG}_full_$k -f python tools/bench_kernels.py attn > gpurun_out/${TAG}_ncu_$k.log 2>&1
  done
fi
tail -3 gpurun_out/${TAG}_test.txt; cat gpurun_out/${TAG}_bench.jsonl
