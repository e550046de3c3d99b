#!/bin/bash
# quick iteration: kernel tests, attention A/B, ncu of the attention kernels, optional bench
T=${1:-it}
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x > gpurun_out/${T}_pytest_k.txt 2>&1; echo "exit $?" >> gpurun_out/${T}_pytest_k.txt
timeout 200 python tools/bench_kernels.py attn > gpurun_out/${T}_attn.jsonl 2>&1
RP_ATTN_FWD_POLY=1 timeout 200 python tools/bench_kernels.py attn > gpurun_out/${T}_attn_poly.jsonl 2>&1
for k in attn_fwd_pp attn_bwd_dkv_pp attn_bwd_dq_pp; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 2 -c 1 \
    -o gpurun_out/${T}_full_$k -f python tools/bench_kernels.py attn > gpurun_out/${T}_ncu_$k.log 2>&1
done
if [ "$2" == "bench" ]; then
  timeout 300 python -m pytest tests/test_runtime_gpu.py -q -x > gpurun_out/${T}_pytest_r.txt 2>&1; echo "exit $?" >> gpurun_out/${T}_pytest_r.txt
  timeout 900 python bench.py --report-dir gpurun_out > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
fi
