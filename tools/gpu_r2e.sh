#!/bin/bash
# Round-2 pass E: runtime diagnostics (N=2 sync grads, pool growth) and the
# forward-attention variant A/B with its kernel tests.
TAG=${1:-r2e}
mkdir -p gpurun_out
timeout 600 python tests/diag_pool_and_n2.py pool > gpurun_out/${TAG}_diag_pool.txt 2>&1
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -k "attn" -p no:cacheprovider > gpurun_out/${TAG}_attn_tests.txt 2>&1
timeout 300 python tools/attn_fwd_ab.py 0 1 2 > gpurun_out/${TAG}_attn_fwd_ab.jsonl 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"attn_fwd_pp" -s 3 -c 1 \
    -o gpurun_out/${TAG}_full_attn_fwd -f python tools/bench_kernels.py attn > gpurun_out/${TAG}_ncu_fwd.log 2>&1
timeout 900 python tests/diag_pool_and_n2.py n2 > gpurun_out/${TAG}_diag_n2.txt 2>&1
ls -la gpurun_out | tail -12
