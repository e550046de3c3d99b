#!/bin/bash
# Round-2 pass C: kernel micro-bench (attention + HBM kernels) and full ncu
# captures of the attention fwd / fused bwd and the QK-norm/RoPE kernels.
TAG=${1:-r2c}
mkdir -p gpurun_out
timeout 300 python tools/bench_kernels.py > gpurun_out/${TAG}_kernels.jsonl 2>&1
for k in attn_fwd_pp attn_bwd_fused qk_norm_rope_fwd qk_norm_rope_bwd; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 3 -c 1 \
    -o gpurun_out/${TAG}_full_$k -f python tools/bench_kernels.py > gpurun_out/${TAG}_ncu_$k.log 2>&1
done
ls -la gpurun_out | tail -12
