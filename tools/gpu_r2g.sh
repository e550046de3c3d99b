#!/bin/bash
# Round-2 pass G: whole GPU suite + smoke after the workspace fix, ncu full
# captures of the attention backward and the QK-norm/RoPE kernels, the
# default bench line.
TAG=${1:-r2g}
mkdir -p gpurun_out
for k in attn_bwd_fused qk_norm_rope_fwd qk_norm_rope_bwd; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 3 -c 1 \
    -o gpurun_out/${TAG}_full_$k -f python tools/bench_kernels.py > gpurun_out/${TAG}_ncu_$k.log 2>&1
done
timeout 300 python tools/bench_kernels.py > gpurun_out/${TAG}_kernels.jsonl 2>&1
bash tools/gpu_r2d.sh ${TAG}
