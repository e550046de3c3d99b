#!/bin/bash
# Full ncu captures of the attention kernels and the wgrad GEMM, plus the
# launch list of the bench command on qwen3-1.7b (the 8B run's 115 GB of
# pinned optimizer state OOMs the 196 GB host under ncu). One GPU.
TAG=${1:-r}
mkdir -p gpurun_out
for k in attn_fwd_pp attn_bwd_dkv_pp attn_bwd_dq_pp; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 2 -c 1 \
    -o gpurun_out/${TAG}_full_$k -f python tools/bench_kernels.py attn > gpurun_out/${TAG}_ncu_$k.log 2>&1
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"gemm" -s 6 -c 1 \
  -o gpurun_out/${TAG}_full_gemm_gu_wgrad -f python tools/bench_gemm.py gu_wgrad > gpurun_out/${TAG}_ncu_wg.log 2>&1
if [ "$2" == "launches" ]; then
  SKIP=${SKIP:-20000} COUNT=${COUNT:-4000} REPLAY=application bash tools/ncu_launchlist.sh ${TAG}_17b qwen3-1.7b
fi
ls -la gpurun_out | tail -12
