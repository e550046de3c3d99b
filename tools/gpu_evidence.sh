#!/bin/bash
# ncu --set full captures of the step's top kernels + one profiled 8B step.
#   bash tools/gpu_evidence.sh <tag>
mkdir -p gpurun_out
T=${1:-ev}
timeout 600 python tools/step_profile.py --out gpurun_out/${T}_prof.npz > gpurun_out/${T}_step_profile.json 2>&1
for k in attn_fwd_pp attn_bwd_fused; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 2 -c 1 \
    -o gpurun_out/${T}_full_$k -f python tools/bench_kernels.py attn > gpurun_out/${T}_ncu_$k.log 2>&1
done
for g in gu_fwd gu_wgrad down_fwd o_fwd; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"gemm" -s 6 -c 1 \
    -o gpurun_out/${T}_full_gemm_$g -f python tools/bench_gemm.py $g > gpurun_out/${T}_ncu_$g.log 2>&1
done
# the two SwiGLU-fused GEMMs as the step runs them (dual gate/up fwd, down dgrad)
timeout 300 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"gemm_pair_kernel<\\(int\\)0, \\(int\\)0, \\(int\\)4" -s 3 -c 1 \
  -o gpurun_out/${T}_full_gemm_gu_fwd_swiglu -f python tools/bench_gemm.py swiglu > gpurun_out/${T}_ncu_sw1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"gemm_pair_kernel<\\(int\\)0, \\(int\\)1, \\(int\\)3" -s 3 -c 1 \
  -o gpurun_out/${T}_full_gemm_down_dgrad_swiglu -f python tools/bench_gemm.py swiglu > gpurun_out/${T}_ncu_sw2.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:"rmsnorm_bwd|qk_norm_rope|adamw" -c 4 \
  -o gpurun_out/${T}_full_hbm -f python tools/bench_kernels.py > gpurun_out/${T}_ncu_hbm.log 2>&1
