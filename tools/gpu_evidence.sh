mkdir -p gpurun_out
T=r01s31
timeout 600 python tools/step_profile.py > gpurun_out/${T}_step_profile.json 2>&1
for k in attn_fwd_pp attn_bwd_dkv_pp attn_bwd_dq3; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 2 -c 1 \
    -o gpurun_out/${T}_full_$k -f python tools/bench_kernels.py attn > gpurun_out/${T}_ncu_$k.log 2>&1
done
for g in gu_fwd gu_wgrad down_fwd o_fwd; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"gemm" -s 6 -c 1 \
    -o gpurun_out/${T}_full_gemm_$g -f python tools/bench_gemm.py $g > gpurun_out/${T}_ncu_$g.log 2>&1
done
timeout 300 ncu --set full --clock-control none -k regex:"rmsnorm_bwd|swiglu_bwd|adamw" -c 3 \
  -o gpurun_out/${T}_full_hbm -f python tools/bench_kernels.py > gpurun_out/${T}_ncu_hbm.log 2>&1
