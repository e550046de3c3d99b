#!/bin/bash
# in-step kernel breakdown of one profiled 8B step, new HBM kernels vs the
# library before them (same box); then the LoRA and C5 reduced-depth lines
TAG=${1:-r2z4}
mkdir -p gpurun_out
timeout 900 python tools/step_profile.py --warmup 3 --out gpurun_out/${TAG}_prof.npz > gpurun_out/${TAG}_step_profile.json 2>&1
timeout 120 python tools/step_breakdown.py gpurun_out/${TAG}_prof.npz 40 > gpurun_out/${TAG}_step_breakdown.txt 2>&1
RP_LIB=ab_libs/lib_before_qk.so timeout 900 python tools/step_profile.py --warmup 3 --out gpurun_out/${TAG}_prof_before.npz > gpurun_out/${TAG}_step_profile_before.json 2>&1
timeout 120 python tools/step_breakdown.py gpurun_out/${TAG}_prof_before.npz 40 > gpurun_out/${TAG}_step_breakdown_before.txt 2>&1
timeout 900 python bench.py --steps 8 --warmup 3 --lora-rank 32 --lora-alpha 64 --no-variants \
  --no-cpu-baseline > gpurun_out/${TAG}_bench_lora.json 2> gpurun_out/${TAG}_bench_lora.err
timeout 1500 python bench.py --model qwen3-235b-a22b-l8 --seq 31744 --micro-batches 4 --lora-rank 32 \
  --lora-alpha 64 --steps 4 --warmup 2 --no-variants --no-cpu-baseline --host-publish --residency-factor 1.0 \
  > gpurun_out/${TAG}_bench_c5.json 2> gpurun_out/${TAG}_bench_c5.err
