#!/bin/bash
# Round-2 final evidence pass: whole GPU suite (margins printed), smoke, the
# default bench line, LoRA / C5 / reference-arm lines, kernel micro-benches,
# ncu full captures of the top kernels and the launch list of the 1.7B bench.
TAG=${1:-r2final}
mkdir -p gpurun_out
: > gpurun_out/${TAG}_pytest.txt
for f in tests/test_*gpu*.py; do
  timeout 1800 python -m pytest $f -m gpu -q -s -rA -p no:cacheprovider >> gpurun_out/${TAG}_pytest.txt 2>&1
  echo "pytest $f exit $?" >> gpurun_out/${TAG}_pytest.txt
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
echo "smoke exit $?" >> gpurun_out/${TAG}_smoke.txt
timeout 1200 python bench.py --steps 20 --warmup 5 --report-dir gpurun_out/${TAG}_report \
  > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench exit $?" >> gpurun_out/${TAG}_bench.err
timeout 900 python bench.py --steps 8 --warmup 3 --lora-rank 32 --lora-alpha 64 --no-variants \
  --no-cpu-baseline > gpurun_out/${TAG}_bench_lora.json 2> gpurun_out/${TAG}_bench_lora.err
timeout 1500 python bench.py --model qwen3-235b-a22b-l8 --seq 31744 --micro-batches 4 --lora-rank 32 \
  --lora-alpha 64 --steps 4 --warmup 2 --no-variants --no-cpu-baseline --host-publish --residency-factor 1.0 \
  --report-dir gpurun_out/${TAG}_report_c5 > gpurun_out/${TAG}_bench_c5.json 2> gpurun_out/${TAG}_bench_c5.err
timeout 1200 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
timeout 300 python tools/bench_kernels.py > gpurun_out/${TAG}_kernels.jsonl 2>&1
timeout 300 python tools/bench_gemm.py > gpurun_out/${TAG}_gemm.jsonl 2>&1
for k in attn_fwd_pp attn_bwd_fused qk_norm_rope_bwd rmsnorm_bwd; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 3 -c 1 \
    -o gpurun_out/${TAG}_full_$k -f python tools/bench_kernels.py > gpurun_out/${TAG}_ncu_$k.log 2>&1
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_pair -s 6 -c 1 \
  -o gpurun_out/${TAG}_full_gemm_gu_fwd -f python tools/bench_gemm.py gu_fwd > gpurun_out/${TAG}_ncu_gemm.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 30000 -c 3000 --csv \
  --log-file gpurun_out/${TAG}_launches_17b.csv python bench.py --model qwen3-1.7b --steps 1 --warmup 3 \
  --no-variants --no-cpu-baseline > gpurun_out/${TAG}_ncu_launches.log 2>&1
ls -la gpurun_out | tail -20
