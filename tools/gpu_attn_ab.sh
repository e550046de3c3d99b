mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -k "attention" > gpurun_out/r01s19_pytest_k.txt 2>&1; echo "exit $?" >> gpurun_out/r01s19_pytest_k.txt
for r in 1 2; do
timeout 200 python tools/bench_kernels.py attn > gpurun_out/r01s19_attn_pt_$r.jsonl 2>&1
RP_ATTN_FWD_PSMEM=1 timeout 200 python tools/bench_kernels.py attn > gpurun_out/r01s19_attn_ps_$r.jsonl 2>&1
done
