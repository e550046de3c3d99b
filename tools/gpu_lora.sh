mkdir -p gpurun_out
T=r01s28
timeout 600 python -m pytest tests/test_runtime_gpu.py -q > gpurun_out/${T}_pytest_r.txt 2>&1; echo "exit $?" >> gpurun_out/${T}_pytest_r.txt
timeout 900 python bench.py --lora-rank 32 --lora-alpha 64 --no-cpu-baseline > gpurun_out/${T}_bench_lora.json 2> gpurun_out/${T}_bench_lora.err
