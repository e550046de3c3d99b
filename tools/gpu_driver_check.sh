#!/bin/bash
# What the driver runs at round end, in its order: the whole GPU suite in ONE
# pytest process, smoke(), then the default bench line.
TAG=${1:-r2re}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 3000 python -m pytest tests/ -x -q -m gpu -rA -p no:cacheprovider > gpurun_out/${TAG}_pytest_onepass.txt 2>&1
echo "pytest exit $?" >> gpurun_out/${TAG}_pytest_onepass.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
echo "smoke exit $?" >> gpurun_out/${TAG}_smoke.txt
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench exit $?" >> gpurun_out/${TAG}_bench.err
timeout 1200 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
echo "ref exit $?" >> gpurun_out/${TAG}_bench_ref.err
