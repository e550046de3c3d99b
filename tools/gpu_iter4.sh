#!/bin/bash
T=${1:-it}
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_runtime_gpu.py -q > gpurun_out/${T}_pytest_r.txt 2>&1; echo "exit $?" >> gpurun_out/${T}_pytest_r.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.txt 2>&1; echo "exit $?" >> gpurun_out/${T}_smoke.txt
timeout 900 python bench.py --report-dir gpurun_out > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 600 python tools/step_profile.py > gpurun_out/${T}_step_profile.json 2>&1
