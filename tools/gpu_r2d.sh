#!/bin/bash
# Round-2 pass D: the whole GPU suite (one pytest process per file, margins
# printed with -s), smoke, the default bench line and the MoE bench.
TAG=${1:-r2d}
mkdir -p gpurun_out
: > gpurun_out/${TAG}_pytest.txt
for f in tests/test_*gpu*.py; do
  timeout 1800 python -m pytest $f -m gpu -q -s -rA -p no:cacheprovider >> gpurun_out/${TAG}_pytest.txt 2>&1
  echo "pytest $f exit $?" >> gpurun_out/${TAG}_pytest.txt
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
echo "smoke exit $?" >> gpurun_out/${TAG}_smoke.txt
if [ "$2" != "skip-bench" ]; then
  timeout 1200 python bench.py --steps ${STEPS:-20} --warmup 5 --report-dir gpurun_out/${TAG}_report > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
  echo "bench exit $?" >> gpurun_out/${TAG}_bench.err
fi
ls -la gpurun_out | tail -12
