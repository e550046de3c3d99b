#!/bin/bash
# Round-2 GPU pass B: runtime / protocol suites, transfer probe, the default
# bench line (C3) and the reference arm. Outputs in gpurun_out/.
TAG=${1:-r2b}
mkdir -p gpurun_out
: > gpurun_out/${TAG}_pytest.txt
for f in tests/test_protocol_gpu.py tests/test_runtime_gpu.py ${EXTRA_TESTS}; do
  timeout 1800 python -m pytest $f -m gpu -q -s -rA -p no:cacheprovider >> gpurun_out/${TAG}_pytest.txt 2>&1
  echo "pytest $f exit $?" >> gpurun_out/${TAG}_pytest.txt
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
echo "smoke exit $?" >> gpurun_out/${TAG}_smoke.txt
timeout 300 python tools/transfer_probe.py > gpurun_out/${TAG}_transfer_probe.json 2>&1
if [ "$2" != "skip-bench" ]; then
  timeout 1200 python bench.py --steps ${STEPS:-20} --warmup 5 --report-dir gpurun_out/${TAG}_report > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
  echo "bench exit $?" >> gpurun_out/${TAG}_bench.err
fi
if [ "$3" == "ref" ]; then
  timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
  echo "ref exit $?" >> gpurun_out/${TAG}_bench_ref.err
fi
ls -la gpurun_out | tail -12
