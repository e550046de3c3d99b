#!/bin/bash
# ncu launch list of the bench command (one metric, one pass) with host-memory monitoring.
TAG=${1:-r}
MODEL=${2:-qwen3-8b}
mkdir -p gpurun_out
free -g > gpurun_out/${TAG}_mem.txt
( while true; do date +%T >> gpurun_out/${TAG}_mem.txt; free -g | sed -n 2p >> gpurun_out/${TAG}_mem.txt; sleep 5; done ) &
MON=$!
timeout 1500 ncu --replay-mode ${REPLAY:-application} --metrics gpu__time_duration.sum --clock-control none \
  -s ${SKIP:-47000} -c ${COUNT:-3000} --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --model $MODEL --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu_bench.log 2>&1
echo "ncu exit $?" >> gpurun_out/${TAG}_ncu_bench.log
kill $MON
dmesg 2>/dev/null | tail -20 > gpurun_out/${TAG}_dmesg.txt
