#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/tc_launches.csv python tools/tc_bench.py --steps 1 --no-graph --cases mc > gpurun_out/tc_ncu.log 2>&1
echo "ncu rc=$?"
