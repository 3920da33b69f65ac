#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:k_tc_gateup -c 1 -o gpurun_out/tc_gateup_mc \
   python tools/tc_bench.py --steps 1 --no-graph --cases mc > gpurun_out/tc_ncu_mc.log 2>&1
echo "ncu rc=$?"
