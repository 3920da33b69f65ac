#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 400 python -m pytest tests/test_gpu_tc.py -x -q -m gpu 2>&1 | tail -3
for g in 0; do echo "== grid $g"; CD_TC_GRID=$g timeout -s KILL 200 python tools/tc_timeline.py; done 2>&1 | tee gpurun_out/tc_tl.log
for g in 0; do echo "== grid $g"; CD_TC_GRID=$g timeout -s KILL 300 python tools/tc_bench.py --steps 20 2>&1 | grep case; done | tee gpurun_out/tc_bench.log
