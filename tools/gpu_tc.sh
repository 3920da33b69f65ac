#!/bin/bash
mkdir -p gpurun_out
for pf in 0 8 16 32; do echo "== pf $pf"; CD_TC_PB_PF=$pf timeout -s KILL 300 python tools/tc_bench.py --steps 20 --cases dc,mc 2>&1 | grep "case\|Error\|error"; done | tee gpurun_out/tc_bench.log
CD_TC_PB_PF=16 timeout -s KILL 200 python tools/tc_timeline.py 2>&1 | head -10
