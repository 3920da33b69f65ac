#!/bin/bash
# Round evidence (one GPU): ncu launch lists (duration + DRAM bytes) and full captures of the
# dominant kernels.  Outputs under gpurun_out/ev/; summarised into profiles/ by tools/evidence.py.
mkdir -p gpurun_out/ev
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
timeout -s KILL 600 ncu $M -s 40 -c 60 --log-file gpurun_out/ev/launches_dc.csv python tools/prof_step.py dc 0.9 60 bf16 > /dev/null 2>&1
timeout -s KILL 600 ncu $M -s 40 -c 60 --log-file gpurun_out/ev/launches_mc.csv python tools/prof_step.py mc 0.9 60 bf16 > /dev/null 2>&1
timeout -s KILL 600 ncu $M -s 40 -c 60 --log-file gpurun_out/ev/launches_dense.csv python tools/prof_step.py dense 0 60 bf16 > /dev/null 2>&1
timeout -s KILL 600 ncu $M --log-file gpurun_out/ev/launches_tc.csv python tools/tc_bench.py --steps 2 --no-graph --cases dc,mc,dense,prefill > /dev/null 2>&1
timeout -s KILL 600 ncu $M -s 8 -c 12 --log-file gpurun_out/ev/launches_gemma_b4.csv python tools/prof_batch.py dc 4 10 > /dev/null 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_dc_fused -s 20 -c 1 -o gpurun_out/ev/dc_fused_full python tools/prof_step.py dc 0.9 30 bf16 > /dev/null 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_tc_fused -c 1 -o gpurun_out/ev/tc_fused_full python tools/tc_bench.py --steps 1 --no-graph --cases dc > /dev/null 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_tc_pf_down -c 1 -o gpurun_out/ev/pf_down_full python tools/tc_bench.py --steps 1 --no-graph --cases prefill > /dev/null 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_tc_gateup -c 1 -o gpurun_out/ev/pf_gateup_full python tools/tc_bench.py --steps 1 --no-graph --cases prefill > /dev/null 2>&1
ls -la gpurun_out/ev
