#!/bin/bash
# Round-end evidence: GPU tests, the bench line, ncu launch lists and full captures (one GPU).
mkdir -p gpurun_out/final
timeout -s KILL 900 python -m pytest tests -x -q -m gpu --timeout 300 > gpurun_out/final/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/final/pytest_gpu.log
timeout -s KILL 900 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err
echo "bench rc=$?"
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
timeout -s KILL 600 ncu $M -s 40 -c 60 --log-file gpurun_out/final/launches_dc.csv python tools/prof_step.py dc 0.9 60 bf16 > /dev/null 2>&1
timeout -s KILL 600 ncu $M -s 40 -c 60 --log-file gpurun_out/final/launches_dense.csv python tools/prof_step.py dense 0 60 bf16 > /dev/null 2>&1
timeout -s KILL 600 ncu $M -s 40 -c 60 --log-file gpurun_out/final/launches_mc.csv python tools/prof_step.py mc 0.9 60 bf16 > /dev/null 2>&1
timeout -s KILL 600 ncu $M --log-file gpurun_out/final/launches_tc.csv python tools/tc_bench.py --steps 1 --no-graph --cases dc,mc,dense,prefill > /dev/null 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_dc_fused -s 20 -c 1 -o gpurun_out/final/dc_fused_full python tools/prof_step.py dc 0.9 30 bf16 > /dev/null 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_tc_fused -c 1 -o gpurun_out/final/tc_fused_full python tools/tc_bench.py --steps 1 --no-graph --cases dc > /dev/null 2>&1
echo done
