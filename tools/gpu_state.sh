#!/bin/bash
# Full GPU test suite + default bench line + steps-20 bench (driver's count) on one B200.
mkdir -p gpurun_out/state
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/state/smi.txt
timeout -s KILL 1200 python -m pytest tests -q -m gpu --timeout 300 -x > gpurun_out/state/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/state/pytest_gpu.log
timeout -s KILL 900 python bench.py > gpurun_out/state/bench.json 2> gpurun_out/state/bench.err
echo "bench rc=$?"; tail -3 gpurun_out/state/bench.err
timeout -s KILL 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/state/bench_ref.json 2> gpurun_out/state/bench_ref.err
echo "ref rc=$?"; tail -3 gpurun_out/state/bench_ref.err
