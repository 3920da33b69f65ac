#!/bin/bash
# Round-end evidence: full GPU tests, the bench line, the reference arm, ncu launch lists and
# full captures of the dominant kernels (one GPU).
mkdir -p gpurun_out/state
timeout -s KILL 1200 python -m pytest tests -q -m gpu --timeout 300 > gpurun_out/state/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/state/pytest_gpu.log
timeout -s KILL 900 python bench.py > gpurun_out/state/bench.json 2> gpurun_out/state/bench.err
echo "bench rc=$?"
timeout -s KILL 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/state/bench_ref.json 2> gpurun_out/state/bench_ref.err
echo "ref rc=$?"
bash tools/gpu_evidence.sh > /dev/null 2>&1
echo "evidence done"
