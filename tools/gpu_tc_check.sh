#!/bin/bash
# Tensor-core path parity + the batched/prefill bench section.
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_tc_fuzz.py -x -q -m gpu --timeout 300 2>&1 | tail -3
timeout -s KILL 600 python tools/tc_bench.py 2>&1 | tail -8
