#!/bin/bash
# A/B of the batched (B=64) tensor-core step: previous build (_lib_old) vs current.
timeout -s KILL 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_tc_fuzz.py tests/test_gpu_tp.py -x -q -m gpu --timeout 300 2>&1 | tail -1
for rep in 1 2; do
for lib in _lib_old _lib; do
  echo "$lib"; CD_LIB_DIR=$lib timeout -s KILL 300 python tools/tc_bench.py --steps 20 --cases dc,mc 2>/dev/null | grep case
done
done
