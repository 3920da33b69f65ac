#!/bin/bash
# A/B of the headline step: current build (_lib) vs the previous commit (_lib_old), alternating.
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests -x -q -m gpu --timeout 300 -k "dc or DC or smoke or graph or llama or batched" 2>&1 | tail -2
for rep in 1 2 3; do
for lib in _lib_old _lib; do
  v=$(CD_LIB_DIR=$lib timeout -s KILL 300 python bench.py --no-sweep --no-batched --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['value'], round(d['ms_per_step']*1e3,3))")
  echo "$lib $v"
done
done | tee gpurun_out/ab.log
CD_LIB_DIR=_lib_tl timeout -s KILL 200 python tools/timeline.py dc 0.9 2>&1 | tail -3
