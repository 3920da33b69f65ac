#!/bin/bash
# A/B of the headline step: current build (_lib) vs the previous commit (_lib_old), alternating.
mkdir -p gpurun_out
for rep in 1 2; do
for lib in _lib_old _lib; do
  v=$(CD_LIB_DIR=$lib timeout -s KILL 300 python bench.py --no-sweep --no-batched --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['value'], round(d['ms_per_step']*1e3,3), d['e2e']['value'] if d['e2e'] else None)")
  echo "$lib $v"
done
done | tee gpurun_out/ab.log
