#!/bin/bash
# A/B of the headline step under an env toggle, alternating (usage: gpu_ab.sh VAR).
mkdir -p gpurun_out
VAR=${1:-CD_DC_BSMEM}
env $VAR=1 timeout -s KILL 600 python -m pytest tests -x -q -m gpu --timeout 300 -k "dc or DC or smoke or graph or llama or tp" 2>&1 | tail -1
for rep in 1 2 3; do
for val in 0 1; do
  v=$(env $VAR=$val timeout -s KILL 300 python bench.py --no-sweep --no-batched --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['value'], round(d['ms_per_step']*1e3,3))")
  echo "$VAR=$val $v"
done
done | tee gpurun_out/ab.log
env $VAR=1 CD_LIB_DIR=_lib_tl timeout -s KILL 200 python tools/timeline.py dc 0.9 2>&1 | tail -3
