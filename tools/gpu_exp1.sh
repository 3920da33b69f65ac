#!/bin/bash
# L2-resident vs HBM-streamed headline (layer replicas 1 / 2 / 8) and the per-CTA timeline.
for nl in 1 2 4 8; do
  echo "layers $nl: $(timeout -s KILL 300 python bench.py --layers $nl --steps 64 --warmup 8 --no-sweep --no-configs --no-batched --no-cpu-baseline --no-stack 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"], round(d["ms_per_step"]*1e3,3))')"
done
CD_LIB_DIR=_lib_tl timeout -s KILL 200 python tools/timeline.py dc 0.9 2>&1 | tail -22
