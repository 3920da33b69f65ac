#!/bin/bash
# Headline A/B: layer replicas 1 / 8, L2 prefetch of the next layer's predictor on / off, and the
# per-CTA timeline of one graph step.
for nl in 1 8; do
  for pf in "" "--no-prefetch"; do
    echo "layers $nl $pf: $(timeout -s KILL 300 python bench.py --layers $nl --steps 64 --warmup 8 --no-sweep --no-configs --no-batched --no-cpu-baseline --no-stack $pf 2>gpurun_out/exp1_$nl.err | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"], round(d["ms_per_step"]*1e3,3), d["roofline"]["frac"])')"
  done
done
tail -5 gpurun_out/exp1_8.err
CD_LIB_DIR=_lib_tl timeout -s KILL 200 python tools/timeline.py dc 0.9 2>&1 | tail -22
