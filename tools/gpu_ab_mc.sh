#!/bin/bash
# A/B of the M-CountDown step (90%, batch 1, graph of 20): previous build (_lib_old) vs current.
timeout -s KILL 600 python -m pytest tests -x -q -m gpu --timeout 300 -k "mc or MC or properties or qwen or tp or smoke" 2>&1 | tail -1
for rep in 1 2 3; do
for lib in _lib_old _lib; do
  echo "$lib $(CD_LIB_DIR=$lib timeout -s KILL 200 python tools/mc_timeline.py 2>/dev/null | head -1)"
done
done
