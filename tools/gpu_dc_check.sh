#!/bin/bash
# DC fused-path parity subset + A/B timing of the headline step against other builds.
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -x -q -m gpu --timeout 300 -k "dc or DC or smoke or graph or llama or tp or stack or gemma or fused or parity" 2>&1 | tail -3
for L in "$@"; do CD_LIB_DIR=$L timeout -s KILL 300 python tools/dc_ab.py 0.9 1 2>&1 | grep "pf=0" | sed "s/^/$L /"; done
CD_LIB_DIR=_lib_tl timeout -s KILL 300 python tools/timeline_cta.py 0.9 0 2>&1 | grep -v Warn | head -26
