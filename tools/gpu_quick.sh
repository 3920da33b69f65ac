#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests -x -q -m gpu --timeout 300 -k "mc or MC or properties or qwen or tp or smoke" 2>&1 | tail -2
timeout -s KILL 200 python tools/mc_timeline.py 2>&1 | tail -7
