#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 300 python tools/e2e_probe.py 2>&1 | head -2
CD_COPY_KERNEL=0 timeout -s KILL 300 python tools/e2e_probe.py 2>&1 | head -1
CD_HOST_GRAPH=0 timeout -s KILL 300 python tools/e2e_probe.py 2>&1 | head -1
timeout -s KILL 900 python -m pytest tests -x -q -m gpu --timeout 300 2>&1 | tail -2
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()"
