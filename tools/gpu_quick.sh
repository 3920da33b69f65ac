#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -x -q -m gpu --timeout 300 2>&1 | tail -3
timeout -s KILL 600 python bench.py --no-sweep --no-batched --no-cpu-baseline > gpurun_out/quick_bench.json 2> gpurun_out/quick_bench.err
python -c "import json; d=json.load(open('gpurun_out/quick_bench.json')); print(d['value'], d['e2e'])"
