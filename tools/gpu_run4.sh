timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -4 gpurun_out/pytest_gpu.log
for i in 1 2 3; do timeout 300 python bench.py --no-cpu-baseline --no-sweep 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['ms_per_step']*1e3, j['roofline']['stages'], j['e2e']['value'])"; done
