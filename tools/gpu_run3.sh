timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python tools/timeline.py dc 0.9 > gpurun_out/timeline_fused.log 2>&1
cat gpurun_out/timeline_fused.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench3.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench3.log | cut -c1-600
