set -x
timeout 120 ./tools/bw_micro > gpurun_out/bw_micro.log 2>&1
timeout 300 python tools/timeline.py dc 0.9 > gpurun_out/timeline_dc.log 2>&1
timeout 300 python tools/timeline.py dense 0 > gpurun_out/timeline_dense.log 2>&1
timeout 300 python tools/timeline.py mc 0.9 > gpurun_out/timeline_mc.log 2>&1
