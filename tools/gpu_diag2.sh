timeout 300 python tools/timeline.py dc 0.9 > gpurun_out/timeline_fused.log 2>&1
CD_DC_CHAIN=1 timeout 300 python tools/timeline.py dc 0.9 > gpurun_out/timeline_chain.log 2>&1
