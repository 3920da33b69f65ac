set -x
mkdir -p gpurun_out/prof
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 40 -c 60 --csv --log-file gpurun_out/prof/launches_dc.csv python tools/prof_step.py dc 0.9 60 bf16 > gpurun_out/prof/launches_dc.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 40 -c 60 --csv --log-file gpurun_out/prof/launches_dense.csv python tools/prof_step.py dense 0 60 bf16 > gpurun_out/prof/launches_dense.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 40 -c 60 --csv --log-file gpurun_out/prof/launches_mc.csv python tools/prof_step.py mc 0.9 60 bf16 > gpurun_out/prof/launches_mc.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dc_fused -s 20 -c 2 -o gpurun_out/prof/dc_fused_full python tools/prof_step.py dc 0.9 30 bf16 > gpurun_out/prof/full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sparse -s 20 -c 2 -o gpurun_out/prof/dense_full python tools/prof_step.py dense 0 30 bf16 > gpurun_out/prof/full_dense.log 2>&1
timeout 600 python bench.py > gpurun_out/prof/bench.json 2> gpurun_out/prof/bench.err
