#!/bin/bash
# A/B the headline step across library builds: gpu_ab_libs.sh _lib _lib_x ... (alternating, 2 rounds)
mkdir -p gpurun_out
for rep in 1 2; do
for L in "$@"; do
  CD_LIB_DIR=$L timeout -s KILL 300 python tools/dc_ab.py ${AB_K:-0.9} 1 2>&1 | sed "s/^/$L /" | grep -v Warn
done
done | tee gpurun_out/ab_libs.log
