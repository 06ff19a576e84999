#!/bin/bash
# ncu --set full of one prune kernel on the config-2 bf16 weights:
#   bash tools/gpu_ncu_prune.sh k_prune_hist0w
K=${1:-k_prune_hist0w}
mkdir -p gpurun_out
python tools/prune_one.py > gpurun_out/plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"$K" -s 1 -c ${2:-1} -o gpurun_out/prof_$K python tools/prune_one.py > gpurun_out/ncu_$K.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu_$K.log
