#!/bin/bash
# ncu source-level profile (stall sampling per SASS line) of one solver kernel:
#   bash tools/gpu_ncu_solver.sh partition|diffuse|repack
K=${1:-partition}
mkdir -p gpurun_out
python tools/solver_one.py $K > gpurun_out/plain.log 2>&1 && \
ncu --section SourceCounters --section WarpStateStats --section SchedulerStats --warp-sampling-interval 0 --import-source on --clock-control none -k regex:"k_$K" -s 1 -c 1 -o gpurun_out/prof_$K python tools/solver_one.py $K > gpurun_out/ncu_$K.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu_$K.log
