#!/bin/bash
# Source-level ncu profiles (SourceCounters + warp states) of the partition:
# config-2 latency mode (solver_one.py) and config-5 batched mode.
mkdir -p gpurun_out
python tools/solver_one.py partition > gpurun_out/plain.log 2>&1 || exit 1
ncu --section SourceCounters --section WarpStateStats --section SchedulerStats --section LaunchStats --section Occupancy \
  --import-source on --clock-control none -k regex:"k_partition" -s 2 -c 1 -o gpurun_out/ns_part_cfg2 \
  python tools/solver_one.py partition > gpurun_out/ns_part_cfg2.log 2>&1; echo ncu1=$?
ncu --section SourceCounters --section WarpStateStats --section SchedulerStats --section LaunchStats --section Occupancy \
  --import-source on --clock-control none -k regex:"k_partition" -s 1 -c 1 -o gpurun_out/ns_part_cfg5 \
  python tools/cfg5_solvers.py > gpurun_out/ns_part_cfg5.log 2>&1; echo ncu2=$?
