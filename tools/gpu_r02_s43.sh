#!/bin/bash
# 1 GPU: source-level stall sampling of the three solver kernels on the
# bench's config-2 instance (synthetic CSR payload memory, its cap).
mkdir -p gpurun_out
S="--section SourceCounters --section WarpStateStats --section SchedulerStats --section LaunchStats --section Occupancy --section SpeedOfLight"
for w in diffuse partition repack; do
  python tools/solver_one.py ${w}_bench > gpurun_out/s43_$w.log 2>&1 || { echo "plain $w failed"; cat gpurun_out/s43_$w.log; exit 1; }
  ncu $S --import-source on --clock-control none --warp-sampling-interval 0 -k regex:"k_$w" -s 1 -c 1 \
    -o gpurun_out/s43_ns_$w python tools/solver_one.py ${w}_bench > gpurun_out/s43_ncu_$w.log 2>&1; echo "ncu $w rc=$?"
done
