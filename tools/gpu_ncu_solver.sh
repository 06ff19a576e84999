mkdir -p gpurun_out
python tools/solver_one.py > gpurun_out/plain.log 2>&1 && \
ncu --section SourceCounters --section WarpStateStats --section SchedulerStats --warp-sampling-interval 0 --import-source on --clock-control none -k regex:"k_partition" -s 2 -c 2 -o gpurun_out/prof_solver_fine python tools/solver_one.py > gpurun_out/ncu_fine.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu_fine.log
