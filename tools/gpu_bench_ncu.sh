mkdir -p gpurun_out
set -x
python bench.py --steps 50 --warmup 10 > gpurun_out/bench_r01a.json 2> gpurun_out/bench_r01a.err; echo bench_rc=$?
tail -3 gpurun_out/bench_r01a.err
CMD="python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_profile -s 3 -c 2 -o gpurun_out/prof_k_profile_r01 $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
