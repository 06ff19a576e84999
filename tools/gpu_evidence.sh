mkdir -p gpurun_out
python tools/bench_configs.py > gpurun_out/bench_configs.log 2>&1; echo configs_rc=$?
tail -6 gpurun_out/bench_configs.log
python bench.py --steps 200 --warmup 20 > gpurun_out/ev_n1.json 2> gpurun_out/ev_n1.err; echo bench_rc=$?
CMD="python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01_final.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_profile -s 3 -c 2 -o gpurun_out/prof_k_profile_r01_final $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu=$?
