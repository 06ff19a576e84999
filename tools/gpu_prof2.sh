mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
python tools/bench_configs.py > gpurun_out/bench_configs.log 2>&1; echo configs_rc=$?
grep -E "config" gpurun_out/bench_configs.log | cut -c1-300
python tools/profile_microbench.py > gpurun_out/profmicro.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:k_profile --csv --log-file gpurun_out/pm_new.csv python tools/profile_microbench.py > /dev/null 2>&1; echo ncu=$?
python tools/ncu_groups.py gpurun_out/pm_new.csv
