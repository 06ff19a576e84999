mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "profile or config5 or smoke" 2>&1 | tail -3
python tools/profile_microbench.py > gpurun_out/profmicro.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:k_profile --csv --log-file gpurun_out/launches_profmicro.csv python tools/profile_microbench.py > gpurun_out/ncu_pm.log 2>&1; echo ncu=$?
