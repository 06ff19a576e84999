mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "moe or profile or smoke" 2>&1 | tail -2
python tools/prof_one_moe.py > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_profile --csv --log-file gpurun_out/moe_l.csv python tools/prof_one_moe.py > /dev/null 2>&1; echo ncu=$?
python tools/summarize.py gpurun_out/moe_l.csv
