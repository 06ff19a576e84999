mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q -k "prune" 2>&1 | grep -E "^E |FAILED|passed|failed" | head -12
timeout 120 python tools/bench_prune.py
timeout 120 python tools/prune_one.py && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prune_launches.csv python tools/prune_one.py > /dev/null 2>&1; echo ncu_rc=$?
python tools/ncu_kernel_means.py gpurun_out/prune_launches.csv | head -20
