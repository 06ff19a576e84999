#!/bin/bash
# 1 GPU: slot-major counters: profile parity, bench configs 5 and 2, ncu
# DRAM traffic of k_profile for config 5.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "profile or config5 or exchange or prune_reproduces or sparse or time" > gpurun_out/s27_pytest.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/s27_pytest.log
for c in 5 2; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/s27_bench_cfg$c.json 2>/dev/null; echo "bench $c rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/s27_bench_cfg$c.json').read().strip().splitlines()[-1]);r=d['roofline'];print(d['value'],r['avg_launch_ms'],r['kernel_span_ms'],r['frac'],r['frac_span'])"
done
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_profile -s 5 -c 1 --csv \
  python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s27_ncu_cfg5.csv 2>&1; echo ncu=$?
grep -E "dram__|gpu__time" gpurun_out/s27_ncu_cfg5.csv | tail -3
