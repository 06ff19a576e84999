#!/bin/bash
# 1 GPU: span test + GPU tier, bench configs 2..5 with the two timed passes.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/s6_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/s6_pytest_gpu.log
for c in 2 3 4 5; do
  timeout 600 python bench.py --config $c > gpurun_out/s6_bench_cfg${c}_n1.json 2> gpurun_out/s6_bench_cfg${c}_n1.err; echo "bench cfg$c rc=$?"
  tail -2 gpurun_out/s6_bench_cfg${c}_n1.err
done
