#!/bin/bash
# 1 GPU: per-config timings (config 1 batched partition/repack, configs 3-5,
# by-Time, stage map) with the final build.
mkdir -p gpurun_out
timeout 900 python tools/bench_configs.py > gpurun_out/s35_bench_configs.log 2>&1; echo "rc=$?"
cp gpurun_out/bench_configs.json gpurun_out/s35_bench_configs.json 2>/dev/null
tail -30 gpurun_out/s35_bench_configs.log
