#!/bin/bash
# 1 GPU: fluid round chain latencies (tools/lat/fluid_chain.cu); the
# committed build's fluid slope and config-3 step (reference for A/Bs).
mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/lat/fluid_chain.cu -o /tmp/fc && /tmp/fc | tee gpurun_out/s48_fluid_chain.txt
timeout 120 python tools/fluid_slope.py
for i in 1 2; do timeout 300 python bench.py --config 3 > gpurun_out/s48_cfg3.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/s48_cfg3.json'));print('cfg3',d['value'])"; done
