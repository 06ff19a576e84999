#!/bin/bash
# 1 GPU: source-level ncu (warp-state sampling) of the config-4 MoE profile kernel.
mkdir -p gpurun_out
ncu --set full --import-source on --warp-sampling-interval 0 --clock-control none -k regex:k_profile -s 5 -c 1 -o gpurun_out/s37_moe \
  python bench.py --config 4 --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/s37.log 2>&1; echo "ncu rc=$?"
