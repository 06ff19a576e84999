#!/bin/bash
# 1 GPU: source-level ncu of the batched (config 5) partition and repack.
mkdir -p gpurun_out
python tools/cfg5_solvers.py > gpurun_out/s9_plain.txt 2>&1 || exit 1
cat gpurun_out/s9_plain.txt
for k in partition repack; do
ncu --set full --import-source on --warp-sampling-interval 1 --clock-control none -k regex:"k_$k" -s 1 -c 1 \
  -o gpurun_out/s9_ncu_cfg5_$k python tools/cfg5_solvers.py > gpurun_out/s9_ncu_$k.log 2>&1; echo ncu_$k=$?
done
