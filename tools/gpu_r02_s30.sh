#!/bin/bash
# 1 GPU: ncu of the config-5 epilogue (360 k layers), both counter layouts.
mkdir -p gpurun_out
for lib in ab/libdynmo_prevacc.so paper_2505_14864_b200/libdynmo.so; do
  tag=$(basename $lib .so)
  DYNMO_LIB=$PWD/$lib ncu --set full --import-source on --clock-control none -k regex:k_epilogue -s 3 -c 1 -o gpurun_out/s30_epi_$tag \
    python bench.py --config 5 --steps 4 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/s30_$tag.log 2>&1; echo "$tag rc=$?"
done
