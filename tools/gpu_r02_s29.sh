#!/bin/bash
# 1 GPU: per-kernel launch list of the config-5 step for both counter layouts.
mkdir -p gpurun_out
for lib in ab/libdynmo_prevacc.so paper_2505_14864_b200/libdynmo.so; do
  tag=$(basename $lib .so)
  DYNMO_LIB=$PWD/$lib ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s29_$tag.csv \
    python bench.py --config 5 --steps 8 --warmup 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1; echo "$tag rc=$?"
  python tools/ncu_kernel_means.py gpurun_out/s29_$tag.csv | grep dynmo
done
