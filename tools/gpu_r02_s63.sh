#!/bin/bash
# 1 GPU: device step timeline (L2 flushed) with the fluid modes 1 and 2, and
# the ncu launch list's k_diffuse (cold) for each.
mkdir -p gpurun_out
for sp in 1 2 1 2; do
  DYNMO_FLUID_SPEC=$sp DYNMO_LIB=$PWD/ab/libdynmo_stamps.so timeout 300 python tools/step_stamps.py > gpurun_out/s63_stamps_spec$sp.json 2>&1
  echo "spec$sp $(python -c "import json;d=json.load(open('gpurun_out/s63_stamps_spec$sp.json'));print({k:(v['start_us'],v['end_us']) for k,v in d.items() if isinstance(v,dict) and k.startswith('diff')}, d['graph_replay_events_us'])" 2>&1 | tail -1)"
done
CMD="python bench.py --steps 20 --warmup 5 --e2e-steps 1 --no-cpu-baseline"
for sp in 1 2; do
  DYNMO_FLUID_SPEC=$sp $CMD > /dev/null 2>&1 && DYNMO_FLUID_SPEC=$sp ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_diffuse --log-file gpurun_out/s63_launch_spec$sp.csv $CMD > /dev/null 2>&1
  echo "ncu spec$sp $(python tools/ncu_kernel_means.py gpurun_out/s63_launch_spec$sp.csv | grep k_diffuse)"
done
