#!/bin/bash
# 1 GPU: one CTA per SM for the step's solvers (DYNMO_SOLVER_SPREAD=1) vs
# the default: device step timeline (step_stamps), then config 2/3/4 steps
# interleaved.
mkdir -p gpurun_out
for sp in 0 1; do
  DYNMO_SOLVER_SPREAD=$sp DYNMO_LIB=$PWD/ab/libdynmo_stamps.so timeout 300 python tools/step_stamps.py > gpurun_out/s57_stamps_spread$sp.json 2>&1
  echo "spread$sp $(python -c "import json;d=json.load(open('gpurun_out/s57_stamps_spread$sp.json'));print({k:(v['start_us'],v['end_us']) if isinstance(v,dict) else v for k,v in d.items()})")"
done
for c in 2 3 4; do for sp in 0 1 0 1; do
  DYNMO_SOLVER_SPREAD=$sp timeout 300 python bench.py --config $c --steps 300 > gpurun_out/s57_cfg$c.json 2>/dev/null
  echo "cfg$c spread$sp $(python -c "import json;d=json.load(open('gpurun_out/s57_cfg$c.json'));print(d['value'],d['clocks']['reasons'])" 2>&1 | tail -1)"
done; done
