#!/bin/bash
# 1 GPU: does the step follow the diffusion kernel?  Config 2/3 steps and the
# config-2 step timeline with the fluid per-round (0, ~22 us), speculative (1)
# and overlapped (2), interleaved on one box.
mkdir -p gpurun_out
for c in 3 2; do for sp in 0 1 2 0 1 2; do
  DYNMO_FLUID_SPEC=$sp timeout 300 python bench.py --config $c --steps 300 > gpurun_out/s55_cfg$c.json 2>/dev/null
  echo "cfg$c spec$sp $(python -c "import json;d=json.load(open('gpurun_out/s55_cfg$c.json'));print(d['value'],d['clocks']['reasons'])" 2>&1 | tail -1)"
done; done
for sp in 0 2; do
  DYNMO_FLUID_SPEC=$sp timeout 300 python tools/step_timeline.py 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('spec$sp',d['graph_us'])"
done
