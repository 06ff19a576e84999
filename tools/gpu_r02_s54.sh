#!/bin/bash
# 1 GPU: fluid_spec8 (DYNMO_FLUID_SPEC=2) vs fluid_spec (1) on the same box:
# k_diffuse alone on each bench instance, then the steps interleaved.
mkdir -p gpurun_out
for c in 3 4 2; do for sp in 1 2; do
  DYNMO_FLUID_SPEC=$sp timeout 300 python tools/diffuse_cfg.py $c 2>&1 | tail -1 | sed "s/^/spec$sp /"
done; done
for c in 3 4 2; do for sp in 1 2 1 2; do
  DYNMO_FLUID_SPEC=$sp timeout 300 python bench.py --config $c > gpurun_out/s54_cfg$c.json 2>/dev/null
  echo "cfg$c spec$sp $(python -c "import json;d=json.load(open('gpurun_out/s54_cfg$c.json'));print(d['value'],d['clocks']['reasons'])" 2>&1 | tail -1)"
done; done
