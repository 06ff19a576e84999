#!/bin/bash
# 1 GPU: two-warp fluid pipeline -- diffusion parity in every fluid mode,
# fluid slope, solver microbench, config-2/3/4 steps (modes 1 vs 2).
mkdir -p gpurun_out
for sp in 2 1 0; do
  DYNMO_FLUID_SPEC=$sp timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "diffuse" > gpurun_out/s47_pytest_spec$sp.log 2>&1; echo "pytest spec$sp rc=$?"; tail -2 gpurun_out/s47_pytest_spec$sp.log
done
for sp in 2 1; do DYNMO_FLUID_SPEC=$sp timeout 120 python tools/fluid_slope.py | sed "s/^/spec$sp /"; done
timeout 300 python tools/solver_microbench.py 2>&1 | grep -i "diffuse"
for c in 2 3 4; do
  for sp in 1 2 1 2; do
    DYNMO_FLUID_SPEC=$sp timeout 300 python bench.py --config $c > gpurun_out/s47_cfg${c}_spec$sp.json 2>/dev/null
    echo "cfg$c spec$sp $(python -c "import json;d=json.load(open('gpurun_out/s47_cfg${c}_spec$sp.json'));print(d['value'],d['clocks']['reasons'])" 2>&1 | tail -1)"
  done
done
