#!/bin/bash
# 1 GPU: speculative fluid rounds -- diffusion parity, then the solver
# microbench and config-2/3 steps with DYNMO_FLUID_SPEC=0 / 1 interleaved.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "diffuse" > gpurun_out/s37_pytest.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/s37_pytest.log
for r in 1 2; do
  for sp in 0 1; do
    DYNMO_FLUID_SPEC=$sp timeout 300 python tools/solver_microbench.py 2>&1 | sed "s/^/spec$sp /" | grep -i "diffuse_fluid"
  done
done
for c in 2 3; do
  for sp in 0 1 0 1; do
    DYNMO_FLUID_SPEC=$sp timeout 300 python bench.py --config $c > gpurun_out/s37_cfg${c}_spec$sp.json 2>/dev/null
    echo "cfg$c spec$sp $(python -c "import json,sys;d=json.load(open('gpurun_out/s37_cfg${c}_spec$sp.json'));print(d['value'],d['ms_per_step'])")"
  done
done
