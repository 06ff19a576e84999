#!/bin/bash
# 1 GPU: fluid_spec<OVL> refactor -- diffusion parity in all three fluid
# modes, k_diffuse alone on the bench instances (modes 1 and 2).
mkdir -p gpurun_out
for sp in 2 1 0; do
  DYNMO_FLUID_SPEC=$sp timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "diffuse" > gpurun_out/s62_pytest_spec$sp.log 2>&1; echo "pytest spec$sp rc=$?"; tail -1 gpurun_out/s62_pytest_spec$sp.log
done
for c in 2 3 4; do for sp in 1 2; do
  DYNMO_FLUID_SPEC=$sp timeout 300 python tools/diffuse_cfg.py $c 2>&1 | tail -1 | sed "s/^/spec$sp /"
done; done
