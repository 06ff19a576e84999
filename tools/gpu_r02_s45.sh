#!/bin/bash
# 1 GPU: adaptive lanes per edge in the discrete re-split; diffusion parity,
# solver microbench, fluid cost per round (speculative vs per-round).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "diffuse" > gpurun_out/s45_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/s45_pytest.log
timeout 300 python tools/solver_microbench.py 2>&1 | grep -i "diffuse"
for sp in 1 0; do DYNMO_FLUID_SPEC=$sp timeout 120 python tools/fluid_slope.py | sed "s/^/spec$sp /"; done
