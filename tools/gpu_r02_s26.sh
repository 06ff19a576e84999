#!/bin/bash
# 1 GPU: fluid chain A/B (previous build vs current), diffusion parity.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "diffuse" > gpurun_out/s26_pytest.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/s26_pytest.log
for lib in ab/libdynmo_prev.so paper_2505_14864_b200/libdynmo.so ab/libdynmo_prev.so paper_2505_14864_b200/libdynmo.so; do
  DYNMO_LIB=$PWD/$lib timeout 300 python tools/solver_microbench.py > /dev/null 2>&1
  python -c "import json;d=json.load(open('gpurun_out/solver_microbench.json'));print('$lib', {k:v for k,v in d.items() if 'fluid' in k and ('cfg2' in k or 'L127' in k)})"
done
