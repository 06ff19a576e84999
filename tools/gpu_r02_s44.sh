#!/bin/bash
# 1 GPU: discrete diffusion with lane groups per edge + fluid phi range bound:
# diffusion parity, solver microbench, config-2/3 steps.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "diffuse or bench" > gpurun_out/s44_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s44_pytest.log
timeout 300 python tools/solver_microbench.py 2>&1 | grep -i "diffuse"
for c in 2 3; do
  timeout 300 python bench.py --config $c > gpurun_out/s44_cfg$c.json 2>/dev/null
  echo "cfg$c $(python -c "import json;d=json.load(open('gpurun_out/s44_cfg$c.json'));print(d['value'],d['clocks']['reasons'])")"
done
