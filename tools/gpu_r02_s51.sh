#!/bin/bash
# 1 GPU: fluid_spec<true> (n <= 8: chunk verification overlapped with the next
# chunk's production) -- diffusion parity, fluid slope, microbench, steps.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "diffuse" > gpurun_out/s51_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/s51_pytest.log
timeout 120 python tools/fluid_slope.py
timeout 300 python tools/solver_microbench.py 2>&1 | grep -i "diffuse_fluid"
for c in 2 3 4; do for i in 1 2; do
  timeout 300 python bench.py --config $c > gpurun_out/s51_cfg$c.json 2>/dev/null
  echo "cfg$c $(python -c "import json;d=json.load(open('gpurun_out/s51_cfg$c.json'));print(d['value'],d['clocks']['reasons'])" 2>&1 | tail -1)"
done; done
timeout 300 python tools/step_timeline.py 2>/dev/null | python -c "import json,sys;print(json.load(sys.stdin)['graph_us'])"
