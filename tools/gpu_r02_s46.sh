#!/bin/bash
# 1 GPU: dynmo_solve_group -- its test, solver parity, the step timeline,
# bench configs 2..5 with --solvers group / branches interleaved.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "group or partition or repack or diffuse or config5 or publish" > gpurun_out/s46_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s46_pytest.log
timeout 300 python tools/step_timeline.py > gpurun_out/s46_timeline.json 2>gpurun_out/s46_timeline.err; echo "timeline rc=$?"; python -c "import json;print(json.load(open('gpurun_out/s46_timeline.json'))['graph_us'])"
for c in 2 3 4 5; do
  for m in branches group branches group; do
    timeout 300 python bench.py --config $c --solvers $m > gpurun_out/s46_cfg${c}_$m.json 2>gpurun_out/s46_cfg${c}_$m.err
    echo "cfg$c $m rc=$? $(python -c "import json;d=json.load(open('gpurun_out/s46_cfg${c}_$m.json'));print(d['value'],d['e2e']['value'],d['gpu_launches'],d['clocks']['reasons'])" 2>&1 | tail -1)"
  done
done
