#!/bin/bash
# 1 GPU: dynmo_publish (result read by a kernel store into mapped pinned
# memory) -- its test, the step timeline, bench configs 2..5 with
# --result-read publish / copy interleaved.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "publish or bench" > gpurun_out/s40_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s40_pytest.log
timeout 300 python tools/step_timeline.py > gpurun_out/s40_timeline.json 2>gpurun_out/s40_timeline.err; echo "timeline rc=$?"; cat gpurun_out/s40_timeline.json
for c in 2 3 4 5; do
  for m in copy publish copy publish; do
    timeout 300 python bench.py --config $c --result-read $m > gpurun_out/s40_cfg${c}_$m.json 2>gpurun_out/s40_cfg${c}_$m.err
    echo "cfg$c $m rc=$? $(python -c "import json;d=json.load(open('gpurun_out/s40_cfg${c}_$m.json'));print(d['value'],d['e2e']['value'],d['gpu_launches'],d['clocks'].get('reasons'))" 2>&1 | tail -1)"
  done
done
