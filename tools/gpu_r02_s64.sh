#!/bin/bash
# 1 GPU: epilogue code warm-up pass before griddepcontrol.wait
# (DYNMO_EPI_WARM=1, default) vs off: profile parity, device step timeline,
# config 2-5 steps interleaved.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "profile or config5 or sparse or exchange or time" > gpurun_out/s64_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 1 gpurun_out/s64_pytest.log
for w in 0 1; do
  DYNMO_EPI_WARM=$w DYNMO_LIB=$PWD/ab/libdynmo_stamps.so timeout 300 python tools/step_stamps.py > gpurun_out/s64_stamps_warm$w.json 2>&1
  echo "warm$w $(python -c "import json;d=json.load(open('gpurun_out/s64_stamps_warm$w.json'));print({k:(v['start_us'],v['end_us']) if isinstance(v,dict) else v for k,v in d.items()})" 2>&1 | tail -1)"
done
for c in 2 3 4 5; do for w in 0 1 0 1; do
  DYNMO_EPI_WARM=$w timeout 300 python bench.py --config $c --steps 300 > gpurun_out/s64_cfg$c.json 2>/dev/null
  echo "cfg$c warm$w $(python -c "import json;d=json.load(open('gpurun_out/s64_cfg$c.json'));print(d['value'],d['roofline']['frac'],d['clocks']['reasons'])" 2>&1 | tail -1)"
done; done
