#!/bin/bash
# 1 GPU: k_diffuse code warm-up before griddepcontrol.wait + the diffusion on
# the main stream: diffusion parity, device timelines (layouts x warm), and
# config 2/3/4 steps (--diffuse-branch main/side, DYNMO_DIFF_WARM 1/0).
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "diffuse" > gpurun_out/s65_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 1 gpurun_out/s65_pytest.log
for lay in 1 0; do for w in 1 0; do
  STAMPS_DIFF_MAIN=$lay DYNMO_DIFF_WARM=$w DYNMO_LIB=$PWD/ab/libdynmo_stamps.so timeout 300 python tools/step_stamps.py > gpurun_out/s65_stamps_main${lay}_warm$w.json 2>&1
  echo "main$lay warm$w $(python -c "import json;d=json.load(open('gpurun_out/s65_stamps_main${lay}_warm$w.json'));print({k:(v['start_us'],v['end_us']) if isinstance(v,dict) else v for k,v in d.items() if k!='profile'})" 2>&1 | tail -1)"
done; done
for c in 2 3 4; do for v in "main 1" "side 1" "main 0" "main 1" "side 1" "main 0"; do
  set -- $v
  DYNMO_DIFF_WARM=$2 timeout 300 python bench.py --config $c --steps 300 --diffuse-branch $1 > gpurun_out/s65_cfg$c.json 2>/dev/null
  echo "cfg$c branch=$1 warm=$2 $(python -c "import json;d=json.load(open('gpurun_out/s65_cfg$c.json'));print(d['value'],d['clocks']['reasons'])" 2>&1 | tail -1)"
done; done
