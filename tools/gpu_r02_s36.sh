#!/bin/bash
# 1 GPU: two candidates per lane in the batched mode: solver parity, config-5
# solvers and step vs the final-evidence build.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "repack or partition or config5 or search_paths" > gpurun_out/s36_pytest.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/s36_pytest.log
for lib in ab/libdynmo_enumlat.so paper_2505_14864_b200/libdynmo.so ab/libdynmo_enumlat.so paper_2505_14864_b200/libdynmo.so; do
  tag=$(basename $lib .so)
  DYNMO_LIB=$PWD/$lib timeout 300 python tools/cfg5_solvers.py 2>&1 | sed "s/^/$tag /" | grep -v nomem
  DYNMO_LIB=$PWD/$lib timeout 600 python bench.py --config 5 --no-cpu-baseline --steps 300 > gpurun_out/s36.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/s36.json').read().strip().splitlines()[-1]);print('$tag cfg5 step', d['value'])"
done
