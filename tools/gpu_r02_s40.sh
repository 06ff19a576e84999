#!/bin/bash
# 1 GPU: CTA-combined final flushes: profile parity, k_profile span/events
# for configs 4, 2, 5 vs the final-evidence build.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "profile or config5 or moe or exchange or sparse or time" > gpurun_out/s40_pytest.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/s40_pytest.log
for rep in 1 2; do for lib in ab/libdynmo_enumlat.so paper_2505_14864_b200/libdynmo.so; do for c in 4 2 5; do
  tag=$(basename $lib .so)
  DYNMO_LIB=$PWD/$lib timeout 600 python bench.py --config $c --no-cpu-baseline --steps 300 > gpurun_out/s40.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/s40.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$tag cfg$c', d['value'],r['avg_launch_ms'],r['kernel_span_ms'])"
done; done; done
