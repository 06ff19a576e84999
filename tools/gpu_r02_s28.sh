#!/bin/bash
# 1 GPU: A/B of the counter layout (field-major vs slot-major), configs 5, 2.
mkdir -p gpurun_out
for rep in 1 2; do for lib in ab/libdynmo_prevacc.so paper_2505_14864_b200/libdynmo.so; do for c in 5 2; do
  DYNMO_LIB=$PWD/$lib timeout 600 python bench.py --config $c --no-cpu-baseline --steps 300 > gpurun_out/s28.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/s28.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$lib cfg$c', d['value'],r['avg_launch_ms'],r['kernel_span_ms'],d['clocks']['sm_mhz'])"
done; done; done
