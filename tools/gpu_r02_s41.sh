#!/bin/bash
# 1 GPU: regression of the final code: GPU tier, smoke, bench config 2.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/s41_pytest_gpu.log 2>&1; echo "tier rc=$?"; tail -2 gpurun_out/s41_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/s41_bench.json 2>/dev/null; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/s41_bench.json').read().strip().splitlines()[-1]);r=d['roofline'];print(d['value'],r['frac'],r['frac_span'],d['clocks'])"
