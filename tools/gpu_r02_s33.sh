#!/bin/bash
# 1 GPU: interval-sum search: solver parity, config-5 solvers, solver
# microbench (latency mode), bench configs 5 and 2.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "repack or partition or config5 or search_paths or map_stages or bench_configs" > gpurun_out/s33_pytest.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/s33_pytest.log
timeout 300 python tools/cfg5_solvers.py 2>&1
timeout 300 python tools/solver_microbench.py > /dev/null 2>&1; python -c "import json;d=json.load(open('gpurun_out/solver_microbench.json'));print({k:v for k,v in d.items() if k.startswith(('partition','repack'))})"
for c in 5 2; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --steps 300 > gpurun_out/s33.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/s33.json').read().strip().splitlines()[-1]);print('cfg$c step', d['value'])"
done
