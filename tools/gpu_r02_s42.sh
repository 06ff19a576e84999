#!/bin/bash
# 2 GPUs: fence-skip in the fused migration: worker (2 ranks), bench configs 3
# and 2 at N = 2 (two runs each).
mkdir -p gpurun_out
export DYNMO_MGPU_LOG_DIR=gpurun_out DYNMO_MGPU_TIMEOUT=300
timeout 400 python -m pytest "tests/test_multigpu.py::test_exchange_and_migration[2]" -q -p no:cacheprovider > gpurun_out/s42_pytest_w2.log 2>&1; echo "w2 rc=$?"
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29642"
for rep in 1 2; do for c in 3 2; do
  timeout 300 $TR bench.py --config $c --gpus 2 --steps 300 > gpurun_out/s42.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/s42.json').read().strip().splitlines()[-1]);print('cfg$c', d['value'], d['phases_ms_per_launch_diagnostic'].get('migrate'))"
done; done
