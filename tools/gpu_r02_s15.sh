#!/bin/bash
# 2 GPUs: worker (fused device migration, multi-chunk backward migration),
# bench configs 2 and 3 at N = 2 with the fused / three-kernel migration.
mkdir -p gpurun_out
export DYNMO_MGPU_LOG_DIR=gpurun_out
timeout 600 python -m pytest tests/test_multigpu.py -m gpu -q -p no:cacheprovider > gpurun_out/s15_pytest_mgpu.log 2>&1; echo "mgpu rc=$?"; tail -2 gpurun_out/s15_pytest_mgpu.log
grep -E "Error|assert" gpurun_out/mgpu_worker_w2.log | head -5
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29618"
for f in 1 0; do for c in 3 2; do
  DYNMO_MIG_FUSED=$f timeout 300 $TR bench.py --config $c --gpus 2 --steps 200 > gpurun_out/s15_bench_cfg${c}_f$f.json 2> gpurun_out/s15_bench_cfg${c}_f$f.err; echo "cfg$c fused=$f rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/s15_bench_cfg${c}_f$f.json').read().strip().splitlines()[-1]);print(d['value'],d['step_ms']['median'],d['phases_ms_per_launch_diagnostic'])"
done; done
