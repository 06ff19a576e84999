#!/bin/bash
# 2 GPUs: GPU tier (1-GPU tests on GPU 0 + the 2-rank worker), then the
# exchange-fusion A/B on configs 3 and 2 at N = 2.
mkdir -p gpurun_out
export DYNMO_MGPU_LOG_DIR=gpurun_out DYNMO_MGPU_TIMEOUT=300
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/s23_pytest_gpu.log 2>&1; echo "gpu tier rc=$?"; tail -2 gpurun_out/s23_pytest_gpu.log
cp gpurun_out/mgpu_worker_w2.log gpurun_out/s23_worker_w2.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29619"
for f in 1 0; do for c in 3 2; do
  DYNMO_EXCH_FUSED=$f timeout 300 $TR bench.py --config $c --gpus 2 --steps 300 > gpurun_out/s23_bench_cfg${c}_x$f.json 2> gpurun_out/s23_bench_cfg${c}_x$f.err; echo "cfg$c exch_fused=$f rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/s23_bench_cfg${c}_x$f.json').read().strip().splitlines()[-1]);print(d['value'],d['step_ms']['median'],d['phases_ms_per_launch_diagnostic'])"
done; done
