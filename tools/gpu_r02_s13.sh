#!/bin/bash
# 4 GPUs: bench configs 2-5 at N = 4.
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29624"
for c in 2 3 4 5; do
  timeout 420 $TR bench.py --config $c --gpus 4 > gpurun_out/s13_bench_cfg${c}_n4.json 2> gpurun_out/s13_bench_cfg${c}_n4.err; echo "bench cfg$c n4 rc=$?"
done
