#!/bin/bash
# Pruning at 1..N GPUs (+ the multi-rank parity worker), each under its own timeout.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l); echo "gpus=$N"
CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((N-1))) timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29511 tests/mgpu_worker.py > gpurun_out/mgpu_worker.log 2>&1; echo mgpu_rc=$?
CUDA_VISIBLE_DEVICES=0 timeout 200 python tools/bench_prune.py > gpurun_out/prune_n1.json 2>/dev/null; echo prune1_rc=$?
for n in 2 4; do
  [ $n -gt $N ] && continue
  CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((n-1))) timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 2954$n tools/bench_prune.py 2>/dev/null | grep "{" > gpurun_out/prune_n$n.json; echo prune${n}_rc=$?
done
cat gpurun_out/prune_n*.json
python tools/prune_one.py > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prune_launches.csv python tools/prune_one.py > /dev/null 2>&1; echo prune_ncu_rc=$?
