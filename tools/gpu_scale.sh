#!/bin/bash
# Multi-GPU evidence: mgpu_worker (parity) and the bench at 1/2/4 GPUs
# (identity placement and --map-stages), each run under its own timeout.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l); echo "gpus=$N"
CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((N-1))) timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29511 tests/mgpu_worker.py > gpurun_out/mgpu_worker.log 2>&1; echo mgpu_rc=$?
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py > gpurun_out/s_n1.json 2> gpurun_out/s_n1.err; echo n1_rc=$?
for n in 2 4; do
  [ $n -gt $N ] && continue
  for m in "" "--map-stages"; do
    CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((n-1))) timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 2952$n bench.py --gpus $n $m > gpurun_out/s_n$n$m.json 2> gpurun_out/s_n$n$m.err; echo "n${n}${m}_rc=$?"
  done
  CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((n-1))) timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 2953$n bench.py --gpus $n --host-migrate --e2e-steps 3 > gpurun_out/s_n${n}_host.json 2> gpurun_out/s_n${n}_host.err; echo n${n}host_rc=$?
done
for f in gpurun_out/s_n*.json; do python tools/summarize.py $f 2>/dev/null | head -3; done
# Alg. 1 global pruning at 1..N GPUs
CUDA_VISIBLE_DEVICES=0 timeout 200 python tools/bench_prune.py > gpurun_out/prune_n1.json 2>/dev/null; echo prune1_rc=$?
for n in 2 4; do
  [ $n -gt $N ] && continue
  CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((n-1))) timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 2954$n tools/bench_prune.py 2>/dev/null | grep "{" > gpurun_out/prune_n$n.json; echo prune${n}_rc=$?
done
cat gpurun_out/prune_n*.json
