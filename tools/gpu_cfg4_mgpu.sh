#!/bin/bash
# Config 4 (Mixtral-shaped MoE, 2.90 GB per moved layer) at 1/2/4 GPUs.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
for a in 4 64; do
  CUDA_VISIBLE_DEVICES=0 timeout 600 python tools/bench_cfg4_mgpu.py --alpha $a --force-shift 0 > gpurun_out/cfg4_a${a}_n1.json 2> gpurun_out/cfg4_a${a}_n1.err; echo "a=$a n=1 rc=$?"; tail -1 gpurun_out/cfg4_a${a}_n1.json
  for n in 2 4; do
    [ $n -gt $N ] && continue
    CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((n-1))) timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 2961$n tools/bench_cfg4_mgpu.py --alpha $a > gpurun_out/cfg4_a${a}_n$n.json 2> gpurun_out/cfg4_a${a}_n$n.err; echo "a=$a n=$n rc=$?"; tail -1 gpurun_out/cfg4_a${a}_n$n.json
  done
done
