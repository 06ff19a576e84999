#!/bin/bash
# 2 GPUs: interleaved backward-overlap measurement (drain / hints), then the
# ncu source profile of the config-5 solvers on GPU 0.
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29617"
for cfg in "1 0" "1 1" "0 0"; do
  set -- $cfg
  DYNMO_BWD_DRAIN=$1 DYNMO_PULL_HINT=$2 timeout 300 $TR tools/bench_bwd_overlap.py > gpurun_out/s12_bwd_d$1_h$2.json 2> gpurun_out/s12_bwd_d$1_h$2.err; echo "d=$1 h=$2 rc=$?"
  tail -1 gpurun_out/s12_bwd_d$1_h$2.json
done
CUDA_VISIBLE_DEVICES=0 bash tools/gpu_r02_s9.sh
