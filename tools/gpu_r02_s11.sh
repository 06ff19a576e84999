#!/bin/bash
# 2 GPUs: backward-overlap A/B (drain on/off x streaming hints), 2 reps each.
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29617"
for rep in 1 2; do
for d in 1 0; do for h in 0 1; do
  DYNMO_BWD_DRAIN=$d DYNMO_PULL_HINT=$h timeout 300 $TR tools/bench_bwd_overlap.py > gpurun_out/s11_bwd_d${d}_h${h}_r$rep.json 2>/dev/null
  echo "drain=$d hint=$h rep=$rep rc=$? $(python -c "import json;d=json.load(open('gpurun_out/s11_bwd_d${d}_h${h}_r$rep.json'));print(d['bwd_alone_ms'],d['seq_ms'],[(r['ctas'],r['overlap_ms'],r['hidden_frac']) for r in d['overlap']])")"
done; done; done
