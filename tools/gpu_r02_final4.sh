#!/bin/bash
# Round-2 final evidence (session 4) on 4 B200s: the multi-GPU worker at 2 and 4 ranks,
# bench configs 2-5 at N = 2 and 4, the backward-overlap measurement.
T=r02g
mkdir -p gpurun_out
export DYNMO_MGPU_LOG_DIR=gpurun_out DYNMO_MGPU_TIMEOUT=300
timeout 700 python -m pytest tests/test_multigpu.py -m gpu -q -p no:cacheprovider > gpurun_out/${T}_pytest_mgpu.log 2>&1; echo mgpu_rc=$?
tail -2 gpurun_out/${T}_pytest_mgpu.log
for n in 2 4; do
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2963$n"
  for c in 2 3 4 5; do
    timeout 300 $TR bench.py --config $c --gpus $n > gpurun_out/${T}_bench_cfg${c}_n${n}.json 2> gpurun_out/${T}_bench_cfg${c}_n${n}.err; echo "bench cfg$c n$n rc=$? $(python -c "import json;d=json.load(open('gpurun_out/${T}_bench_cfg${c}_n${n}.json'));print(d['value'],d['clocks']['reasons'])" 2>&1 | tail -1)"
  done
done
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29639"
timeout 300 $TR tools/bench_bwd_overlap.py > gpurun_out/${T}_bwd_overlap.json 2> gpurun_out/${T}_bwd_overlap.err; echo bwd_rc=$?
