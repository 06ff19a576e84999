#!/bin/bash
# 2 GPUs: GPU tier (incl. the 2-rank worker: backward-overlapped migration
# v2 with stream-memory waits), the overlap benchmark, fluid-ballot solver
# timings, and the phase-event A/B of the step graph (configs 2 and 5).
mkdir -p gpurun_out
export DYNMO_MGPU_LOG_DIR=gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/s4_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/s4_pytest_gpu.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611"
timeout 600 $TR tools/bench_bwd_overlap.py > gpurun_out/s4_bwd_overlap.json 2> gpurun_out/s4_bwd_overlap.err; echo "bwd_overlap rc=$?"
cat gpurun_out/s4_bwd_overlap.json
timeout 300 python tools/solver_microbench.py > /dev/null 2>&1; cp gpurun_out/solver_microbench.json gpurun_out/s4_solver_microbench.json
for c in 2 5; do
  for pt in profile none; do
    timeout 600 python bench.py --config $c --phase-timing $pt --no-cpu-baseline > gpurun_out/s4_bench_cfg${c}_${pt}.json 2> gpurun_out/s4_bench_cfg${c}_${pt}.err; echo "bench cfg$c $pt rc=$?"
  done
done
