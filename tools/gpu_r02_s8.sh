#!/bin/bash
# 4 GPUs: multi-GPU worker (2 and 4 ranks), bench configs 2-5 at N = 2 and 4,
# the 2-rank backward overlap, and compute-sanitizer (memcheck / racecheck /
# synccheck) on the mixed-source + solver run on one GPU.
mkdir -p gpurun_out
export DYNMO_MGPU_LOG_DIR=gpurun_out
timeout 900 python -m pytest tests/test_multigpu.py -m gpu -q -p no:cacheprovider > gpurun_out/s8_pytest_mgpu.log 2>&1; echo "mgpu rc=$?"; tail -2 gpurun_out/s8_pytest_mgpu.log
for n in 2 4; do
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2961$n"
  for c in 2 3 4 5; do
    timeout 900 $TR bench.py --config $c --gpus $n > gpurun_out/s8_bench_cfg${c}_n${n}.json 2> gpurun_out/s8_bench_cfg${c}_n${n}.err; echo "bench cfg$c n$n rc=$?"
  done
done
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29619"
timeout 600 $TR tools/bench_bwd_overlap.py > gpurun_out/s8_bwd_overlap.json 2> gpurun_out/s8_bwd_overlap.err; echo "bwd rc=$?"
export CUDA_VISIBLE_DEVICES=0
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/s8_sanitize_$tool.log 2>&1; echo "sanitizer $tool rc=$?"
  tail -3 gpurun_out/s8_sanitize_$tool.log
done
