#!/bin/bash
# 4 GPUs: bench configs 2-5 at N = 4; then compute-sanitizer on GPU 0
# (memcheck on the mixed-source + solver run; racecheck / synccheck on its
# small variant), each bounded.
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29624"
for c in 2 3 4 5; do
  timeout 420 $TR bench.py --config $c --gpus 4 > gpurun_out/s13_bench_cfg${c}_n4.json 2> gpurun_out/s13_bench_cfg${c}_n4.err; echo "bench cfg$c n4 rc=$?"
done
export CUDA_VISIBLE_DEVICES=0
timeout 420 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_run.py > gpurun_out/s13_sanitize_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -3 gpurun_out/s13_sanitize_memcheck.log
export DYNMO_SANITIZE_SMALL=1
for tool in racecheck synccheck; do
  timeout 420 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/s13_sanitize_$tool.log 2>&1; echo "$tool rc=$?"; tail -3 gpurun_out/s13_sanitize_$tool.log
done
