#!/bin/bash
# Round-2 session 3 on 2 B200s: GPU tests incl. the 2-rank worker (lazy-load
# fix for the backward-ordered migration), the backward-overlap benchmark, and
# per-config bench lines + ncu captures of k_profile (traffic per workload).
mkdir -p gpurun_out
export DYNMO_MGPU_LOG_DIR=gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/s3_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/s3_pytest_gpu.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611"
timeout 600 $TR tools/bench_bwd_overlap.py > gpurun_out/s3_bwd_overlap.json 2> gpurun_out/s3_bwd_overlap.err; echo "bwd_overlap rc=$?"
cat gpurun_out/s3_bwd_overlap.json
for c in 2 3 4 5; do
  timeout 600 python bench.py --config $c > gpurun_out/s3_bench_cfg${c}_n1.json 2> gpurun_out/s3_bench_cfg${c}_n1.err; echo "bench cfg$c n1 rc=$?"
  timeout 900 $TR bench.py --config $c --gpus 2 > gpurun_out/s3_bench_cfg${c}_n2.json 2> gpurun_out/s3_bench_cfg${c}_n2.err; echo "bench cfg$c n2 rc=$?"
done
for c in 3 4 5; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_profile -s 5 -c 1 \
    -o gpurun_out/s3_ncu_cfg${c}_k_profile python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/s3_ncu_cfg${c}.log 2>&1
  echo "ncu cfg$c rc=$?"
done
echo done
