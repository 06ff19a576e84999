#!/bin/bash
# Round-2 session on 2 B200s: GPU tests (incl. the 2-rank worker), the
# backward-overlap benchmark, bench.py --config 2..5 at N=1 and N=2, and the
# plain-read / TMA-read ceilings at the profile's sizes.
mkdir -p gpurun_out
export DYNMO_MGPU_LOG_DIR=gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/s2_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/s2_pytest_gpu.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611"
timeout 600 $TR tools/bench_bwd_overlap.py > gpurun_out/s2_bwd_overlap.json 2> gpurun_out/s2_bwd_overlap.err; echo "bwd_overlap rc=$?"
for c in 2 3 4 5; do
  timeout 600 python bench.py --config $c > gpurun_out/s2_bench_cfg${c}_n1.json 2> gpurun_out/s2_bench_cfg${c}_n1.err; echo "bench cfg$c n1 rc=$?"
  timeout 900 $TR bench.py --config $c --gpus 2 > gpurun_out/s2_bench_cfg${c}_n2.json 2> gpurun_out/s2_bench_cfg${c}_n2.err; echo "bench cfg$c n2 rc=$?"
done
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/hbm_read tools/lat/hbm_read.cu && \
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/tma_read tools/lat/tma_read.cu
for b in 67108864 75497472 151000000 603979776; do
  echo "== bytes=$b" >> gpurun_out/s2_read_ceiling.txt
  timeout 120 /tmp/hbm_read $b >> gpurun_out/s2_read_ceiling.txt 2>&1
  timeout 120 /tmp/tma_read $b >> gpurun_out/s2_read_ceiling.txt 2>&1
done
echo done
