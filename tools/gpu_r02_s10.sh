#!/bin/bash
# 2 GPUs: worker (drain + chunked backward pulls), overlap benchmark, bench
# N = 2 exit check, then the GPU tier.
mkdir -p gpurun_out
export DYNMO_MGPU_LOG_DIR=gpurun_out
timeout 600 python -m pytest tests/test_multigpu.py -m gpu -q -p no:cacheprovider > gpurun_out/s10_pytest_mgpu.log 2>&1; echo "mgpu rc=$?"; tail -2 gpurun_out/s10_pytest_mgpu.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29617"
timeout 300 $TR tools/bench_bwd_overlap.py > gpurun_out/s10_bwd_overlap.json 2> gpurun_out/s10_bwd_overlap.err; echo "bwd rc=$?"; cat gpurun_out/s10_bwd_overlap.json
timeout 300 $TR bench.py --config 2 --gpus 2 --steps 100 > gpurun_out/s10_bench_cfg2_n2.json 2> gpurun_out/s10_bench_cfg2_n2.err; echo "bench n2 rc=$?"
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_multigpu.py > gpurun_out/s10_pytest_gpu.log 2>&1; echo "gpu tier rc=$?"; tail -2 gpurun_out/s10_pytest_gpu.log
