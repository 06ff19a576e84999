mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | grep -E "^E |FAILED|passed|failed" | head -12
bash tools/gpu_scale.sh
# NEXT-3 migration overlapped with compute (2 GPUs)
CUDA_VISIBLE_DEVICES=0,1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29612 tools/bench_overlap.py 2>/dev/null | grep "^{" > gpurun_out/overlap.json; echo overlap_rc=$?
# per-kernel prune launch list (G = 1)
python tools/prune_one.py > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prune_launches.csv python tools/prune_one.py > /dev/null 2>&1; echo prune_ncu_rc=$?
