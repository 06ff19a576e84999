mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l); echo "gpus=$N"
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29511 tests/mgpu_worker.py > gpurun_out/mgpu_worker.log 2>&1; echo mgpu_rc=$?
grep -E "MGPU_OK|Error|error|assert" gpurun_out/mgpu_worker.log | head -20
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $N --steps 50 --warmup 10 > gpurun_out/bench_n${N}_p2p.json 2> gpurun_out/bench_n${N}_p2p.err; echo bench_p2p_rc=$?
tail -3 gpurun_out/bench_n${N}_p2p.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus $N --steps 50 --warmup 10 --migrate nccl --exchange nccl --e2e-steps 2 > gpurun_out/bench_n${N}_nccl.json 2> gpurun_out/bench_n${N}_nccl.err; echo bench_nccl_rc=$?
