mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l); echo "gpus=$N"
nvidia-smi topo -m | head -8
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29511 tests/mgpu_worker.py > gpurun_out/mgpu_worker4.log 2>&1; echo mgpu_rc=$?
grep -E "MGPU_OK|Error|error|assert" gpurun_out/mgpu_worker4.log | head -20
for ex in p2p nccl; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $N --steps 50 --warmup 10 --exchange $ex --e2e-steps 3 > gpurun_out/bench_n${N}_ex$ex.json 2> gpurun_out/bench_n${N}_ex$ex.err; echo bench_${ex}_rc=$?
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus $N --steps 50 --warmup 10 --exchange nccl --migrate nccl --e2e-steps 2 > gpurun_out/bench_n${N}_allnccl.json 2> gpurun_out/bench_n${N}_allnccl.err; echo bench_allnccl_rc=$?
