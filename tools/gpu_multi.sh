mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l); echo "gpus=$N"
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29511 tests/mgpu_worker.py > gpurun_out/mgpu_worker.log 2>&1; echo mgpu_rc=$?
grep -E "MGPU_OK|Error|error" gpurun_out/mgpu_worker.log | head -20
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $N --steps 50 --warmup 10 > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; echo bench_rc=$?
tail -5 gpurun_out/bench_n$N.err
