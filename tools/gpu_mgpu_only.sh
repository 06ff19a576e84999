mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29511 tests/mgpu_worker.py > gpurun_out/mgpu_worker.log 2>&1; echo mgpu_rc=$?
grep -E "MGPU_OK|Error|error|assert|Traceback" gpurun_out/mgpu_worker.log | head -20
