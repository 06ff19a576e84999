mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l); echo "gpus=$N"
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29511 tests/mgpu_worker.py > gpurun_out/mgpu_worker.log 2>&1; echo mgpu_rc=$?
grep -c MGPU_OK gpurun_out/mgpu_worker.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 200 --warmup 20 --cpu-seconds 12 > gpurun_out/s_n1.json 2> gpurun_out/s_n1.err; echo n1_rc=$?
for n in 2 4; do
  [ $n -gt $N ] && continue
  CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((n-1))) timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 2952$n bench.py --gpus $n --steps 200 --warmup 20 > gpurun_out/s_n$n.json 2> gpurun_out/s_n$n.err; echo n${n}_rc=$?
  CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((n-1))) timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 2953$n bench.py --gpus $n --steps 200 --warmup 20 --host-migrate --e2e-steps 3 > gpurun_out/s_n${n}_host.json 2> gpurun_out/s_n${n}_host.err; echo n${n}host_rc=$?
done
tail -3 gpurun_out/s_n*.err | grep -v OMP | grep -v "\*\*\*"
