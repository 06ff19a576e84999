mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
for mode in graph serial; do
  extra=""; [ $mode = serial ] && extra="--serial-solvers"
  if [ $N -gt 1 ]; then
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $N --steps 100 --warmup 10 --e2e-steps 3 $extra > gpurun_out/b_n${N}_$mode.json 2> gpurun_out/b_n${N}_$mode.err; echo "$mode rc=$?"
  else
    timeout 600 python bench.py --steps 100 --warmup 10 --e2e-steps 3 --no-cpu-baseline $extra > gpurun_out/b_n${N}_$mode.json 2> gpurun_out/b_n${N}_$mode.err; echo "$mode rc=$?"
  fi
  tail -2 gpurun_out/b_n${N}_$mode.err
done
