mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
run() { tag=$1; shift; env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus $N --steps 30 --warmup 5 --e2e-steps 2 > gpurun_out/sweep_$tag.json 2> gpurun_out/sweep_$tag.err; echo "$tag rc=$? $(python tools/summarize.py gpurun_out/sweep_$tag.json | grep -E "value|migrate'|exchange" | tr '\n' ' ' | cut -c1-400)"; }
run base X=1
run ch8 NCCL_NCHANNELS_PER_PEER=8
run ch16 NCCL_NCHANNELS_PER_PEER=16 NCCL_MAX_NCHANNELS=32
run cemem NCCL_P2P_USE_CUDA_MEMCPY=1
run ll NCCL_PROTO=LL,LL128,Simple NCCL_NCHANNELS_PER_PEER=8
