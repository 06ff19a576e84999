mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | grep -E "^E |FAILED|passed|failed" | head -12
bash tools/gpu_scale.sh
