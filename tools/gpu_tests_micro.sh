mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
python tools/solver_microbench.py > gpurun_out/micro.log 2>&1
cat gpurun_out/pytest_gpu.log; grep -v "^rounds" gpurun_out/micro.log | head -14
