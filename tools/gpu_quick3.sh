mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/pytest_gpu.log
python tools/solver_microbench.py > gpurun_out/micro.log 2>&1
python bench.py --steps 50 --warmup 10 --cpu-seconds 3 > gpurun_out/bench_graph.json 2> gpurun_out/bench_graph.err; echo bench_graph_rc=$?
cat gpurun_out/pytest_gpu.log; grep -v "^rounds" gpurun_out/micro.log | tail -34
