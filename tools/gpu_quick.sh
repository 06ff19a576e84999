mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
python bench.py --steps 50 --warmup 10 --cpu-seconds 3 > gpurun_out/bench_graph.json 2> gpurun_out/bench_graph.err; echo bench_graph_rc=$?
python bench.py --steps 50 --warmup 10 --no-graph --no-cpu-baseline > gpurun_out/bench_eager.json 2> gpurun_out/bench_eager.err; echo bench_eager_rc=$?
tail -5 gpurun_out/bench_graph.err gpurun_out/bench_eager.err
cat gpurun_out/pytest_gpu.log
