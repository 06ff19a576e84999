mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
python bench.py --steps 50 --warmup 10 --cpu-seconds 3 > gpurun_out/bench_graph.json 2> gpurun_out/bench_graph.err; echo bench_graph_rc=$?
CMD="python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-graph"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01b.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_partition|k_diffuse|k_repack" -s 3 -c 3 -o gpurun_out/prof_solvers_r01 $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu=$?
cat gpurun_out/pytest_gpu.log
