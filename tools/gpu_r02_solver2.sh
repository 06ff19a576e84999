#!/bin/bash
# Solver v2 (32-bit views, probe round, jumps in the batched mode): parity,
# timings, bench 2/5; ncu stall profile of the fluid diffusion; in-situ
# k_profile durations of the config-5 bench (no cache flush by ncu).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "partition or repack or config5 or diffuse or map_stages or bench_configs" > gpurun_out/sv2_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/sv2_pytest.log
timeout 300 python tools/solver_microbench.py > /dev/null 2> gpurun_out/sv2_solver_microbench.err; echo "micro rc=$?"
cp gpurun_out/solver_microbench.json gpurun_out/sv2_solver_microbench.json
timeout 300 python tools/cfg5_solvers.py > gpurun_out/sv2_cfg5_solvers.txt 2>&1; echo "cfg5 rc=$?"
cat gpurun_out/sv2_cfg5_solvers.txt
for c in 2 5; do
  timeout 600 python bench.py --config $c > gpurun_out/sv2_bench_cfg${c}_n1.json 2> gpurun_out/sv2_bench_cfg${c}_n1.err; echo "bench cfg$c rc=$?"
done
ncu --section SourceCounters --section WarpStateStats --warp-sampling-interval 0 --import-source on --clock-control none \
  -k regex:"k_diffuse" -s 1 -c 1 -o gpurun_out/sv2_ncu_diffuse python tools/solver_one.py diffuse > gpurun_out/sv2_ncu_diffuse.log 2>&1; echo ncu_diff=$?
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:k_profile --csv \
  --log-file gpurun_out/sv2_insitu_cfg5.csv python bench.py --config 5 --steps 8 --warmup 3 > gpurun_out/sv2_insitu_cfg5.log 2>&1; echo ncu_insitu=$?
