#!/bin/bash
# Solver rewrite check (1 GPU): solver parity tests, isolated solver timings
# (config 2 shapes and config 5's 4096-instance batch), bench configs 2 and 5.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "partition or repack or config5 or diffuse or map_stages or bench_configs" > gpurun_out/sv_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/sv_pytest.log
timeout 300 python tools/solver_microbench.py > gpurun_out/sv_solver_microbench.json 2> gpurun_out/sv_solver_microbench.err; echo "micro rc=$?"
timeout 300 python tools/cfg5_solvers.py > gpurun_out/sv_cfg5_solvers.json 2> gpurun_out/sv_cfg5_solvers.err; echo "cfg5 rc=$?"
cat gpurun_out/sv_cfg5_solvers.json
for c in 2 5; do
  timeout 600 python bench.py --config $c > gpurun_out/sv_bench_cfg${c}_n1.json 2> gpurun_out/sv_bench_cfg${c}_n1.err; echo "bench cfg$c rc=$?"
done
