#!/bin/bash
# Round-2 final evidence on one B200: GPU tier, smoke, bench N=1 for configs
# 2-5, the config-2 ncu launch list (same command, after it exited 0 without
# ncu) and one ncu --set full capture of k_profile (traffic).
T=r02f
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${T}_smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/${T}_smoke.log
for c in 2 3 4 5; do
  timeout 600 python bench.py --config $c > gpurun_out/${T}_bench_cfg${c}_n1.json 2> gpurun_out/${T}_bench_cfg${c}_n1.err; echo "bench cfg$c rc=$?"
done
CMD="python bench.py --steps 20 --warmup 5 --e2e-steps 1 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_n1.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch=$?
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_profile -s 5 -c 1 -o gpurun_out/${T}_ncu_k_profile $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu_full=$?
