#!/bin/bash
# Round evidence on one B200: GPU tests, per-config timings, the N=1 bench
# line, its ncu launch list, and one full ncu capture of k_profile (each ncu
# pass only after the same command exited 0 without ncu).
#   bash tools/gpu_evidence.sh TAG
T=${1:-r01}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/${T}_pytest_gpu.log
timeout 600 python tools/bench_configs.py > gpurun_out/${T}_bench_configs.log 2>&1; echo configs_rc=$?
cp gpurun_out/bench_configs.json gpurun_out/${T}_bench_configs.json 2>/dev/null
timeout 600 python bench.py > gpurun_out/${T}_bench_n1.json 2> gpurun_out/${T}_bench_n1.err; echo bench_rc=$?
timeout 300 python tools/step_timeline.py > gpurun_out/${T}_timeline.json 2>&1; echo timeline_rc=$?
CMD="python bench.py --steps 20 --warmup 5 --e2e-steps 1 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_n1.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch=$?
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_profile -s 5 -c 1 -o gpurun_out/${T}_ncu_k_profile $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu_full=$?
