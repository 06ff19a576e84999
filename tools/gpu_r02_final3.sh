#!/bin/bash
# Round-2 final evidence (session 3) on one B200: GPU tier, smoke, bench N=1
# for configs 2-5, the config-2 ncu launch list (same command, after it
# exited 0 without ncu), the step timeline and the fluid phase cycles.
T=r02g
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${T}_smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/${T}_smoke.log
for c in 2 3 4 5; do
  timeout 600 python bench.py --config $c > gpurun_out/${T}_bench_cfg${c}_n1.json 2> gpurun_out/${T}_bench_cfg${c}_n1.err; echo "bench cfg$c rc=$? $(python -c "import json;d=json.load(open('gpurun_out/${T}_bench_cfg${c}_n1.json'));print(d['value'],d['roofline']['frac'],d['clocks']['reasons'])" 2>&1 | tail -1)"
done
CMD="python bench.py --steps 20 --warmup 5 --e2e-steps 1 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_n1.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch=$?
timeout 300 python tools/step_timeline.py > gpurun_out/${T}_step_timeline.json 2>&1; echo timeline=$?
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Ipaper_2505_14864_b200/csrc -Iinclude -I/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/include -fmad=false -DDYNMO_FLUID_PROF -c paper_2505_14864_b200/csrc/k_solve.cu -o /tmp/kp.o 2>/dev/null && \
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o /tmp/libdynmo_fprof.so $(ls paper_2505_14864_b200/csrc/build/*.o | grep -v k_solve.o) /tmp/kp.o -L/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib -l:libnccl.so.2 && \
DYNMO_LIB=/tmp/libdynmo_fprof.so timeout 120 python tools/fluid_prof.py > gpurun_out/${T}_fluid_phases.jsonl 2>&1; echo fluid_prof=$?
