#!/bin/bash
# 1 GPU: fluid A/B (register-replicated rounds vs shuffles) + diffusion parity.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "diffuse or config5" > gpurun_out/s7_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/s7_pytest.log
for m in 1 0; do
  DYNMO_FLUID_REP8=$m timeout 300 python tools/solver_microbench.py > /dev/null 2>&1; cp gpurun_out/solver_microbench.json gpurun_out/s7_micro_rep8_$m.json
  DYNMO_FLUID_REP8=$m timeout 600 python bench.py --config 3 --no-cpu-baseline > gpurun_out/s7_bench_cfg3_rep8_$m.json 2>/dev/null; echo "bench3 $m rc=$?"
done
python - <<'PY'
import json
for m in (1, 0):
    d = json.load(open(f"gpurun_out/s7_micro_rep8_{m}.json"))
    print(m, {k: v for k, v in d.items() if "fluid" in k})
    b = json.loads(open(f"gpurun_out/s7_bench_cfg3_rep8_{m}.json").read().strip().splitlines()[-1])
    print(m, "cfg3 step", b["value"])
PY
