#!/bin/bash
# 1 GPU: the epilogue's inputs prefetched into L2 by k_profile
# (DYNMO_EPI_PREFETCH=1, default) vs not: profile parity, device step
# timeline, config 2-5 steps interleaved.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "profile or config5 or sparse" > gpurun_out/s61_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/s61_pytest.log
for pf in 0 1; do
  DYNMO_EPI_PREFETCH=$pf DYNMO_LIB=$PWD/ab/libdynmo_stamps.so timeout 300 python tools/step_stamps.py > gpurun_out/s61_stamps_pf$pf.json 2>&1
  echo "pf$pf $(python -c "import json;d=json.load(open('gpurun_out/s61_stamps_pf$pf.json'));print({k:(v['start_us'],v['end_us']) if isinstance(v,dict) else v for k,v in d.items()})" 2>&1 | tail -1)"
done
for c in 2 3 4 5; do for pf in 0 1 0 1; do
  DYNMO_EPI_PREFETCH=$pf timeout 300 python bench.py --config $c --steps 300 > gpurun_out/s61_cfg$c.json 2>/dev/null
  echo "cfg$c pf$pf $(python -c "import json;d=json.load(open('gpurun_out/s61_cfg$c.json'));print(d['value'],d['roofline']['frac'],d['clocks']['reasons'])" 2>&1 | tail -1)"
done; done
