#!/bin/bash
# 1 GPU: device step timeline (L2 flushed) with the solvers pre-run on a
# stale profile during k_profile (instruction/data warm-up) vs without.
mkdir -p gpurun_out
for pw in 0 1 0 1; do
  STAMPS_PREWARM=$pw DYNMO_LIB=$PWD/ab/libdynmo_stamps.so timeout 300 python tools/step_stamps.py > gpurun_out/s59_stamps_prewarm$pw.json 2>&1
  echo "prewarm$pw $(python -c "import json;d=json.load(open('gpurun_out/s59_stamps_prewarm$pw.json'));print({k:(v['start_us'],v['end_us']) if isinstance(v,dict) else v for k,v in d.items()})" 2>&1 | tail -1)"
done
