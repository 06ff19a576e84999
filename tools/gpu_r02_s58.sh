#!/bin/bash
# 1 GPU: device step timeline with and without the L2 flush before each replay
# (cold vs warm data and kernel code).
mkdir -p gpurun_out
for nf in 0 1; do
  STAMPS_NOFLUSH=$nf DYNMO_LIB=$PWD/ab/libdynmo_stamps.so timeout 300 python tools/step_stamps.py > gpurun_out/s58_stamps_noflush$nf.json 2>&1
  echo "noflush$nf $(python -c "import json;d=json.load(open('gpurun_out/s58_stamps_noflush$nf.json'));print({k:(v['start_us'],v['end_us']) if isinstance(v,dict) else v for k,v in d.items()})")"
done
