#!/bin/bash
# 1 GPU: config-2 step graph -- three solver branches vs one stream, PDL on/off.
mkdir -p gpurun_out
for pdl in 1 0; do
  DYNMO_PDL=$pdl timeout 300 python tools/step_timeline.py > gpurun_out/s39_timeline_pdl$pdl.json 2> gpurun_out/s39_timeline_pdl$pdl.err; echo "pdl$pdl rc=$?"
  cat gpurun_out/s39_timeline_pdl$pdl.json; tail -3 gpurun_out/s39_timeline_pdl$pdl.err
done
