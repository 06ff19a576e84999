#!/bin/bash
# 1 GPU: config-2 step timeline (branch completion offsets) with the
# speculative fluid rounds and with the per-round chain.
mkdir -p gpurun_out
for sp in 1 0; do
  DYNMO_FLUID_SPEC=$sp timeout 300 python tools/step_timeline.py > gpurun_out/s38_timeline_spec$sp.json 2> gpurun_out/s38_timeline_spec$sp.err; echo "spec$sp rc=$?"
  cat gpurun_out/s38_timeline_spec$sp.json; tail -3 gpurun_out/s38_timeline_spec$sp.err
done
