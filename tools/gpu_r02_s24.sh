#!/bin/bash
# 1 GPU: step timeline of the config-2 N=1 graph (branch offsets) with the
# current kernels.
mkdir -p gpurun_out
timeout 300 python tools/step_timeline.py > gpurun_out/s24_step_timeline.json 2> gpurun_out/s24_step_timeline.err; echo "timeline rc=$?"
cat gpurun_out/s24_step_timeline.json; tail -3 gpurun_out/s24_step_timeline.err
