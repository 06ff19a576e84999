#!/bin/bash
# 1 GPU: event-bracket overhead of the k_profile timing (tools/event_overhead.py)
# and the ramp of short HBM reads (tools/lat/ramp.cu).
mkdir -p gpurun_out
timeout 600 python tools/event_overhead.py > gpurun_out/s5_event_overhead.jsonl 2> gpurun_out/s5_event_overhead.err; echo "evo rc=$?"
cat gpurun_out/s5_event_overhead.jsonl; tail -3 gpurun_out/s5_event_overhead.err
nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/lat/ramp.cu -o /tmp/ramp && \
for b in 67108864 75497472 151000000 184170496 603979776; do timeout 120 /tmp/ramp $b; done > gpurun_out/s5_ramp.txt 2>&1; echo "ramp rc=$?"
cat gpurun_out/s5_ramp.txt
