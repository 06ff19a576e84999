#!/bin/bash
# 1 GPU: k_profile at the per-GPU shares of config 2; compute-sanitizer, bounded (memcheck on the mixed-source + solver
# run; racecheck / synccheck on its small variant).
mkdir -p gpurun_out
timeout 300 python tools/profile_shares.py > gpurun_out/s14_profile_shares.jsonl 2> gpurun_out/s14_profile_shares.err; echo "shares rc=$?"; cat gpurun_out/s14_profile_shares.jsonl
export CUDA_VISIBLE_DEVICES=0
timeout 420 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_run.py > gpurun_out/s13_sanitize_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -3 gpurun_out/s13_sanitize_memcheck.log
export DYNMO_SANITIZE_SMALL=1
for tool in racecheck synccheck; do
  timeout 420 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/s13_sanitize_$tool.log 2>&1; echo "$tool rc=$?"; tail -3 gpurun_out/s13_sanitize_$tool.log
done
