#!/bin/bash
# 2 GPUs: traced 2-rank worker, short timeout.
mkdir -p gpurun_out
export DYNMO_MGPU_LOG_DIR=gpurun_out DYNMO_MGPU_TIMEOUT=150
timeout 300 python -m pytest "tests/test_multigpu.py::test_exchange_and_migration[2]" -q -p no:cacheprovider > gpurun_out/s17_pytest_w2.log 2>&1; echo "w2 rc=$?"
grep -h "TRACE\|TIMEOUT\|Error\|error" gpurun_out/mgpu_worker_w2.log | tail -30
cp gpurun_out/mgpu_worker_w2.log gpurun_out/s17_worker_w2.log
