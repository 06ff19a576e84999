#!/bin/bash
# 2 GPUs: the traced worker with the window watchdog.
mkdir -p gpurun_out
export DYNMO_MGPU_LOG_DIR=gpurun_out DYNMO_MGPU_TIMEOUT=300
timeout 300 python -m pytest "tests/test_multigpu.py::test_exchange_and_migration[2]" -q -p no:cacheprovider > gpurun_out/s22_pytest_w2.log 2>&1; echo "w2 warm rc=$?"
grep -h "TRACE 0\|TRACE 1\|TIMEOUT\|Error" gpurun_out/mgpu_worker_w2.log | tail -8
cp gpurun_out/mgpu_worker_w2.log gpurun_out/s22_worker_w2_wd.log
