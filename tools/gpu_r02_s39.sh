#!/bin/bash
# 4 GPUs: the 4-rank worker with the abort scenario (traced, watchdog).
mkdir -p gpurun_out
export DYNMO_MGPU_LOG_DIR=gpurun_out DYNMO_MGPU_TIMEOUT=300
timeout 400 python -m pytest "tests/test_multigpu.py::test_exchange_and_migration[4]" -q -p no:cacheprovider > gpurun_out/s39_pytest_w4.log 2>&1; echo "w4 rc=$?"
grep -h "TRACE 0 chunks\|TIMEOUT\|Error\|WATCHDOG\|assert" gpurun_out/mgpu_worker_w4.log | tail -12
cp gpurun_out/mgpu_worker_w4.log gpurun_out/s39_worker_w4.log
