#!/bin/bash
# 2 GPUs: the 2-rank worker with section traces (fused device migration by
# default); on failure once more with the three-kernel migration.
mkdir -p gpurun_out
export DYNMO_MGPU_LOG_DIR=gpurun_out
timeout 500 python -m pytest "tests/test_multigpu.py::test_exchange_and_migration[2]" -q -p no:cacheprovider > gpurun_out/s16_pytest_w2.log 2>&1; rc=$?; echo "w2 fused rc=$rc"
grep -h "TRACE 0\|TIMEOUT\|Error" gpurun_out/mgpu_worker_w2.log | tail -4
cp gpurun_out/mgpu_worker_w2.log gpurun_out/s16_worker_w2_fused.log
if [ $rc -ne 0 ]; then
  DYNMO_MIG_FUSED=0 timeout 500 python -m pytest "tests/test_multigpu.py::test_exchange_and_migration[2]" -q -p no:cacheprovider > gpurun_out/s16_pytest_w2_nofuse.log 2>&1; echo "w2 3-kernel rc=$?"
  grep -h "TRACE 0\|TIMEOUT\|Error" gpurun_out/mgpu_worker_w2.log | tail -4
  cp gpurun_out/mgpu_worker_w2.log gpurun_out/s16_worker_w2_nofuse.log
fi
