#!/bin/bash
# Bounds-checked pass (stands in for compute-sanitizer memcheck, which this
# pool does not allow): every GPU test and the mixed-source run against
# libdynmo_dbg.so, whose kernels assert each scratch / smem / table index.
mkdir -p gpurun_out
export DYNMO_DEBUG=1
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/bounds_pytest.log 2>&1; echo bounds_pytest_rc=$?
tail -3 gpurun_out/bounds_pytest.log
timeout 300 python tools/sanitize_run.py > gpurun_out/bounds_sanitize_run.log 2>&1; echo bounds_run_rc=$?
grep -h DYNMO_BOUNDS gpurun_out/bounds_*.log | head
