#!/bin/bash
# 1 GPU: the new search-path parity test + the solver tests.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "search_paths or partition or repack" > gpurun_out/s25_pytest.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/s25_pytest.log
