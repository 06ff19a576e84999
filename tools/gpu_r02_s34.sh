#!/bin/bash
# 1 GPU: gated interval-sum enumeration in the batched mode too: solver
# parity, config-5 solvers and step vs the latency-mode-only build.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "repack or partition or config5 or search_paths" > gpurun_out/s34_pytest.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/s34_pytest.log
for lib in ab/libdynmo_enumlat.so paper_2505_14864_b200/libdynmo.so ab/libdynmo_enumlat.so paper_2505_14864_b200/libdynmo.so; do
  tag=$(basename $lib .so)
  DYNMO_LIB=$PWD/$lib timeout 300 python tools/cfg5_solvers.py 2>&1 | sed "s/^/$tag /" | grep -v nomem
done
