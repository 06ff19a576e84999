#!/bin/bash
# 1 GPU: publish test; result-read microbench over bytes per CTA.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "publish" > gpurun_out/s41_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s41_pytest.log
for cb in 16384 4096 1024 256; do
  DYNMO_PUBLISH_CTA_BYTES=$cb timeout 300 python tools/publish_bench.py
done
