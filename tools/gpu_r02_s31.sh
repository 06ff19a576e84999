#!/bin/bash
# 1 GPU: epilogue rewrite: profile parity, per-kernel launch list of the
# config-5 step (previous build vs this one), bench configs 5 and 2.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "profile or config5 or exchange or prune_reproduces or sparse or time or overflow" > gpurun_out/s31_pytest.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/s31_pytest.log
for lib in ab/libdynmo_prevacc.so paper_2505_14864_b200/libdynmo.so; do
  tag=$(basename $lib .so)
  DYNMO_LIB=$PWD/$lib ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s31_$tag.csv \
    python bench.py --config 5 --steps 8 --warmup 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1; echo "$tag rc=$?"
  python tools/ncu_kernel_means.py gpurun_out/s31_$tag.csv | grep dynmo
  for c in 5 2; do
    DYNMO_LIB=$PWD/$lib timeout 600 python bench.py --config $c --no-cpu-baseline --steps 300 > gpurun_out/s31.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/s31.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$tag cfg$c', d['value'],r['avg_launch_ms'],r['kernel_span_ms'])"
  done
done
