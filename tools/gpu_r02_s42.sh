#!/bin/bash
# 1 GPU: publish test (kernel <= 4 KiB, copy engine above), full GPU tier,
# bench configs 2..5 (default = publish) and the publish microbench.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/s42_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s42_pytest_gpu.log
timeout 300 python tools/publish_bench.py > gpurun_out/s42_publish_bench.jsonl 2>&1; cat gpurun_out/s42_publish_bench.jsonl
for c in 2 3 4 5; do
  timeout 300 python bench.py --config $c > gpurun_out/s42_bench_cfg${c}_n1.json 2>gpurun_out/s42_bench_cfg${c}_n1.err
  echo "cfg$c rc=$? $(python -c "import json;d=json.load(open('gpurun_out/s42_bench_cfg${c}_n1.json'));print(d['value'],d['e2e']['value'],d['gpu_launches'],d['roofline']['frac'],d['clocks'])" 2>&1 | tail -1)"
done
