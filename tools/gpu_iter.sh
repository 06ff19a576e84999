#!/bin/bash
# One development iteration on the GPU box: every GPU test, the solver
# microbenchmark, and a short N=1 bench (summarised).
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/solver_microbench.py > gpurun_out/smb.log 2>&1; echo smb_rc=$?
tail -c 1200 gpurun_out/smb.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/b1.log 2>&1; echo bench_rc=$?
python tools/summarize.py gpurun_out/b1.log
