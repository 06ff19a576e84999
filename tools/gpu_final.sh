#!/bin/bash
# Round-end regression: every GPU test, smoke(), the N=1 bench and the scaling benches.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | grep -E "^E |FAILED|passed|failed" | head -12
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE_OK')" 2>&1 | tail -2
bash tools/gpu_scale.sh
