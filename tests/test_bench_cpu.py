"""CPU checks of bench.py's host side: the reference (oracle) arm of every
config prints one JSON line with the contract's keys, and the GPU arm's
`config` object is the same function of the workload (same_config)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("cfg", [3, 4, 5])
def test_reference_arm_json(cfg):
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", str(cfg), "--steps", "1",
                        "--warmup", "0", "--ref-budget", "3"], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["cpu_baseline"]["kind"] == "oracle" and d["value"] > 0
    sys.path.insert(0, ROOT)
    import bench
    assert d["config"] == json.loads(json.dumps(bench.WORKLOADS[cfg]().config(1)))


def test_cfg2_weights_topk_is_the_mask():
    """synth.cfg2_topk_weights_bf16: the oracle's global top-k (Alg. 1,
    P:L455-480) of the weights with k = the masks' kept count is exactly the
    masks (small shape, every tensor of every layer in one global pool)."""
    shape = synth.GPTShape(L=6, h=48)
    p = synth.cfg2_keep_probs(shape, 0.9, 4)
    masks, w = [], []
    for layer in range(shape.L):
        for t, m in enumerate(synth.cfg2_layer_masks_u8(shape, layer, p[layer], 4)):
            masks.append(m.reshape(-1))
            w.append(oracle.bf16_to_f64(synth.cfg2_topk_weights_bf16(m, layer, t).reshape(-1)))
    k = int(sum(int(m.sum()) for m in masks))
    st, got = oracle.global_prune(w, k)
    assert st == 0 and 0 < k < sum(m.size for m in masks)
    for a, b in zip(got, masks):
        assert np.array_equal(a, b)
