"""Summaries of gpurun outputs: bench JSON line and ncu launch lists."""
import collections
import signal
import csv
import json
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            agg[r[ki][:60]].append(float(r[vi].replace(",", "")))
    for k, v in agg.items():
        print(f"{len(v):5d} {sum(v) / len(v) / 1e3:10.2f} us  {k}")


def bench(path):
    d = json.loads(open(path).read().strip().splitlines()[-1])
    keys = ["value", "n_gpus", "gpu_launches"]
    print({k: d.get(k) for k in keys})
    for k in ["roofline", "phases_ms_per_step", "step_ms", "migrate", "solution", "e2e", "clocks", "cpu_baseline"]:
        if k in d:
            print(" ", k, d[k])


if __name__ == "__main__":
    signal.signal(signal.SIGPIPE, signal.SIG_DFL)  # quiet under | head
    for p in sys.argv[1:]:
        print("==", p)
        (launches if p.endswith(".csv") else bench)(p)
