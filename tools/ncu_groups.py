"""Median k_profile duration per DRAM-read size from an ncu --csv launch list."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hdr]
mi, vi, idi = h.index('Metric Name'), h.index('Metric Value'), h.index('ID')
by = collections.OrderedDict()
for r in rows[hdr + 1:]:
    if len(r) > vi:
        by.setdefault(r[idi], {})[r[mi]] = float(r[vi].replace(',', ''))
groups = collections.OrderedDict()
for v in by.values():
    groups.setdefault(round(v.get('dram__bytes_read.sum', 0) / 1e6), []).append(v['gpu__time_duration.sum'])
for b, t in groups.items():
    t = sorted(t)
    med = t[len(t) // 2]
    print(f"read~{b:6d} MB  n={len(t):3d} median {med / 1e3:8.2f} us -> {b * 1e6 / (med * 1e-9) / 1e9:8.1f} GB/s")
