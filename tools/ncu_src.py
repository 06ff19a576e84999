"""Summarise an ncu source page (SASS, stall sampling): hottest lines and
totals per stall reason.  python tools/ncu_src.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) > 5 and r[0].startswith("0x")]
si = hdr.index("Warp Stall Sampling (All Samples)")
ii = hdr.index("Instructions Executed")
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = {hdr[i]: sum(int(r[i]) for r in data if r[i].isdigit()) for i in cols}
print("samples", sum(int(r[si]) for r in data if r[si].isdigit()), "instr", len(data),
      "warp-instr executed", sum(int(r[ii]) for r in data if r[ii].isdigit()))
print(sorted([(v, k) for k, v in tot.items() if v], reverse=True))
acc = 0
for r in data:
    s = int(r[si]) if r[si].isdigit() else 0
    acc += s
    r.append(acc)
for r in sorted(data, key=lambda r: -(int(r[si]) if r[si].isdigit() else 0))[:top]:
    why = {hdr[i][6:]: r[i] for i in cols if r[i] not in ("0", "", "-")}
    print(r[0][-5:], r[ii].rjust(6), r[si].rjust(5), str(r[-1]).rjust(6), r[1][:60], why)
