"""Per-source-line stall samples of one kernel in an ncu report, mapping
SASS offsets to lines with nvdisasm -g on the object that ran.
python tools/ncu_lines.py report.ncu-rep obj.o kernel_substring [N]"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, obj, kname = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) > 5 and r[0].startswith("0x")]
si = hdr.index("Warp Stall Sampling (All Samples)")
ii = hdr.index("Instructions Executed")
base = int(data[0][0], 16)
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cubin = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
sass = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cubin)], capture_output=True, text=True).stdout
# several instantiations may match the name: take the one whose instruction
# count equals the profiled kernel's (else the first match)
cands = []
for sec in re.split(r"\n\s*\.section\s+", sass):
    h = sec.split("\n")[0]
    if not sec.startswith(".text.") or kname not in h:
        continue
    lo, cur = {}, None
    for ln in sec.split("\n"):
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        mm = re.match(r"\s+/\*([0-9a-f]+)\*/", ln)
        if mm:
            lo[int(mm.group(1), 16)] = cur
    cands.append((h, lo))
pick = [c for c in cands if len(c[1]) == len(data)] or cands
print("section", pick[0][0][:100], "of", len(cands))
line_of = pick[0][1]
agg = collections.Counter()
ex = collections.Counter()
for r in data:
    off = int(r[0], 16) - base
    k = line_of.get(off, ("?", 0))
    agg[k] += int(r[si]) if r[si].isdigit() else 0
    ex[k] += int(r[ii]) if r[ii].isdigit() else 0
tot = sum(agg.values())
print("samples", tot)
for k, v in agg.most_common(top):
    print(f"{v:6d} {100 * v / tot:5.1f}%  exec {ex[k]:6d}  {k[0]}:{k[1]}")
