"""Instruction / stall share by kernel region (source-line ranges given as name=a-b)."""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
regions = []
for spec in sys.argv[2:]:
    name, rng = spec.split("=")
    a, b = rng.split("-")
    regions.append((name, int(a), int(b)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr, cur = None, None
ins, smp = defaultdict(int), defaultdict(int)
fname = ""
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1]
        continue
    if not fname.endswith("drivegrid_b200.cu"):
        continue
    if r and r[0] == "Line No":
        hdr = r
        ii, si = r.index("Instructions Executed"), r.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0]:
        cur = int(r[0])
        continue
    try:
        ins[cur] += int(r[ii])
        smp[cur] += int(r[si])
    except ValueError:
        pass
TI, TS = sum(ins.values()), sum(smp.values())
print(f"total inst {TI}  samples {TS}")
for name, a, b in regions:
    i = sum(v for k, v in ins.items() if a <= k <= b)
    s = sum(v for k, v in smp.items() if a <= k <= b)
    print(f"{name:14s} inst {100*i/TI:5.1f}%  samples {100*s/TS:5.1f}%")
