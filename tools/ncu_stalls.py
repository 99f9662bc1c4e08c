"""Stall-reason breakdown for given source lines of an ncu report."""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
lines = set(int(x) for x in sys.argv[2:])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr = None
cur = None
agg = defaultdict(lambda: defaultdict(int))
tot = defaultdict(int)
fname = ""
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1]
        continue
    if not fname.endswith("drivegrid_b200.cu"):
        continue
    if r and r[0] == "Line No":
        hdr = r
        cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0]:
        cur = int(r[0])
        continue
    for i in cols:
        try:
            v = int(r[i])
        except ValueError:
            continue
        tot[hdr[i]] += v
        if cur in lines:
            agg[cur][hdr[i]] += v
print("all lines:", sorted(((k, v) for k, v in tot.items() if v), key=lambda kv: -kv[1])[:12])
for ln, d in agg.items():
    print(ln, sorted(((k, v) for k, v in d.items() if v), key=lambda kv: -kv[1])[:8])
