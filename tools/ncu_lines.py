"""Per-source-line hot spots from an ncu report (instructions + stall samples)."""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr = None
agg = defaultdict(lambda: [0, 0, ""])
cur = None
fname = ""
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1]
        continue
    if not ((fname.endswith("drivegrid_b200.cu") or fname.endswith("dg_policy.cu") or fname.endswith("dg_umma.cuh")) or fname.endswith(sys.argv[-1] if sys.argv[-1].endswith(".cu") else "drivegrid_b200.cu")):
        continue
    if r and r[0] == "Line No":
        hdr = r
        i_samp = r.index("Warp Stall Sampling (All Samples)")
        i_inst = r.index("Instructions Executed")
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0]:
        cur = int(r[0])
        agg[cur][2] = r[1][:90]
        continue
    if cur is None:
        continue
    try:
        agg[cur][0] += int(r[i_inst])
        agg[cur][1] += int(r[i_samp])
    except ValueError:
        pass
tot_i = sum(v[0] for v in agg.values()) or 1
tot_s = sum(v[1] for v in agg.values()) or 1
print(f"total warp-instructions {tot_i}, stall samples {tot_s}")
key = 0 if (len(sys.argv) > 3 and sys.argv[3] == "inst") else 1
for line, (ins, samp, src) in sorted(agg.items(), key=lambda kv: -kv[1][key])[:top]:
    print(f"{line:5d} inst {100*ins/tot_i:5.1f}%  samples {100*samp/tot_s:5.1f}%  {src}")
