"""Key metrics of every kernel in an ncu report as a markdown table row set."""
import csv
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, units = rows[0], rows[1]
names = [r[h.index("Kernel Name")].split("(")[0].split("::")[-1] for r in rows[2:]]
print("| metric | " + " | ".join(names) + " |")
print("|---|" + "---|" * len(names))
for w in WANT:
    if w in h:
        i = h.index(w)
        print(f"| {w} ({units[i]}) | " + " | ".join(r[i] for r in rows[2:]) + " |")
