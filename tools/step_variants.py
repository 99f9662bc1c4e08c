"""A/B of step-kernel compile-time variants in ONE process tree on one box
(argv: name=FLAGS, e.g. base= f32=-DDG_EXP_F32RANK): each variant is built
into its own .so and timed by tools/variant_sweep.py (bench workload, device
time per tick), interleaved twice to expose drift."""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2605_08528_b200 import _native as N  # noqa: E402

variants = [a.split("=", 1) for a in sys.argv[1:]]
for name, flags in variants:
    # "--src=PATH" swaps the step-kernel source (e.g. a committed revision, git show REV:path > PATH)
    srcs = [str(x) for x in N.SOURCES]
    fl = []
    for f in flags.split():
        if f.startswith("--src="):
            srcs[0] = f[len("--src="):]
        else:
            fl.append(f)
    subprocess.run(["/usr/local/cuda/bin/nvcc", *N.NVCC_FLAGS, *fl, "-I", str(ROOT / "include"),
                    "-I", str(ROOT / "paper_2605_08528_b200" / "csrc"), "-o", f"/tmp/libdg_{name}.so", *srcs],
                   check=True, capture_output=True)
for rnd in range(2):
    for name, flags in variants:
        env = dict(os.environ, DG_LIB_PATH=f"/tmp/libdg_{name}.so", SWEEP_COUNT="1")
        out = subprocess.run([sys.executable, str(ROOT / "tools" / "variant_sweep.py"), f"V={name}"], env=env,
                             capture_output=True, text=True)
        print(out.stdout.strip() or out.stderr[-800:], flush=True)
