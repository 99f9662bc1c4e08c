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
    subprocess.run(["/usr/local/cuda/bin/nvcc", *N.NVCC_FLAGS, *flags.split(), "-I", str(ROOT / "include"),
                    "-o", f"/tmp/libdg_{name}.so", *map(str, N.SOURCES)], check=True, capture_output=True)
for rnd in range(2):
    for name, flags in variants:
        env = dict(os.environ, DG_LIB_PATH=f"/tmp/libdg_{name}.so", SWEEP_COUNT="1")
        out = subprocess.run([sys.executable, str(ROOT / "tools" / "variant_sweep.py"), f"V={name}"], env=env,
                             capture_output=True, text=True)
        print(out.stdout.strip() or out.stderr[-800:], flush=True)
