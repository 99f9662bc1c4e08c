"""Policy-forward variants built from compile-time switches (argv: name=FLAGS,
e.g. base= elu2=-DDG_EXP_ELU2), each its own .so, timed by tools/policy_time.py."""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2605_08528_b200 import _native as N  # noqa: E402

for arg in sys.argv[1:]:
    name, flags = arg.split("=", 1)
    lib = Path(f"/tmp/libdg_{name}.so")
    subprocess.run(["/usr/local/cuda/bin/nvcc", *N.NVCC_FLAGS, *flags.split(), "-I", str(ROOT / "include"),
                    "-o", str(lib), *map(str, N.SOURCES)], check=True, capture_output=True)
    env = dict(os.environ, DG_LIB_PATH=str(lib))
    out = subprocess.run([sys.executable, str(ROOT / "tools" / "policy_time.py")], env=env, capture_output=True,
                         text=True)
    print(f"== {name} ({flags})\n{out.stdout}{out.stderr[-500:] if out.returncode else ''}", flush=True)
