"""Per-phase cycle breakdown of the fused step (debug build with -DDG_PHASE_TIMERS)."""
import ctypes as ct
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

from paper_2605_08528_b200 import _native as N  # noqa: E402

dbg = ROOT / "paper_2605_08528_b200" / "libdrivegrid_b200_timers.so"
subprocess.run(["/usr/local/cuda/bin/nvcc", *N.NVCC_FLAGS, "-DDG_PHASE_TIMERS", "-I", str(ROOT / "include"),
                "-o", str(dbg), *map(str, N.SOURCES)], check=True)
N.LIB_PATH = dbg
import torch  # noqa: E402

from paper_2605_08528_b200 import config as C  # noqa: E402
from paper_2605_08528_b200.engine import Engine  # noqa: E402

lib = N.load_library(build_if_missing=False)
lib.dg_debug_phase_clocks.argtypes = [ct.c_void_p, ct.c_int]
W = int(sys.argv[1]) if len(sys.argv) > 1 else 256
nw = int(sys.argv[2]) if len(sys.argv) > 2 else 8
cfg = C.RootConfig()
cfg.env.num_envs = W
eng = Engine(**C.build_inputs(cfg).as_kwargs(), device=torch.device("cuda:0"), warps_per_world=nw)
acts = torch.zeros((W, 16, 3), dtype=torch.float64, device="cuda:0")
bufs = eng.new_step_buffers()
obs = eng.observe_device()
for i in range(5):
    eng.lane_follower(bufs.obs if i else obs, out=acts)
    eng.launch_step(acts, bufs, autoreset=True)
torch.cuda.synchronize()
out = np.zeros((W, 40), dtype=np.int64)
assert lib.dg_debug_phase_clocks(out.ctypes.data, W) == 0
names = ["act-check", "phys+zero(w0)", "bar1", "geo-fixup", "phase2a/2b", "bar3", "finalize"]
d = np.diff(out[:, :7], axis=1)
print(f"W={W} warps={nw}: median cycles per phase (per CTA)")
for i, nme in enumerate(names[:6]):
    print(f"  {nme:14s} median {np.median(d[:, i]):8.0f}  p90 {np.percentile(d[:, i], 90):8.0f}")
tot = out[:, 6] - out[:, 0]
print(f"  total          median {np.median(tot):8.0f}  max {tot.max():8.0f}")
wend = out[:, 8:8 + nw] - out[:, 4:5]
ph = out[:, [1, 25, 26, 27, 2]]
print("  warp0: loads", np.median(ph[:, 1] - ph[:, 0]), " substeps", np.median(ph[:, 2] - ph[:, 1]),
      " derived+tables", np.median(ph[:, 3] - ph[:, 2]), " zero-fill", np.median(ph[:, 4] - ph[:, 3]))
print("  substep ends (cycles after state loads):", np.median(out[:, 28:32] - out[:, 25:26], axis=0).astype(int))
w1 = out[:, [4, 34]]
print("  warp1: pairs (phase 2a)", np.median(w1[:, 1] - w1[:, 0]))
gs, ge = out[:, 32], out[:, 33]
t0 = gs.min()
print(f"  globaltimer: CTA start spread {(gs.max() - t0) / 1e3:.2f} us, first end {(ge.min() - t0) / 1e3:.2f} us, "
      f"last end {(ge.max() - t0) / 1e3:.2f} us, median CTA duration {np.median(ge - gs) / 1e3:.2f} us")
print("  phase2 per-warp end (cycles after phase2 start), median over CTAs:", np.median(wend, axis=0).astype(int))
