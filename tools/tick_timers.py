"""Per-tick phase cycle sums of the persistent fused step (debug build with
-DDG_TICK_TIMERS): bench-shaped 256 x 16 LaneFollower + autoreset launches of
T ticks, every launch shape given on the command line (e.g. 8:0 8:2)."""
import ctypes as ct
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

from paper_2605_08528_b200 import _native as N  # noqa: E402

dbg = ROOT / "paper_2605_08528_b200" / "libdrivegrid_b200_ticktimers.so"
import os  # noqa: E402
extra = os.environ.get("DG_EXTRA_FLAGS", "").split()
subprocess.run(["/usr/local/cuda/bin/nvcc", *N.NVCC_FLAGS, "-DDG_TICK_TIMERS", *extra, "-I", str(ROOT / "include"),
                "-o", str(dbg), *map(str, N.SOURCES)], check=True)
N.LIB_PATH = dbg
import torch  # noqa: E402

from paper_2605_08528_b200 import config as C  # noqa: E402
from paper_2605_08528_b200.engine import Engine  # noqa: E402

lib = N.load_library(build_if_missing=False)
lib.dg_debug_tick_clocks.argtypes = [ct.c_void_p, ct.c_int, ct.c_int]
W = int(sys.argv[1]) if len(sys.argv) > 1 else 256
T = int(sys.argv[2]) if len(sys.argv) > 2 else 64
shapes = sys.argv[3:] or ["8:0", "7:2"]
cfg = C.RootConfig()
cfg.env.num_envs = W
inp = C.build_inputs(cfg)
dev = torch.device("cuda:0")
for sh in shapes:
    nw, mode = (int(v) for v in sh.split(":"))
    eng = Engine(**inp.as_kwargs(), device=dev, warps_per_world=nw, launch_mode=mode)
    rb = eng.new_rollout_buffers(T)
    acts = torch.zeros((W, 16, 3), dtype=torch.float64, device=dev)
    eng.observe(out=rb.obs[T - 1], as_numpy=False, next_actions=acts)
    eng.launch_step(acts, rb, autoreset=True, next_actions=acts, ticks=T)
    torch.cuda.synchronize()
    assert lib.dg_debug_tick_clocks(None, W, 1) == 0
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    eng.launch_step(acts, rb, autoreset=True, next_actions=acts, ticks=T)
    s1.record()
    torch.cuda.synchronize()
    out = np.zeros((W, 48), dtype=np.int64)
    assert lib.dg_debug_tick_clocks(out.ctypes.data, W, 0) == 0
    per = out / T
    names = ["check", "phase1", "phase2+bar", "tail-rest", "end-bar"]
    print(f"[{' '.join(extra)}] W={W} T={T} warps={nw} mode={mode} ({eng.launch_shape()}): {s0.elapsed_time(s1) / T * 1e3:.2f} us/tick "
          f"(timer build)")
    for i, nme in enumerate(names):
        print(f"  {nme:12s} median {np.median(per[:, i]):8.0f}  p90 {np.percentile(per[:, i], 90):8.0f}")
    print(f"  sum          median {np.median(per[:, :8].sum(1)):8.0f}")
    print(f"  tail split: to-finalize {np.median(per[:, 5]):.0f}  finalize {np.median(per[:, 6]):.0f}  "
          f"count_events {np.median(per[:, 7]):.0f}  rest {np.median(per[:, 3]):.0f}")
    print("  pairs (2a) per warp (median over CTAs):", np.median(per[:, 20:20 + nw], axis=0).astype(int))
    print("  scans (2b) per warp (median over CTAs):", np.median(per[:, 8:8 + nw], axis=0).astype(int))
    sub = per[:, 32:41]
    if sub.any():
        print("  2a sub-phases per 2a warp slot (key+rank | ttc+rows+contact | reduce+store):",
              np.median(sub[:, 0:3], axis=0).astype(int), np.median(sub[:, 3:6], axis=0).astype(int),
              np.median(sub[:, 6:9], axis=0).astype(int))
    if mode == 2:
        print(f"  physics warp: zero-issue {np.median(per[:, 29]):.0f}  ego {np.median(per[:, 30]):.0f}  "
              f"physics {np.median(per[:, 31]):.0f}")
