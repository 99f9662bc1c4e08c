"""Where the reference-facing numpy step's time goes (256 x 16, default pool,
LaneFollower + autoreset): the body of Engine._step_host replayed with host
timers around each call and CUDA events between the device stages.

  python tools/e2e_breakdown.py [steps]   -> one JSON object (profiles/)
"""
import ctypes as ct
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_08528_b200 import _native as N  # noqa: E402
from paper_2605_08528_b200 import config as C  # noqa: E402
from paper_2605_08528_b200.engine import Engine, _ptr  # noqa: E402
from paper_2605_08528_b200.policies import LaneFollower  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
dev = torch.device("cuda:0")
eng = Engine(**C.build_inputs(C.RootConfig()).as_kwargs(), device=dev)
pol = LaneFollower(obs_config=eng.obs_config)
lib = eng._lib
stream = torch.cuda.current_stream(dev)
obs = eng.observe()
for _ in range(5):
    obs = eng.step(pol(obs), autoreset=True).obs
torch.cuda.synchronize()

host = {k: 0.0 for k in ("policy", "validate+pin", "launch_h2d", "launch_step", "launch_to_host", "sync_wait",
                         "views")}
devt = {k: 0.0 for k in ("h2d", "step_kernel", "obs_to_host", "aux_d2h")}
ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
bytes0 = int(eng.d2h_bytes.item())
t_all = time.perf_counter()
out_keep = None
for _ in range(steps):
    t0 = time.perf_counter()
    a = pol(obs)
    t1 = time.perf_counter()
    a = np.asarray(a, dtype=np.float64)
    assert np.isfinite(a).all()
    eng._act_host.numpy()[...] = a
    t2 = time.perf_counter()
    ev[0].record(stream)
    eng._act_dev.copy_(eng._act_host, non_blocking=True)
    ev[1].record(stream)
    t3 = time.perf_counter()
    key = (True, eng._metrics_on)
    io = eng._host_io.get(key) or eng._host_io.setdefault(key, eng._step_io(eng._act_dev, eng._host_bufs,
                                                                              autoreset=True,
                                                                              prefix_out=eng._prefix_dev))
    N.check(lib, lib.dg_step(eng._h, ct.byref(io), ct.c_void_p(stream.cuda_stream)), "dg_step")
    ev[2].record(stream)
    t4 = time.perf_counter()
    ptr, prev, hb = eng._mapped_pool.acquire()
    ob = eng._host_obs_bytes
    N.check(lib, lib.dg_to_host(eng._h, _ptr(eng._obs_dev), _ptr(eng._prefix_dev), ct.c_void_p(ptr), _ptr(prev),
                                _ptr(eng._host_bufs.aux),
                                ct.c_void_p(ptr + ob), eng._host_blob.numel() - ob, _ptr(eng.d2h_bytes),
                                ct.c_void_p(stream.cuda_stream)), "dg_to_host")
    ev[4].record(stream)
    t5 = time.perf_counter()
    stream.synchronize()
    t6 = time.perf_counter()
    obs = hb[:ob].view(np.float32)[:eng.W * eng.M * eng.obs_config.obs_dim].reshape(eng.W, eng.M, -1)
    hv = eng._host_views(hb[ob:])
    dones = hv["dones"].astype(bool)
    t7 = time.perf_counter()
    for k, (x, y) in zip(host, ((t0, t1), (t1, t2), (t2, t3), (t3, t4), (t4, t5), (t5, t6), (t6, t7))):
        host[k] += y - x
    devt["h2d"] += ev[0].elapsed_time(ev[1]) / 1e3
    devt["step_kernel"] += ev[1].elapsed_time(ev[2]) / 1e3
    devt["obs_to_host"] += ev[2].elapsed_time(ev[4]) / 1e3
wall = time.perf_counter() - t_all
obs_bytes = (int(eng.d2h_bytes.item()) - bytes0) / steps
res = {"workload": "256x16 default pool, LaneFollower (numpy) + autoreset, Engine.step(numpy) body",
       "steps": steps, "ms_per_step": 1e3 * wall / steps,
       "host_ms": {k: round(1e3 * v / steps, 4) for k, v in host.items()},
       "device_ms": {k: round(1e3 * v / steps, 4) for k, v in devt.items()},
       "obs_bytes_per_step": obs_bytes, "aux_bytes_per_step": int(eng._host_blob.numel() - eng._host_obs_bytes),
       "obs_gbps": obs_bytes / (devt["obs_to_host"] / steps) / 1e9 if devt["obs_to_host"] else None}
print(json.dumps(res))
