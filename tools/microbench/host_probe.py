"""Host-side probe for the e2e path: CPU topology, host memory write
bandwidth (memset / copy into pinned and pageable buffers, 1..N threads),
and pinned D2H bandwidth for the 256x16 observation block."""
import os, time, json, threading, subprocess
import numpy as np
import torch

out = {}
out["cores"] = len(os.sched_getaffinity(0))
try:
    out["lscpu"] = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
except Exception as e:
    out["lscpu"] = str(e)
N = 256 * 16 * 1929 * 4
pinned = torch.empty(N, dtype=torch.uint8, pin_memory=True).numpy()
page = np.empty(N, dtype=np.uint8)
page[:] = 1
src = np.ones(N, dtype=np.uint8)

def bw(fn, reps=20):
    fn(); t = time.perf_counter()
    for _ in range(reps): fn()
    return N * reps / (time.perf_counter() - t) / 1e9

out["memset_pinned_1t"] = bw(lambda: pinned.fill(0))
out["memset_page_1t"] = bw(lambda: page.fill(0))
out["copy_pinned_1t"] = bw(lambda: np.copyto(pinned, src))
for nt in (2, 4, 8, 16):
    chunks = np.array_split(np.arange(N), nt)
    bounds = [(c[0], c[-1] + 1) for c in chunks]
    def par():
        ths = [threading.Thread(target=lambda a=a, b=b: pinned[a:b].fill(0)) for a, b in bounds]
        [t.start() for t in ths]; [t.join() for t in ths]
    out[f"memset_pinned_{nt}t"] = bw(par)
d = torch.empty(N, dtype=torch.uint8, device="cuda")
h = torch.empty(N, dtype=torch.uint8, pin_memory=True)
s = torch.cuda.current_stream()
for _ in range(3): h.copy_(d, non_blocking=True); s.synchronize()
t = time.perf_counter()
for _ in range(50): h.copy_(d, non_blocking=True); s.synchronize()
out["d2h_pinned_GBs"] = N * 50 / (time.perf_counter() - t) / 1e9
t = time.perf_counter()
for _ in range(50): d.copy_(h, non_blocking=True); s.synchronize()
out["h2d_pinned_GBs"] = N * 50 / (time.perf_counter() - t) / 1e9
t = time.perf_counter()
for _ in range(50): x = torch.empty(N, dtype=torch.uint8, pin_memory=True)
out["pinned_alloc_us"] = (time.perf_counter() - t) / 50 * 1e6
print(json.dumps({k: v for k, v in out.items() if k != "lscpu"}, indent=1))
print(out["lscpu"])
