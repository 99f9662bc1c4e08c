import torch, time
src=torch.empty(32325632//4, dtype=torch.float32, device="cuda")
for n in (1,2,4):
    dst=torch.empty(src.shape, dtype=torch.float32, pin_memory=True)
    streams=[torch.cuda.Stream() for _ in range(n)]
    ch=src.numel()//n
    for rep in range(3):
        torch.cuda.synchronize(); t=time.perf_counter()
        for i,s in enumerate(streams):
            with torch.cuda.stream(s):
                dst[i*ch:(i+1)*ch].copy_(src[i*ch:(i+1)*ch], non_blocking=True)
        torch.cuda.synchronize(); dt=time.perf_counter()-t
    print(n, "streams:", round(dt*1e3,3), "ms", round(src.numel()*4/dt/1e9,1), "GB/s")
