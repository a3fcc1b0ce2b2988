import torch, time, json
dev = torch.device("cuda", 0)
n = 1 << 30
res = {}
for nstreams in (1, 2, 3, 4):
    hs = [torch.empty(n // nstreams, dtype=torch.uint8).pin_memory() for _ in range(nstreams)]
    ds = [torch.empty(n // nstreams, dtype=torch.uint8, device=dev) for _ in range(nstreams)]
    sts = [torch.cuda.Stream() for _ in range(nstreams)]
    best = 0
    for rep in range(6):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in sts: s.wait_event(e0)
        for h, d, s in zip(hs, ds, sts):
            with torch.cuda.stream(s):
                d.copy_(h, non_blocking=True)
        for s in sts: torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, n / (e0.elapsed_time(e1) / 1e3) / 1e9)
    res[nstreams] = round(best, 2)
# chunked single stream: 64 MB chunks
h = torch.empty(n, dtype=torch.uint8).pin_memory(); d = torch.empty(n, dtype=torch.uint8, device=dev)
for chunk in (8 << 20, 64 << 20):
    best = 0
    for rep in range(4):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for o in range(0, n, chunk):
            d[o:o+chunk].copy_(h[o:o+chunk], non_blocking=True)
        e1.record(); torch.cuda.synchronize()
        best = max(best, n / (e0.elapsed_time(e1) / 1e3) / 1e9)
    res[f"chunk{chunk>>20}MB"] = round(best, 2)
print(json.dumps(res))
