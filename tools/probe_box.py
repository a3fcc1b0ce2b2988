import os, subprocess, time, json, torch
out = {}
out["cpu_count"] = os.cpu_count()
out["meminfo"] = open("/proc/meminfo").read().split("\n")[:4]
out["shm"] = subprocess.run(["df","-h","/dev/shm"],capture_output=True,text=True).stdout
out["nvsmi"] = subprocess.run(["nvidia-smi","--query-gpu=name,memory.total,clocks.max.sm,pcie.link.gen.max,pcie.link.width.max","--format=csv"],capture_output=True,text=True).stdout
out["numa"] = subprocess.run(["bash","-c","ls /sys/devices/system/node | grep node; nproc"],capture_output=True,text=True).stdout
dev = torch.device("cuda:0")
for gib in [1, 4]:
    n = gib << 30
    t0 = time.time()
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    out[f"pin_alloc_{gib}GiB_s"] = time.time() - t0
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream()
    best = 0
    for i in range(6):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s); d.copy_(h, non_blocking=True); e1.record(s)
        e1.synchronize()
        best = max(best, n / (e0.elapsed_time(e1) / 1e3) / 1e9)
    out[f"h2d_{gib}GiB_GBs"] = best
    best = 0
    for i in range(4):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s); h.copy_(d, non_blocking=True); e1.record(s)
        e1.synchronize()
        best = max(best, n / (e0.elapsed_time(e1) / 1e3) / 1e9)
    out[f"d2h_{gib}GiB_GBs"] = best
    del h, d
# big pinned alloc timing (32 GiB) to gauge 90 GB feasibility
try:
    t0 = time.time(); h = torch.empty(32 << 30, dtype=torch.uint8, pin_memory=True); out["pin_alloc_32GiB_s"] = time.time() - t0; del h
except Exception as e:
    out["pin_alloc_32GiB_err"] = str(e)
print(json.dumps(out, indent=1))
json.dump(out, open("gpurun_out/probe.json","w"), indent=1)
