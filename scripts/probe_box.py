"""Probe the GPU box: host RAM, memlock, CPU, PCIe topology and pinned H2D/D2H bandwidth."""
import os, subprocess, time, json
import torch

out = {}
def sh(c):
    try:
        return subprocess.run(c, shell=True, capture_output=True, text=True, timeout=60).stdout
    except Exception as e:
        return str(e)
out["free"] = sh("free -g")
out["ulimit_l"] = sh("ulimit -l")
out["nproc"] = os.cpu_count()
out["cpu"] = sh("grep -m1 'model name' /proc/cpuinfo")
out["numa"] = sh("lscpu | grep -i numa")
out["topo"] = sh("nvidia-smi topo -m")
out["smi"] = sh("nvidia-smi --query-gpu=name,pcie.link.gen.current,pcie.link.gen.max,pcie.link.width.current,memory.total,clocks.max.sm --format=csv")
dev = torch.device("cuda:0")
res = {}
for size_mb in [64, 256, 1024]:
    n = size_mb << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h.fill_(1)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream()
    best_h2d = best_d2h = 0
    for it in range(10):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s); d.copy_(h, non_blocking=True); e1.record(s)
        e1.synchronize()
        best_h2d = max(best_h2d, n / (e0.elapsed_time(e1) * 1e-3) / 1e9)
        with torch.cuda.stream(s):
            e0.record(s); h.copy_(d, non_blocking=True); e1.record(s)
        e1.synchronize()
        best_d2h = max(best_d2h, n / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    res[size_mb] = (round(best_h2d, 2), round(best_d2h, 2))
out["pinned_bw_GBps_h2d_d2h"] = res
# large pinned allocation test
t0 = time.time()
sizes = {}
for gb in [8, 32, 64]:
    try:
        t0 = time.time()
        x = torch.empty(gb << 30, dtype=torch.uint8, pin_memory=True)
        sizes[gb] = round(time.time() - t0, 2)
        del x
    except Exception as e:
        sizes[gb] = "fail: " + str(e)[:100]
        break
out["pin_alloc_seconds"] = sizes
print(json.dumps(out, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe.json", "w"), indent=1)
