"""H2D bandwidth of one vs several concurrent copy streams and of 8 MB chunks on one stream
(tools only): does splitting the transfer engine's copies raise the link rate?  SM loads from
mapped pinned memory are probed in scripts/pcie_zero_copy.py."""
import json
import torch

n = 1 << 30
h = torch.empty(n, dtype=torch.uint8).pin_memory()
h.fill_(1)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
res = {}
for ns in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(ns)]
    best = 0
    for rep in range(5):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record()
        for i, s in enumerate(ss):
            s.wait_event(a)
            with torch.cuda.stream(s):
                lo, hi = i * n // ns, (i + 1) * n // ns
                d[lo:hi].copy_(h[lo:hi], non_blocking=True)
        for s in ss:
            torch.cuda.current_stream().wait_stream(s)
        b.record()
        torch.cuda.synchronize()
        best = max(best, n / (a.elapsed_time(b) * 1e-3) / 1e9)
    res[f"streams_{ns}"] = round(best, 2)
# chunked on one stream (8 MB pieces) as the transfer engine issues them
s = torch.cuda.Stream()
best = 0
for rep in range(5):
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(s)
    with torch.cuda.stream(s):
        for off in range(0, n, 8 << 20):
            d[off:off + (8 << 20)].copy_(h[off:off + (8 << 20)], non_blocking=True)
    b.record(s)
    torch.cuda.synchronize()
    best = max(best, n / (a.elapsed_time(b) * 1e-3) / 1e9)
res["chunks_8MB_1stream"] = round(best, 2)
print(json.dumps(res))
