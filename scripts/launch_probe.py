"""Launch / event overhead under a saturated H2D link (tools only).

For a tiny kernel (x.add_(1) on 16 floats): (a) one event pair per launch, (b) one event pair
around 200 back-to-back launches, (c) like (a) with only every 10th launch bracketed —
each with and without a background 1 GiB pinned H2D copy loop on another stream."""
import json
import threading
import time

import torch


def measure(n=200):
    s = torch.cuda.Stream()
    x = torch.zeros(16, device="cuda")
    out = {}
    with torch.cuda.stream(s):
        for _ in range(20):
            x.add_(1)
        torch.cuda.synchronize()
        torch.cuda._sleep(20_000_000)   # ~10 ms: the host enqueues everything below before the GPU reaches it
        evs = []
        for _ in range(n):
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(s); x.add_(1); b.record(s)
            evs.append((a, b))
        torch.cuda.synchronize()
        out["per_launch_pair_us"] = sum(a.elapsed_time(b) for a, b in evs) / n * 1e3
        torch.cuda._sleep(20_000_000)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(n):
            x.add_(1)
        b.record(s)
        torch.cuda.synchronize()
        out["batched_us_per_launch"] = a.elapsed_time(b) / n * 1e3
        torch.cuda._sleep(20_000_000)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(n):
            c = torch.cuda.Event(enable_timing=True); c.record(s)
            x.add_(1)
        b.record(s)
        torch.cuda.synchronize()
        out["batched_with_1_event_each_us"] = a.elapsed_time(b) / n * 1e3
        torch.cuda._sleep(20_000_000)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(n):
            c = torch.cuda.Event(enable_timing=False); c.record(s)
            x.add_(1)
        b.record(s)
        torch.cuda.synchronize()
        out["batched_with_1_nontiming_event_each_us"] = a.elapsed_time(b) / n * 1e3
    return out


def main():
    res = {"idle": measure()}
    hsrc = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
    hdst = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
    cs = torch.cuda.Stream()
    with torch.cuda.stream(cs):
        for _ in range(40):
            hdst.copy_(hsrc, non_blocking=True)
    time.sleep(0.05)
    res["h2d_load"] = measure()
    torch.cuda.synchronize()
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
