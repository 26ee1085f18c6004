"""Attention stand-in timing vs KV length (tools): GPU time per call with the stream held while
the host enqueues, and the achieved cache bandwidth."""
import json
import sys
import os
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2509_08342_b200 import api

B, Hq, Hkv = 1, 32, 8
for S in (256, 1024, 4096, 16384, 65536):
    g = torch.Generator(device="cuda").manual_seed(0)
    k = torch.randn(B, S, Hkv, 128, generator=g, device="cuda").to(torch.bfloat16)
    v = torch.randn(B, S, Hkv, 128, generator=g, device="cuda").to(torch.bfloat16)
    q = torch.randn(B, Hq, 128, generator=g, device="cuda").to(torch.bfloat16)
    o = torch.empty(B, Hq, 128, device="cuda")
    att = api.Attention(B, S, Hq, Hkv)
    s = torch.cuda.Stream()
    for _ in range(3):
        att(q, k, v, S, o, stream=s)
    torch.cuda.synchronize()
    n = 50
    with torch.cuda.stream(s):
        torch.cuda._sleep(100_000_000)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(n):
        att(q, k, v, S, o, stream=s)
    b.record(s)
    torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / n
    print(json.dumps({"S": S, "us": round(us, 2), "GBps": round(2 * S * Hkv * 128 * 2 / (us * 1e-6) / 1e9, 1)}), flush=True)
