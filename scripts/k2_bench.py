"""Microbenchmark of the split-expert kernel (K2) and the per-layer GPU critical path.

Fully resident layers (theta = 1, every expert cached, no PCIe): one layer_forward = K1 + one K2
launch over every activated expert's rows + K3.  Reports K2 achieved HBM GB/s (event-timed on
the launching stream, algorithmic bytes = rows x 6d + activations) per BJ shape and batch.

    python scripts/k2_bench.py [--steps 50]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2509_08342_b200 import api  # noqa: E402


def run(shape, B, steps, L=2, theta=1.0, pcie_load=False, profile=True, weights="bf16"):
    S = synth.SHAPES[shape]
    desc = api.model_desc(L, S.N, S.K, S.d, S.I, n_shared=S.n_shared, row_granule=64, max_batch=B,
                          renorm_topk=S.renorm, L_host=1, v_e_max=L * S.N,
                          weight_format=api.M.Q4G64 if weights == "q4" else api.M.BF16)
    ctx = api.MoEpic(desc)
    for i in range(L):
        ctx.load_router(i, synth.bf16_bits(synth.router_weights(0, i, S.N, S.d)))
    for e in range(S.N):
        g, u, dn = synth.expert_weights(0, 0, e, S.d, S.I, device="cuda")
        ctx.load_expert(0, e, *(synth.bf16_bits(x) for x in (g, u, dn)))
    for i in range(L):
        for s in range(S.n_shared):
            g, u, dn = synth.shared_expert_weights(0, i, s, S.d, S.I, device="cuda")
            ctx.load_expert(i, -1 - s, *(synth.bf16_bits(x) for x in (g, u, dn)))
    ctx.configure(v_e=L * S.N * theta, theta_i=[theta] * L, prefetch=False)
    H = synth.hidden_states(3, steps + 5, L, S.d, scale=1.0).to("cuda")
    Hb = synth.batch_hidden(4, B * (steps + 5), S.d).to("cuda").view(steps + 5, B, S.d)
    y = torch.empty(B, S.d, dtype=torch.float32, device="cuda")
    st = torch.cuda.Stream()
    hsel = (lambda t, i: H[t, i][None]) if B == 1 else (lambda t, i: Hb[t])
    for t in range(5):
        for i in range(L):
            ctx.layer_forward(i, hsel(t, i), y, stream=st, trace=False)
    torch.cuda.synchronize()
    ctx.profile(profile)   # (resets with a device sync: start the background load after it)
    if pcie_load:   # saturate the H2D link with a background copy loop on another stream
        hsrc = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
        hdst = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
        bg = torch.cuda.Stream()
        with torch.cuda.stream(bg):
            for _ in range(4 + steps // 4):
                hdst.copy_(hsrc, non_blocking=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for t in range(5, steps + 5):
        for i in range(L):
            ctx.layer_forward(i, hsel(t, i), y, stream=st, trace=False)
    e1.record(st)
    torch.cuda.synchronize()
    k2 = ctx.profile_read(api.M.KERNEL_EXPERT)
    k1 = ctx.profile_read(api.M.KERNEL_ROUTER)
    k3 = ctx.profile_read(api.M.KERNEL_COMBINE)
    ms = e0.elapsed_time(e1)
    n = steps * L
    out = dict(shape=shape, B=B, pcie_load=pcie_load, layer_us=round(ms * 1e3 / n, 2),
               k2_us=round(k2["total_ms"] * 1e3 / max(1, k2["launches"]), 2),
               k2_launches_per_layer=k2["launches"] / n,
               k2_MB=round(k2["bytes"] / max(1, k2["launches"]) / 1e6, 2),
               k2_GBps=round(k2["bytes"] / max(k2["total_ms"] * 1e-3, 1e-12) / 1e9, 1),
               k2_kernel_us=round(k2["kernel_ms"] * 1e3 / max(1, k2["launches"]), 2),
               k1_us=round(k1["total_ms"] * 1e3 / max(1, k1["launches"]), 2),
               k1_kernel_us=round(k1["kernel_ms"] * 1e3 / max(1, k1["launches"]), 2),
               k3_us=round(k3["total_ms"] * 1e3 / max(1, k3["launches"]), 2),
               layer_GBps=round(k2["bytes"] / n / (ms * 1e-3 / n) / 1e9, 1))
    ctx.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--cases", default="mixtral:1,qwen3:1,qwen3:4,qwen3:16,deepseek:1")
    ap.add_argument("--pcie-load", action="store_true")
    ap.add_argument("--no-profile", action="store_true", help="no per-kernel events (layer_us only)")
    ap.add_argument("--weights", default="bf16", choices=["bf16", "q4"])
    args = ap.parse_args()
    for c in args.cases.split(","):
        shape, B = c.split(":")
        print(json.dumps(run(shape, int(B), args.steps, pcie_load=args.pcie_load, profile=not args.no_profile,
                             weights=args.weights)), flush=True)


if __name__ == "__main__":
    main()
