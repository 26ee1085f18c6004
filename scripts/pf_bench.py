"""Microbenchmark of the prefill tcgen05 GEMMs (A12) on a fully resident layer (theta = 1, every
expert cached, no PCIe): one layer_forward(T tokens) = K1 + permute + gate/up GEMM + down GEMM
+ combine.  Reports the GEMMs' achieved TFLOP/s (event-timed on the launching stream, algorithmic
FLOPs = 2 * 3 * d * I per routed (token, expert) pair) against the measured bf16 peak.

    python scripts/pf_bench.py [--shape mixtral] [--T 2048] [--steps 10] [--pair auto|0|1]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="mixtral")
    ap.add_argument("--T", type=int, default=2048)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--pair", default="auto", choices=["auto", "0", "1"])
    a = ap.parse_args()
    if a.pair != "auto":
        os.environ["MOEPIC_PF_CTA_PAIR"] = a.pair
    import torch
    import synth
    from paper_2509_08342_b200 import api
    S = synth.SHAPES[a.shape]
    desc = api.model_desc(1, S.N, S.K, S.d, S.I, n_shared=S.n_shared, row_granule=64, max_batch=a.T,
                          renorm_topk=S.renorm, L_host=1, v_e_max=S.N)
    ctx = api.MoEpic(desc)
    ctx.load_router(0, synth.bf16_bits(synth.router_weights(0, 0, S.N, S.d)))
    for e in range(S.N):
        g, u, dn = synth.expert_weights(0, 0, e, S.d, S.I, device="cuda")
        ctx.load_expert(0, e, *(synth.bf16_bits(x) for x in (g, u, dn)))
    for s in range(S.n_shared):
        g, u, dn = synth.shared_expert_weights(0, 0, s, S.d, S.I, device="cuda")
        ctx.load_expert(0, -1 - s, *(synth.bf16_bits(x) for x in (g, u, dn)))
    ctx.configure(v_e=float(S.N), theta_i=[1.0], prefetch=False)
    H = synth.batch_hidden(4, a.T * (a.steps + 3), S.d).to("cuda").view(a.steps + 3, a.T, S.d)
    y = torch.empty(a.T, S.d, dtype=torch.float32, device="cuda")
    st = torch.cuda.Stream()
    for t in range(3):
        ctx.layer_forward(0, H[t], y, stream=st, trace=False)
    torch.cuda.synchronize()
    ctx.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for t in range(3, a.steps + 3):
        ctx.layer_forward(0, H[t], y, stream=st, trace=False)
    e1.record(st)
    torch.cuda.synchronize()
    kg = ctx.profile_read(api.M.KERNEL_GEMM)
    ctx.profile(False)
    ms = e0.elapsed_time(e1) / a.steps
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    peak = float(peaks.get("bf16_tflops", 1590.0))
    tf = kg["bytes"] / (kg["total_ms"] * 1e-3) / 1e12
    print(json.dumps({"shape": a.shape, "T": a.T, "pair": a.pair, "layer_ms": round(ms, 3),
                      "gemm_ms_per_layer": round(kg["total_ms"] / a.steps, 3),
                      "gemm_launches_per_layer": kg["launches"] / a.steps, "gemm_tflops": round(tf, 1),
                      "peak_tflops": peak, "frac": round(tf / peak, 4),
                      "layer_tflops": round(kg["bytes"] / a.steps / (ms * 1e-3) / 1e12, 1)}))
    ctx.close()


if __name__ == "__main__":
    main()
