"""Where does the host-buffer (e2e) path lose time against the device path?  Runs a bench config
three ways for a few tokens: device buffers without per-layer sync (the bench's `value`), device
buffers with a stream sync after every layer, and moepic_layer_forward_host (the bench's e2e).

    python scripts/e2e_probe.py --config deepseek --tokens 4
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="deepseek")
    ap.add_argument("--tokens", type=int, default=4)
    ap.add_argument("--adapt", type=int, default=0, help="tokens of the Alg. 1 profiling phase (bench: 128)")
    a = ap.parse_args()
    import torch
    import synth
    import bench
    from paper_2509_08342_b200 import api
    cfg = bench.CONFIGS[a.config]
    ctx, desc, S, v_e, keep = bench.build_model(api, synth, torch, cfg, max_batch=cfg["B"], log=lambda *x: None)
    L, B = cfg["L"], cfg["B"]
    ctx.configure(v_e=v_e, theta_i=[cfg["theta"]] * L, y_cap_i=[S.K * B] * L, seed=0)
    T = 4 * a.tokens + 4 + a.adapt
    H = synth.hidden_states(1, T * B, L, S.d).permute(1, 0, 2).contiguous().to("cuda")
    Hh = H.cpu()
    y = torch.empty(B, S.d, dtype=torch.float32, device="cuda")
    st = torch.cuda.Stream()
    F = api.M.FUSE_PREDICT
    t = 0

    def run(mode, ntok):
        nonlocal t
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(ntok):
            for i in range(L):
                if mode == "host":
                    ctx.layer_forward_host(i, synth.bf16_bits(Hh[i, t * B:(t + 1) * B]), stream=st, flags=F, trace=False)
                else:
                    ctx.layer_forward(i, H[i, t * B:(t + 1) * B], y, stream=st, flags=F, trace=False)
                    if mode == "sync":
                        st.synchronize()
            t += 1
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / (ntok * L) * 1e6

    if a.adapt:   # the bench's Alg. 1 step (bench.py run_ours)
        ctx.profile(True)
        run("device", a.adapt)
        k2w = ctx.profile_read(api.M.KERNEL_EXPERT)
        ctx.profile(False)
        pcie = bench.pcie_probe(torch)
        t_load = 6 * S.d * S.I / (pcie * 1e9) * 1e3
        t_moe = k2w["total_ms"] / (a.adapt * L)
        r = ctx.configure(use_solver=True, t_att=0.0, t_moe=t_moe, t_head=0.0, t_load_exp=t_load, zeta=0.01,
                          v_e=v_e, y_cap_i=[S.K * B] * L, seed=0)
        print("theta", min(r["theta_eff_i"]), max(r["theta_eff_i"]), flush=True)
    run("device", 2)
    for mode in ("device", "sync", "host", "device"):
        print(f"{a.config} {mode:7s} {run(mode, a.tokens):8.1f} us/layer", flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
