"""PCIe bytes per token of the decode modes on the host control plane alone (tools; no GPU).

The GPU decode path is PCIe-bound (path fraction ~0.9-0.99), so tokens/s follows the bytes the
control plane decides to move: on-demand + prefetch.  `moepic_hostsim` is the library's own
control plane (bit-exact with the GPU path, tests/test_hostsim_vs_oracle.py), so long token
sequences can be compared here in seconds instead of GPU minutes.

    python scripts/bytes_sim.py [--shape mixtral] [--tokens 512] [--warm 128]

Routing: the bench's synthetic process (synth/ routers + organic hidden states), ids and the
fused next-layer ranking from fp64 logits.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402
from paper_2509_08342_b200 import api  # noqa: E402

ALG1_PCIE_GBS, ALG1_HBM_GBS, ALG1_LAUNCH_MS = 55.6, 6200.0, 0.015


def routing(S, L, T, seed=1):
    W = [synth.router_weights(0, i, S.N, S.d).double().numpy() for i in range(L)]
    H = synth.hidden_states(seed, T, L, S.d).double().numpy()          # [T][L][d]
    ids = np.zeros((T, L, S.K), np.int32)
    rank = np.zeros((T, L, S.N), np.int32)
    for i in range(L):
        lg = H[:, i] @ W[i].T
        ids[:, i] = np.argsort(-lg, axis=1, kind="stable")[:, :S.K]
        lp = H[:, i] @ W[(i + 1) % L].T                                 # fused predictor (Eq. 3)
        rank[:, i] = np.argsort(-lp, axis=1, kind="stable")
    return ids, rank


def run(S, L, ids, rank, mode, warm, tokens, window_rows=None, t_moe_ms=None):
    desc = api.model_desc(L, S.N, S.K, S.d, S.I, n_shared=S.n_shared, row_granule=64, max_batch=1,
                          v_e_max=float(L * S.N))
    hs = api.HostSim(desc)
    v_e = 0.5 * L * S.N
    base = dict(v_e=v_e, theta_i=[0.5] * L, y_cap_i=[S.K] * L, seed=0)
    if window_rows is not None:
        base["prefetch_rows_i"] = [window_rows] * L
    solver = mode in ("moepic", "no-lcp", "moepic-int")
    if mode == "cache-only":
        base.update(theta_i=[1.0] * L, prefetch=False)
    if mode == "lru":
        base.update(theta_i=[1.0] * L, prefetch=False, policy=api.M.LRU)
    if mode == "no-lcp":
        base["policy"] = api.M.RND
    hs.configure(**base)
    rb = 6 * S.d
    U_e = rb * S.I
    od = pf = 0

    def tok(t):
        nonlocal od, pf
        o = p = 0
        for i in range(L):
            tr = hs.step(i, ids[t, i][None], (i + 1) % L, rank[t, i])
            o += tr.pcie_ondemand
            p += tr.pcie_prefetch
        return o, p

    for t in range(warm):
        tok(t)
    if solver:
        t_load = U_e / (ALG1_PCIE_GBS * 1e9) * 1e3
        t_moe = S.K * U_e / (ALG1_HBM_GBS * 1e9) * 1e3 + ALG1_LAUNCH_MS if t_moe_ms is None else t_moe_ms
        res = hs.configure(use_solver=True, t_att=0.0, t_moe=t_moe, t_head=0.0, t_load_exp=t_load, zeta=0.01,
                           **{k: v for k, v in base.items() if k != "theta_i"})
        if mode == "moepic-int":   # experiment: Alg. 1's budgets rounded to whole experts, theta = 1
            V = np.array(res["V_i"])
            Vr = np.floor(V)
            rest = int(round(V.sum() - Vr.sum()))
            for i in np.argsort(-(V - Vr))[:rest]:
                Vr[i] += 1
            hs.configure(**dict(base, v_i=[float(x) for x in Vr], theta_i=[1.0] * L, prefetch=False))
    for t in range(warm, warm + tokens):
        o, p = tok(t)
        od += o
        pf += p
    return dict(mode=mode, od_GB_per_tok=round(od / tokens / 1e9, 3), pf_GB_per_tok=round(pf / tokens / 1e9, 3),
                total_GB_per_tok=round((od + pf) / tokens / 1e9, 3),
                tok_s_at_link=round(ALG1_PCIE_GBS / max((od + pf) / tokens / 1e9, 1e-9), 3))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="mixtral")
    ap.add_argument("--layers", type=int, default=None)
    ap.add_argument("--tokens", type=int, default=512)
    ap.add_argument("--warm", type=int, default=128)
    ap.add_argument("--modes", nargs="+", default=["moepic", "cache-only", "lru", "no-lcp"])
    ap.add_argument("--t-moe-ms", type=float, nargs="*", default=[None],
                    help="Alg. 1's T_moe (default: the bench's modelled value)")
    a = ap.parse_args()
    S = synth.SHAPES[a.shape]
    L = a.layers or S.L
    ids, rank = routing(S, L, a.warm + a.tokens)
    for m in a.modes:
        for tm in (a.t_moe_ms if m in ("moepic", "no-lcp") else [None]):
            print(json.dumps(dict(shape=a.shape, L=L, t_moe_ms=tm, **run(S, L, ids, rank, m, a.warm, a.tokens,
                                                                       t_moe_ms=tm))), flush=True)


if __name__ == "__main__":
    main()
