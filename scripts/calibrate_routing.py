"""Calibrate the synthetic "organic" routing (synth/) against the paper's regimes with the oracle.

Targets: LCP hit rate at a cache of 20 of 60 experts near Table 1's 45.36 %
(Qwen1.5-MoE shape N = 60, K = 4), and next-layer prediction accuracy inside the
2.07-3.39 of 4 band (52-85 %).  Prints one JSON line per (kappa, eps).

    python scripts/calibrate_routing.py [--tokens 1500]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402
from oracle import numeric as ON  # noqa: E402
from oracle.replay import OracleEngine, CacheConfig, GAMMA  # noqa: E402


def run(kappa, eps, tokens, a=0.8, N=60, K=4, d=512, L=3):
    routers = [synth.bf16_bits(synth.router_weights(0, i, N, d, kappa=kappa)) for i in range(L)]
    H = synth.hidden_states(1, tokens, L, d, eps=eps, a=a)
    ids = []
    acc = []
    for i in range(L):
        hb = synth.bf16_bits(H[:, i])
        lg = ON.router_logits(hb, routers[i])
        ids.append(np.argsort(-lg, axis=1, kind="stable")[:, :K])
        if i > 0:
            pred = np.argsort(-ON.router_logits(synth.bf16_bits(H[:, i - 1]), routers[i]), axis=1, kind="stable")[:, :K]
            acc.append(np.mean([len(set(a) & set(p)) for a, p in zip(ids[i], pred)]))
    # LCP hit rate at C = 20 of 60 (cache-only, full experts, theta = 1)
    e = OracleEngine(1, N, K, d, 64, row_granule=16)
    e.configure(CacheConfig(v_e=20.0, theta_i=[1.0], prefetch=False))
    hits = tot = 0
    for t in range(tokens):
        tr = e.step(0, ids[1][t][None])
        if t >= tokens // 5:
            hits += sum(1 for (_, c) in tr.act if c != GAMMA)
            tot += K
    return dict(kappa=kappa, eps=eps, a=a, lcp_hit_C20=round(hits / tot, 4), pred_correct_of_K=round(float(np.mean(acc)), 3))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=1500)
    ap.add_argument("--kappas", default="0.25,0.5,0.75,1.0")
    ap.add_argument("--eps", default="0.35")
    ap.add_argument("--a", default="0.8")
    a = ap.parse_args()
    for k in map(float, a.kappas.split(",")):
        for e in map(float, a.eps.split(",")):
            for ar in map(float, a.a.split(",")):
                print(json.dumps(run(k, e, a.tokens, a=ar)), flush=True)


if __name__ == "__main__":
    main()
