"""Helpers for the GPU parity tests: build a library context and the oracle from the same
seeded synthetic inputs (synth/), run both, and compare.  Test infrastructure only."""
from __future__ import annotations

import numpy as np
import torch

import synth
from oracle import numeric as ON
from oracle.replay import OracleEngine, CacheConfig

TOL = 2e-3   # BASELINE north_star: max|gpu - ref| / max|ref| <= 2e-3


class Model:
    """Synthetic MoE stack: routers per logical layer, experts per physical layer."""

    def __init__(self, L, N, K, d, I, n_shared=0, L_host=None, seed=0, kappa=1.0, gen_device="cpu"):
        self.L, self.N, self.K, self.d, self.I, self.n_shared = L, N, K, d, I, n_shared
        self.L_host = L if L_host is None else L_host
        self.seed = seed
        self.routers = [synth.bf16_bits(synth.router_weights(seed, i, N, d, kappa)) for i in range(L)]
        self.experts = {}
        for pl in range(self.L_host):
            for e in range(N):
                g, u, dn = synth.expert_weights(seed, pl, e, d, I, device=gen_device)
                self.experts[(pl, e)] = tuple(synth.bf16_bits(x) for x in (g, u, dn))
        self.shared = {}
        for i in range(L):
            for s in range(n_shared):
                g, u, dn = synth.shared_expert_weights(seed, i, s, d, I, device=gen_device)
                self.shared[(i, s)] = tuple(synth.bf16_bits(x) for x in (g, u, dn))

    def expert(self, layer, e):
        return self.experts[(layer % self.L_host, e)]

    def load_into(self, ctx):
        for i in range(self.L):
            ctx.load_router(i, self.routers[i])
        for (pl, e), (g, u, dn) in self.experts.items():
            ctx.load_expert(pl, e, g, u, dn)
        for (i, s), (g, u, dn) in self.shared.items():
            ctx.load_expert(i, -1 - s, g, u, dn)

    def oracle_layer(self, layer, h_bits, renorm=True):
        """fp64 dense reference of one layer (the plain definition, oracle/numeric.py)."""
        shared = [self.shared[(layer, s)] for s in range(self.n_shared)]
        return ON.moe_layer(h_bits, self.routers[layer], lambda e: self.expert(layer, e), self.K,
                            shared=shared, renorm=renorm)


def rel_err(y_gpu, y_ref):
    return float(np.abs(y_gpu - y_ref).max() / np.abs(y_ref).max())
