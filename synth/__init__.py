"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no routing, no SwiGLU, no cache
policy): it only draws weights and hidden states with the shapes and structure of the
paper's workloads.  Both sides (oracle/ and the CUDA path)
consume its outputs; neither imports the other.

Recipe:
  * expert weights: W_gate, W_up ~ N(0, 1/d) of shape [I][d]; W_down ~ N(0, 1/I) of
    shape [d][I] (HuggingFace layout), rounded to bf16 (round-to-nearest-even).
  * router rows ("organic" routing; long tail P:323, temporal locality P:324,
    cross-layer similarity P:283-286):  W_r^i[j] = g_j + kappa * c_{i,j} * u, with
    g_j ~ N(0, 1/d), u a fixed unit vector, c_{i,j} = -ln(rank_i(j)) for a per-layer
    random permutation rank_i (Zipf-like popularity).
  * hidden states: x_t = a*x_{t-1} + sqrt(1-a^2)*n_t  (AR(1), unit variance per coord),
    h_t^i = bf16(mu*u + x_t + eps*z_{t,i}).
bf16 values are returned as torch.bfloat16 tensors (or their uint16 bit patterns).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

__all__ = [
    "ModelShape", "SHAPES", "bf16_bits", "bits_to_bf16",
    "expert_weights", "router_weights", "hidden_states", "shared_expert_weights",
]


@dataclass(frozen=True)
class ModelShape:
    name: str
    L: int
    N: int
    K: int
    d: int
    I: int
    n_shared: int = 0
    renorm: int = 1


# BASELINE.json configs.  L for Qwen3/DeepSeek from their public configs.
SHAPES = {
    "toy": ModelShape("toy", L=2, N=8, K=2, d=64, I=128),
    "mixtral": ModelShape("mixtral", L=32, N=8, K=2, d=4096, I=14336),
    "qwen3": ModelShape("qwen3", L=48, N=128, K=8, d=2048, I=768),
    "deepseek": ModelShape("deepseek", L=26, N=64, K=6, d=2048, I=1408, n_shared=2),
}


def bf16_bits(t: torch.Tensor) -> np.ndarray:
    """bf16 tensor -> numpy uint16 bit patterns (host)."""
    return t.detach().to("cpu").contiguous().view(torch.int16).numpy().view(np.uint16)


def bits_to_bf16(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16)


def _gen(seed: int, *stream: int, device="cpu") -> torch.Generator:
    # one independent Philox/MT stream per (seed, stream ids)
    s = seed & 0xFFFFFFFF
    for x in stream:
        s = (s * 1000003 + (x & 0xFFFFFFFF) + 0x9E3779B9) & 0x7FFFFFFFFFFFFFFF
    g = torch.Generator(device=device)
    g.manual_seed(s)
    return g


def expert_weights(seed: int, layer: int, expert: int, d: int, I: int, device="cpu"):
    """(gate [I][d], up [I][d], down [d][I]) bf16, HF layout.  expert < 0 => shared expert."""
    g = _gen(seed, 1, layer, expert + 1000, device=device)
    gate = (torch.randn(I, d, generator=g, device=device) / math.sqrt(d)).to(torch.bfloat16)
    up = (torch.randn(I, d, generator=g, device=device) / math.sqrt(d)).to(torch.bfloat16)
    down = (torch.randn(d, I, generator=g, device=device) / math.sqrt(I)).to(torch.bfloat16)
    return gate, up, down


def shared_expert_weights(seed: int, layer: int, s: int, d: int, I: int, device="cpu"):
    return expert_weights(seed, layer, -1 - s, d, I, device=device)


def _unit_u(seed: int, d: int) -> torch.Tensor:
    g = _gen(seed, 2)
    u = torch.randn(d, generator=g, dtype=torch.float64)
    return u / u.norm()


def router_weights(seed: int, layer: int, N: int, d: int, kappa: float = 0.5) -> torch.Tensor:
    """Router R^i as bf16 [N][d] with a Zipf-like popularity bias along u."""
    g = _gen(seed, 3, layer)
    base = torch.randn(N, d, generator=g, dtype=torch.float64) / math.sqrt(d)
    perm = torch.randperm(N, generator=g)           # rank_i(j) = perm[j] + 1
    c = -torch.log((perm + 1).to(torch.float64))
    c = c - c.mean()
    u = _unit_u(seed, d)
    w = base + kappa * c[:, None] * u[None, :]
    return w.to(torch.bfloat16)


def hidden_states(seed: int, T: int, L: int, d: int, mu: float = 1.0, a: float = 0.35,
                  eps: float = 0.35, scale: float = 1.0) -> torch.Tensor:
    """h[t][i] bf16 [T][L][d]: AR(1) token process + per-layer perturbation."""
    g = _gen(seed, 4, L)   # prefix-stable: the first t tokens do not depend on T
    u = _unit_u(seed, d)
    x = torch.randn(d, generator=g, dtype=torch.float64)
    out = torch.empty(T, L, d, dtype=torch.float64)
    for t in range(T):
        if t:
            x = a * x + math.sqrt(1 - a * a) * torch.randn(d, generator=g, dtype=torch.float64)
        z = torch.randn(L, d, generator=g, dtype=torch.float64)
        out[t] = scale * (mu * u[None, :] + x[None, :] + eps * z)
    return out.to(torch.bfloat16)


def batch_hidden(seed: int, B: int, d: int, scale: float = 1.0) -> torch.Tensor:
    """Independent tokens h [B][d] bf16 (prefill / batch parity cases)."""
    g = _gen(seed, 5, B)
    return (scale * torch.randn(B, d, generator=g, dtype=torch.float64)).to(torch.bfloat16)
