"""Cache policies (TEST INFRASTRUCTURE): LCP (Eq. 4) and the LRU / LFU / RND baselines.

  LCP priority   P_{i,j} = mu_{i,j} * rho^(nu_{i,j} / omega)            Eq. 4
                 defaults omega = 128, rho = 0.25
  eviction       "evicts the lowest-priority expert"
  LRU / LFU      Mixtral-offloading / MoE-Infinity policies
  RND            "randomly selecting cached experts"

Victim order (reading Q13): minimum of (key asc, nu desc, id asc).
Retention order for re-layout ("ranks all N experts by their cache priorities"):
(key desc, nu asc, id asc).  RND draws come from splitmix64, which the
C++ side implements independently.
"""
from __future__ import annotations

import math

LCP, LRU, LFU, RND = 0, 1, 2, 3
MASK64 = (1 << 64) - 1


def lcp_priority(mu: int, nu: int, rho: float, omega: int) -> float:
    """Eq. 4, evaluated as float(mu) * pow(rho, float(nu) / float(omega))."""
    return float(mu) * math.pow(rho, float(nu) / float(omega))


def policy_key(policy: int, mu: int, nu: int, last: int, rho: float, omega: int):
    if policy == LCP:
        return lcp_priority(mu, nu, rho, omega)
    if policy == LRU:
        return last            # larger = more recent
    if policy == LFU:
        return mu
    raise ValueError("RND has no key")


def splitmix64_next(state: int):
    """Standard splitmix64 step: returns (new_state, output)."""
    state = (state + 0x9E3779B97F4A7C15) & MASK64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    z = z ^ (z >> 31)
    return state, z


def layer_stream_seed(seed: int, layer: int, salt: int) -> int:
    """Initial splitmix64 state of the per-layer stream `salt` (1 = RND victims, 2 = initial set)."""
    s = (seed ^ ((0xD1B54A32D192ED03 * (layer + 1)) & MASK64) ^ ((0x8CB92BA72F3D8DD7 * salt) & MASK64)) & MASK64
    _, out = splitmix64_next(s)
    return out


def fisher_yates(n: int, state: int):
    """Permutation of range(n) by Fisher-Yates with splitmix64 draws:
    for i = n-1 .. 1: j = draw % (i + 1); swap(p[i], p[j]).  Returns (perm, state)."""
    p = list(range(n))
    for i in range(n - 1, 0, -1):
        state, z = splitmix64_next(state)
        j = z % (i + 1)
        p[i], p[j] = p[j], p[i]
    return p, state
