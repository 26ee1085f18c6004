"""Cache configurator, Algorithm 1 (TEST INFRASTRUCTURE).

Canonical fp64 formulas, evaluated in exactly this order (the C++ solver follows the same
written order independently; DESIGN.md §Alg1 lists them):

  sub-problem (Eq. 10) for layer i with budget V and window W:
    for C = max(1, ceil(V - 1e-9)) .. N:                      (theta <= 1)
      theta = min(1, V / C)                                    (theta_i = V_i / C_i)
      m = (K * H(C)) * theta                                   (A_cache)
      cum = 0; fcum = 0
      for y = 1 .. N:
        f = 1 - PH(y, C) * theta                               (Eq. 9a / 9b bracket)
        c = f * T_load                                         (T_pref, Eq. 9a)
        stop if cum + c > W  or  fcum + f > U_b                (window; buffer S:434)
        cum = cum + c; fcum = fcum + f
        m = m + f * P(y)                                       (A_pref, Eq. 9b; reading Q16)
      keep C if m > m_best (strict: ties -> smaller C)
  exposed   T = max(0, (K - m) * T_load - m * T_cexp)          (Eqs. 5-6 with the
  window    W' = (T_moe - min(m * T_cexp, (K - m) * T_load)) + T_att   m-approx; Eq. 7)
  ExpertSplit: W_1 = T_head + T_att; layers solved in order.
  VramAllocation: probes +-zeta*V_e on every layer at once, i1 = argmax
  (T1 - T2), i2 = argmin_{i != i1, V_i >= zeta V_e} (T3 - T1) (ties -> smaller index; reading
  Q19), move zeta*V_e from i2 to i1, roll back and return if sum(T4 - T1) >= 0; hard cap
  10 * L * ceil(1/zeta) iterations.
  T_comp^exp = T_moe / K.
"""
from __future__ import annotations

import math
from dataclasses import dataclass


@dataclass
class SubResult:
    C: int
    theta: float
    m: float
    T: float
    window_next: float
    Y: int = 0          # prefetch operations that fit the window at C* (Eq. 10)


def solve_subproblem(st, V: float, W: float, K: int, N: int, U_b: float,
                     t_load: float, t_cexp: float, t_moe: float, t_att: float) -> SubResult:
    best_C, best_theta, best_m, best_Y = None, 0.0, 0.0, 0
    C_lo = max(1, int(math.ceil(V - 1e-9)))
    if C_lo > N:
        C_lo = N
    for C in range(C_lo, N + 1):
        theta = V / C
        if theta > 1.0:
            theta = 1.0
        m = (K * st.H(C)) * theta
        cum = 0.0
        fcum = 0.0
        Y = 0
        for y in range(1, N + 1):
            f = 1.0 - st.PH(y, C) * theta
            c = f * t_load
            if cum + c > W or fcum + f > U_b:
                break
            cum = cum + c
            fcum = fcum + f
            m = m + f * st.P(y)
            Y = y
        if best_C is None or m > best_m:
            best_C, best_theta, best_m, best_Y = C, theta, m, Y
    m = best_m
    T = max(0.0, (K - m) * t_load - m * t_cexp)
    w_next = (t_moe - min(m * t_cexp, (K - m) * t_load)) + t_att
    return SubResult(best_C, best_theta, m, T, w_next, best_Y)


def expert_split(stats, V, K, N, U_b, t_att, t_moe, t_head, t_load, Ys=None):
    """Function ExpertSplit.  Returns (T[], theta[], C[]); fills Ys with Y_i if given."""
    t_cexp = t_moe / K
    W = t_head + t_att
    Ts, ths, Cs = [], [], []
    for i in range(len(V)):
        r = solve_subproblem(stats[i], V[i], W, K, N, U_b, t_load, t_cexp, t_moe, t_att)
        Ts.append(r.T)
        ths.append(r.theta)
        Cs.append(r.C)
        if Ys is not None:
            Ys.append(r.Y)
        W = r.window_next
    return Ts, ths, Cs


def vram_allocation(stats, V_init, V_e, zeta, K, N, U_b, t_att, t_moe, t_head, t_load):
    """Function VramAllocation.  Returns (V[], theta[], C[], iterations, converged).
    The final ExpertSplit's per-layer Y (prefetches fitting the window, Eq. 10) is available as
    vram_allocation.last_Y after the call."""
    L = len(V_init)
    delta = zeta * V_e
    V = list(V_init)
    cap = 10 * L * int(math.ceil(1.0 / zeta))
    es = lambda vv: expert_split(stats, vv, K, N, U_b, t_att, t_moe, t_head, t_load)

    def _ys(vv):
        ys = []
        expert_split(stats, vv, K, N, U_b, t_att, t_moe, t_head, t_load, ys)
        return ys
    for it in range(cap):
        T1, th1, C1 = es(V)
        T2, _, _ = es([v + delta for v in V])
        T3, _, _ = es([max(0.0, v - delta) for v in V])
        i1 = 0
        for i in range(1, L):
            if T1[i] - T2[i] > T1[i1] - T2[i1]:
                i1 = i
        i2 = -1
        for i in range(L):
            if i == i1 or V[i] + 1e-9 < delta:
                continue
            if i2 < 0 or T3[i] - T1[i] < T3[i2] - T1[i2]:
                i2 = i
        if i2 < 0:
            vram_allocation.last_Y = _ys(V)
            return V, th1, C1, it, True
        Vn = list(V)
        Vn[i1] = Vn[i1] + delta
        Vn[i2] = Vn[i2] - delta
        if Vn[i2] < 0.0:
            Vn[i2] = 0.0
        T4, _, _ = es(Vn)
        s = 0.0
        for i in range(L):
            s = s + (T4[i] - T1[i])
        if s >= 0.0:
            vram_allocation.last_Y = _ys(V)
            return V, th1, C1, it, True
        V = Vn
    T, th, C = es(V)
    vram_allocation.last_Y = _ys(V)
    return V, th, C, cap, False
