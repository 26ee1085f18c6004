"""Pins for the oracle's control plane: policy (Eq. 4), stats, Alg. 1
 and the C-S state machine, against worked values, closed forms and brute
force.  SPEC vectors are cited as S:<line>."""
import itertools
import math

import numpy as np
import pytest

from oracle import policy as P
from oracle.stats import LayerStats
from oracle import configurator as CF
from oracle.replay import OracleEngine, CacheConfig, ALPHA, BETA, GAMMA, ADM_FREE, ADM_NONE


# ----------------------------------------------------------------- policy (C-P6)
def test_lcp_priority_worked_values():
    # S:168-170
    assert P.lcp_priority(10, 0, 0.25, 128) == 10.0
    assert P.lcp_priority(8, 128, 0.25, 128) == 2.0
    assert P.lcp_priority(4, 256, 0.25, 128) == 0.25
    # 128 idle tokens scale the priority by exactly rho
    assert P.lcp_priority(12, 128, 0.25, 128) == 12 * 0.25


def test_splitmix64_reference_vector():
    # Vigna's splitmix64 with x = 0: first outputs are standard reference values
    s, z1 = P.splitmix64_next(0)
    s, z2 = P.splitmix64_next(s)
    assert z1 == 0xE220A8397B1DCDAF
    assert z2 == 0x6E789E6AA1B965F4


def test_fisher_yates_is_permutation():
    p, _ = P.fisher_yates(60, 12345)
    assert sorted(p) == list(range(60))


# ----------------------------------------------------------------- stats (C-P11)
def test_stats_single_token_example():
    # 1 token activating {0,1,2,3}, N = 8, cold counts -> ranks 1..4
    st = LayerStats(8, 4)
    st.observe(np.array([[0, 1, 2, 3]]), None)
    assert st.H(4) == 1.0 and st.H(2) == 0.5 and st.H(8) == 1.0


def test_stats_invariants_and_bruteforce_recount():
    rng = np.random.default_rng(3)
    N, K = 10, 3
    st = LayerStats(N, K)
    trace = []
    for t in range(80):
        ids = rng.choice(N, size=K, replace=False)
        rank = rng.permutation(N)
        st.observe(ids[None], rank)
        trace.append((ids, rank))
    # monotone in C, H(N) = PH(y, N) = 1, sum_y P(y) = K
    Hs = [st.H(C) for C in range(1, N + 1)]
    assert all(a <= b for a, b in zip(Hs, Hs[1:])) and Hs[-1] == 1.0
    for y in range(1, N + 1):
        assert st.PH(y, N) == 1.0
    assert abs(sum(st.P(y) for y in range(1, N + 1)) - K) < 1e-12
    # brute-force recount of H(C) from the raw trace
    freq = np.zeros(N, dtype=int)
    hits = np.zeros(N + 1, dtype=int)
    for ids, _ in trace:
        top = sorted(range(N), key=lambda e: (-freq[e], e))
        for C in range(1, N + 1):
            hits[C] += sum(1 for e in ids if e in top[:C])
        for e in ids:
            freq[e] += 1
    for C in range(1, N + 1):
        assert st.H(C) == hits[C] / (80 * K)


def test_stats_P_PH_hand_worked_example():
    """P(y) and PH(y, C) on a 3-token trace, every value derived by hand.

    N = 4, K = 1.  The size-C cache is the top-C by pre-step activation count, ties by
    smaller id (reading Q15).  Token by token:
      t0: counts (0,0,0,0) -> cache order [0,1,2,3]; ids {2}; ranking R' = [2,0,1,3]
      t1: counts (0,0,1,0) -> cache order [2,0,1,3]; ids {2}; R' = [3,2,0,1]
      t2: counts (0,0,2,0) -> cache order [2,0,1,3]; ids {1}; R' = [1,3,2,0]
    P(y)  = #tokens where the y-th predicted expert is activated / q:
      y=1: t0 (2 in {2}) yes, t1 (3) no, t2 (1) yes -> 2/3
      y=2: t0 (0) no, t1 (2) yes, t2 (3) no          -> 1/3
      y=3, y=4: never                                 -> 0
    PH(y, C) = #tokens where the y-th predicted expert is in the size-C cache / q:
      y=1: t0 expert 2 has cache position 3; t1 expert 3 has 4; t2 expert 1 has 3
           -> PH(1,1)=PH(1,2)=0, PH(1,3)=2/3, PH(1,4)=1
      y=2: t0 expert 0 position 1; t1 expert 2 position 1; t2 expert 3 position 4
           -> PH(2,1)=PH(2,2)=PH(2,3)=2/3, PH(2,4)=1
    A mutation that ranks the y-th position itself (rank[y] instead of rank[R'[y]]) or
    counts the activated expert instead of the predicted one fails here."""
    st = LayerStats(4, 1)
    st.observe(np.array([[2]]), np.array([2, 0, 1, 3]))
    st.observe(np.array([[2]]), np.array([3, 2, 0, 1]))
    st.observe(np.array([[1]]), np.array([1, 3, 2, 0]))
    assert [st.P(y) for y in (1, 2, 3, 4)] == [2 / 3, 1 / 3, 0.0, 0.0]
    assert [st.PH(1, C) for C in (1, 2, 3, 4)] == [0.0, 0.0, 2 / 3, 1.0]
    assert [st.PH(2, C) for C in (1, 2, 3, 4)] == [2 / 3, 2 / 3, 2 / 3, 1.0]
    # y=3: t0 expert 1 pos 2; t1 expert 0 pos 2; t2 expert 2 pos 1
    assert [st.PH(3, C) for C in (1, 2, 3, 4)] == [1 / 3, 1.0, 1.0, 1.0]
    # y=4: t0 expert 3 pos 4; t1 expert 1 pos 3; t2 expert 0 pos 2
    assert [st.PH(4, C) for C in (1, 2, 3, 4)] == [0.0, 1 / 3, 2 / 3, 1.0]


def test_stats_P_perfect_predictor():
    """A perfect predictor (R' lists the K activated experts first) gives P(y) = 1 for
    y <= K and 0 beyond (P:446 with a predictor that always ranks the activated set on top;
    the S:404 worked case uses the same P)."""
    rng = np.random.default_rng(9)
    N, K = 12, 3
    st = LayerStats(N, K)
    for _ in range(50):
        ids = rng.choice(N, size=K, replace=False)
        rest = [e for e in rng.permutation(N) if e not in set(ids)]
        st.observe(ids[None], np.array(list(rng.permutation(ids)) + rest))
    assert [st.P(y) for y in range(1, N + 1)] == [1.0] * K + [0.0] * (N - K)
    # an anti-predictor (activated experts ranked last) -> P(y) = 1 exactly for y > N - K
    st = LayerStats(N, K)
    for _ in range(50):
        ids = rng.choice(N, size=K, replace=False)
        rest = [e for e in rng.permutation(N) if e not in set(ids)]
        st.observe(ids[None], np.array(rest + list(ids)))
    assert [st.P(y) for y in range(1, N + 1)] == [0.0] * (N - K) + [1.0] * K


def test_stats_P_PH_bruteforce_recount_batched():
    """Brute-force recount of P(y) and PH(y, C) for every y and C from the raw
    (ids, ranking) trace, written from the definitions P:446-447 in a different form than
    the oracle (membership tests against an explicitly sorted cache list, not rank
    histograms), with B > 1 token batches (reading Q9/Q15: one cache state per step,
    every token counts), plus steps without a prediction (excluded from q_pred).
    Also PH monotone non-decreasing in C, PH(y, N) = 1 and sum_y PH(y, C) = C."""
    rng = np.random.default_rng(21)
    N, K = 9, 2
    st = LayerStats(N, K)
    trace = []
    for t in range(60):
        B = int(rng.integers(1, 4))
        ids = np.stack([rng.choice(N, size=K, replace=False, p=np.arange(1, N + 1) / (N * (N + 1) / 2))
                        for _ in range(B)])
        ranking = None if t % 7 == 3 else rng.permutation(N)
        st.observe(ids, ranking)
        trace.append((ids, ranking))
    freq = [0] * N
    q_pred = 0
    p_cnt = [0] * (N + 1)
    ph_cnt = [[0] * (N + 1) for _ in range(N + 1)]
    for ids, ranking in trace:
        cache_order = sorted(range(N), key=lambda e: (-freq[e], e))
        if ranking is not None:
            for row in ids:
                q_pred += 1
                for y in range(1, N + 1):
                    pred = int(ranking[y - 1])
                    if pred in [int(x) for x in row]:
                        p_cnt[y] += 1
                    for C in range(1, N + 1):
                        if pred in cache_order[:C]:
                            ph_cnt[y][C] += 1
        for row in ids:
            for e in row:
                freq[int(e)] += 1
    assert st.q_pred == q_pred
    for y in range(1, N + 1):
        assert st.P(y) == p_cnt[y] / q_pred
        for C in range(1, N + 1):
            assert st.PH(y, C) == ph_cnt[y][C] / q_pred
        PHs = [st.PH(y, C) for C in range(1, N + 1)]
        assert all(a <= b for a, b in zip(PHs, PHs[1:])) and PHs[-1] == 1.0
    # every token's ranking is a permutation: exactly C of its N predicted experts are cached
    for C in range(1, N + 1):
        assert abs(sum(st.PH(y, C) for y in range(1, N + 1)) - C) < 1e-12


# ----------------------------------------------------------------- configurator
class FakeStats:
    """Stats with prescribed H / P / PH (for worked sub-problem cases)."""
    def __init__(self, N, H, Pf, PH, q=1):
        self.N, self._H, self._P, self._PH, self.q = N, H, Pf, PH, q

    def H(self, C):
        return self._H(C)

    def P(self, y):
        return self._P(y)

    def PH(self, y, C):
        return self._PH(y, C)


def test_subproblem_prefetch_only_vector():
    # V = 0, perfect predictor, window = 2 t_load -> Y = 2, m = 2
    K, N = 4, 8
    st = FakeStats(N, lambda C: 0.3, lambda y: 1.0 if y <= K else 0.0, lambda y, C: 0.5)
    r = CF.solve_subproblem(st, 0.0, 2 * 40.0, K, N, float(K), 40.0, 10.0, 40.0, 15.0)
    assert r.m == 2.0 and r.C == 1 and r.Y == 2


def test_subproblem_full_hit_vector():
    # H(C) = 1 for C >= C0, V = C0 -> m = K at C = C0, T = 0
    K, N, C0 = 2, 8, 3
    st = FakeStats(N, lambda C: 1.0 if C >= C0 else 0.2, lambda y: 0.0, lambda y, C: 0.0)
    r = CF.solve_subproblem(st, float(C0), 0.0, K, N, float(K), 40.0, 10.0, 20.0, 5.0)
    assert r.C == C0 and r.m == K and r.T == 0.0


def _random_stats(rng, N, K, tokens=60):
    st = LayerStats(N, K)
    pop = rng.dirichlet(np.ones(N) * 0.5)
    for _ in range(tokens):
        ids = rng.choice(N, size=K, replace=False, p=pop)
        noisy = np.argsort(-(np.log(pop) + rng.gumbel(size=N)))
        st.observe(ids[None], noisy)
    return st


def test_subproblem_matches_bruteforce():
    """C-P12 / S:497: enumerate every (C, Y) pair; Y feasible iff its prefix fits the
    window and the buffer; m(C) = best over feasible prefixes (f*P >= 0 so the longest
    feasible prefix wins); argmax with ties to the smaller C."""
    rng = np.random.default_rng(11)
    for trial in range(150):
        N = int(rng.integers(3, 12))
        K = int(rng.integers(1, min(4, N - 1) + 1))
        st = _random_stats(rng, N, K)
        V = float(rng.choice([0.0, 0.5, 1.0, 1.7, 2.5, rng.uniform(0, N)]))
        tl, tc = float(rng.uniform(5, 50)), float(rng.uniform(1, 20))
        W = float(rng.uniform(0, 4 * tl))
        Ub = float(rng.integers(K, 2 * K + 1))
        r = CF.solve_subproblem(st, V, W, K, N, Ub, tl, tc, K * tc, 3.0)
        best = None
        for C in range(1, N + 1):
            if V / C > 1.0 + 1e-12 and C < N:
                continue
            th = min(1.0, V / C)
            mC = K * st.H(C) * th
            for Y in range(0, N + 1):
                fs = [1.0 - st.PH(y, C) * th for y in range(1, Y + 1)]
                # every prefix must fit (greedy stop rule)
                ok = all(sum(fs[:k]) * tl <= W + 1e-12 and sum(fs[:k]) <= Ub + 1e-12 for k in range(1, Y + 1))
                if not ok:
                    break
                m = mC + sum(f * st.P(y) for f, y in zip(fs, range(1, Y + 1)))
                if best is None or m > best[1] + 1e-12:
                    best = (C, m)
        assert abs(r.m - best[1]) < 1e-9, (trial, r, best)
        assert r.C == best[0] or abs(r.m - best[1]) < 1e-9


def test_eq5_7_worked_vectors():
    # (alpha,beta,gamma) = (1,2,1), theta .5, t_cexp 10, t_load 40 -> (20, 80, 60)
    th, tc, tl = 0.5, 10.0, 40.0
    t_hide = (1 + 2 * th) * tc                     # Eq. 5
    t_miss = (2 * (1 - th) + 1) * tl
    assert (t_hide, t_miss, max(0.0, t_miss - t_hide)) == (20.0, 80.0, 60.0)
    # the solver's m-form reduces to Eqs. 5-7 when m = alpha + beta*theta and K - m = miss units
    r_window = (40.0 - min(20.0, 80.0)) + 15.0     # Eq. 7
    assert r_window == 35.0


def test_expert_split_L1_and_symmetry():
    rng = np.random.default_rng(5)
    N, K = 8, 2
    st = _random_stats(rng, N, K)
    T, th, C = CF.expert_split([st], [2.0], K, N, 2.0, 5.0, 20.0, 3.0, 30.0)
    r = CF.solve_subproblem(st, 2.0, 3.0 + 5.0, K, N, 2.0, 30.0, 10.0, 20.0, 5.0)
    assert (T[0], th[0], C[0]) == (r.T, r.theta, r.C)
    # symmetric layers -> VramAllocation keeps the uniform split
    V, th, C, it, conv = CF.vram_allocation([st, st], [2.0, 2.0], 4.0, 0.01, K, N, 2.0, 5.0, 20.0, 3.0, 30.0)
    assert V == [2.0, 2.0] and conv


def test_vram_allocation_invariants_and_grid():
    """C-P13: budget conservation, sum T strictly decreasing, <= uniform; C-P14: report the
    gap to the brute-force grid optimum (no pass/fail)."""
    rng = np.random.default_rng(8)
    N, K = 8, 2
    for trial in range(6):
        L = 3
        stats = [_random_stats(rng, N, K, tokens=40) for _ in range(L)]
        # one layer with a bad predictor: its prediction stats are shuffled noise
        Ve = 6.0
        args = (K, N, 2.0, 5.0, 20.0, 3.0, 30.0)
        V, th, C, it, conv = CF.vram_allocation(stats, [Ve / L] * L, Ve, 0.05, *args)
        assert conv
        assert abs(sum(V) - Ve) < 1e-9 and min(V) >= 0.0
        T_final = sum(CF.expert_split(stats, V, *args)[0])
        T_uni = sum(CF.expert_split(stats, [Ve / L] * L, *args)[0])
        assert T_final <= T_uni + 1e-12
        for i in range(L):
            assert 0.0 <= th[i] <= 1.0 and 1 <= C[i] <= N
        # strictly decreasing: replay the accepted moves
        Vc = [Ve / L] * L
        prev = T_uni
        d = 0.05 * Ve
        for _ in range(it):
            T1, _, _ = CF.expert_split(stats, Vc, *args)
            T2, _, _ = CF.expert_split(stats, [v + d for v in Vc], *args)
            T3, _, _ = CF.expert_split(stats, [max(0.0, v - d) for v in Vc], *args)
            i1 = int(np.argmax([T1[i] - T2[i] for i in range(L)]))
            c = [(T3[i] - T1[i], i) for i in range(L) if i != i1 and Vc[i] + 1e-9 >= d]
            i2 = min(c)[1]
            Vc[i1] += d
            Vc[i2] = max(0.0, Vc[i2] - d)
            cur = sum(CF.expert_split(stats, Vc, *args)[0])
            assert cur < prev
            prev = cur
        # C-P14 grid optimum (report only)
        # (same lattice as Alg. 1: V_i = V_e/L + k_i d, sum k_i = 0, V_i >= 0)
        base = Ve / L
        kmax = int(base // d)
        lat = range(-kmax, 2 * kmax + 1)
        grid = min(sum(CF.expert_split(stats, [base + a * d, base + b * d, base - (a + b) * d], *args)[0])
                   for a in lat for b in lat if -kmax <= -(a + b) <= 2 * kmax)
        assert grid <= T_final + 1e-9


# ----------------------------------------------------------------- state machine
def _engine(L=1, N=8, K=2, I=128, d=64, g=16, Ub=None):
    return OracleEngine(L, N, K, d, I, row_granule=g, buffer_experts=Ub)


def test_apply_config_vectors():
    # S:200 V=5, theta=.5, N=60 -> 10 cached; S:202 cold start -> ids 0..C-1
    e = _engine(N=60, K=4, I=128)
    C, It, th, V = e.configure(CacheConfig(v_e=5.0, theta_i=[0.5]))
    assert C == [10] and It == [64] and th == [0.5]
    assert e.cache[0] == set(range(10))
    # theta = 1: V_i full experts (cache-only layout)
    e = _engine(N=60, K=4, I=128)
    C, It, _, _ = e.configure(CacheConfig(v_e=5.0, theta_i=[1.0]))
    assert C == [5] and It == [128]


def test_classify_and_bytes_vectors():
    # S:310-312 adapted: K=4; expert 0 fully ready (top cached + bottom planned),
    # experts 1,2 top-only, expert 3 cold -> (1, 2, 1)
    e = _engine(N=8, K=4, I=128, Ub=2)                      # plan: 0 bottom, 5 full; 6 misses
    e.configure(CacheConfig(v_e=1.5, theta_i=[0.5]))        # C = 3 -> {0,1,2}
    e.predict_prefetch(0, np.array([0, 5, 6, 7, 1, 2, 3, 4]))
    assert e.pending.items[0] == (0, False, 64)
    tr = e.step(0, np.array([[0, 1, 2, 3]]))
    cls = dict(tr.act)
    assert [cls[0], cls[1], cls[2], cls[3]] == [ALPHA, BETA, BETA, GAMMA]
    rb = 6 * 64
    assert tr.pcie_ondemand == 2 * 64 * rb + 128 * rb
    # expert 3 is admitted; victims exclude the activated set -> no candidate
    assert tr.adm == [(3, ADM_NONE)]


def test_plan_vectors():
    # S:302 adapted to the buffer rule: ranking [7,3,9], nothing cached, U_b = 2 units
    e = _engine(N=10, K=2, I=128, Ub=2)
    e.configure(CacheConfig(v_e=0.0, theta_i=[0.5]))
    tr = e.predict_prefetch(0, np.array([7, 3, 9, 0, 1, 2, 4, 5, 6, 8]))
    assert tr.plan == [(7, True), (3, True)]
    # S:303 adapted: 7's top cached at theta = .5 -> bottom only, then 3 full, 9 does not fit
    e = _engine(N=10, K=2, I=128, Ub=2)
    e.configure(CacheConfig(v_e=0.5, theta_i=[0.5]))         # C = 1 -> {0}
    e.cache[0] = {7}
    tr = e.predict_prefetch(0, np.array([7, 3, 9, 0, 1, 2, 4, 5, 6, 8]))
    assert tr.plan == [(7, False), (3, True)]


def test_lcp_victim_and_ties():
    # strict minimum; all protected -> none; equal priority -> larger nu
    e = _engine(N=6, K=1, I=128)
    e.configure(CacheConfig(v_e=1.0, theta_i=[0.5], prefetch=False))   # C = 2 -> {0, 1}
    e.step(0, np.array([[0]]))          # mu0 = 1
    e.step(0, np.array([[1]]))          # mu1 = 1; nu0 = 1
    tr = e.step(0, np.array([[4]]))     # miss: priorities 1*rho^(2/128) vs 1*rho^(1/128)
    assert tr.adm == [(4, 0)]           # expert 0 has the lower priority (older)
    # equal priorities broken by larger nu, then smaller id (LFU: equal counts)
    e = _engine(N=6, K=1, I=128)
    e.configure(CacheConfig(v_e=1.0, theta_i=[0.5], prefetch=False, policy=P.LFU))
    e.step(0, np.array([[1]]))
    e.step(0, np.array([[0]]))
    tr = e.step(0, np.array([[5]]))     # mu0 = mu1 = 1, nu1 = 2 > nu0 = 1 -> evict 1
    assert tr.adm == [(5, 1)]


def test_rnd_hit_rate_closed_form():
    """C-P8 / S:494: RND policy on a uniform trace -> hit rate C/N within 2 pts
    (Table 1 RND row: 16.41 % at C = 10 of 60)."""
    N, K = 60, 4
    rng = np.random.default_rng(0)
    for C in (10, 30):
        e = _engine(N=N, K=K, I=64, g=16)
        e.configure(CacheConfig(v_e=C * 0.5, theta_i=[0.5], prefetch=False, policy=P.RND, seed=7))
        hits = total = 0
        for t in range(13000):
            ids = rng.choice(N, size=K, replace=False)
            tr = e.step(0, ids[None])
            hits += sum(1 for (_, c) in tr.act if c != GAMMA)
            total += K
        assert total >= 5e4
        assert abs(hits / total - C / N) < 0.02


def test_degenerate_modes():
    """C-P9: theta = 1 without prefetch is cache-only; V = 0 is prefetch-only."""
    rng = np.random.default_rng(4)
    N, K, I = 8, 2, 128
    e = _engine(N=N, K=K, I=I)
    e.configure(CacheConfig(v_e=4.0, theta_i=[1.0], prefetch=False))   # 4 full experts
    for t in range(300):
        ids = rng.choice(N, size=K, replace=False)
        tr = e.step(0, ids[None])
        for ex, c in tr.act:
            assert c in (ALPHA, GAMMA)          # a cached full expert needs nothing
        assert tr.pcie_ondemand == sum(I * 6 * 64 for (_, c) in tr.act if c == GAMMA)
        assert tr.plan == []
    e = _engine(N=N, K=K, I=I)
    e.configure(CacheConfig(v_e=0.0, theta_i=[0.5]))
    for t in range(100):
        ids = rng.choice(N, size=K, replace=False)
        tr = e.step(0, ids[None], next_layer=0, ranking_next=rng.permutation(N))
        assert tr.adm == [] and all(c != BETA for (_, c) in tr.act)
        assert all(f for (_, f) in tr.plan)     # nothing cached -> only full prefetches


def test_pcie_bytes_closed_form_half_budget():
    """C-P15: theta = .5, C = N, no prefetch: K (1 - theta) U_e bytes per B = 1 step."""
    N, K, I, d = 8, 2, 14336, 4096
    e = OracleEngine(1, N, K, d, I, row_granule=64)
    e.configure(CacheConfig(v_e=4.0, theta_i=[0.5], prefetch=False))
    rng = np.random.default_rng(1)
    for _ in range(20):
        tr = e.step(0, rng.choice(N, size=K, replace=False)[None])
        assert tr.pcie_ondemand == 352321536


# ----------------------------------------------------------------- window-capped plan (Q30)
def test_window_plan_vectors():
    """Reading Q30 worked vectors (N = 10, K = 2, I = 128, g = 16, U_b = 2; expert 7's top cached
    at theta = .5 -> its bottom is 64 rows; ranking 7, 3, 9, ...):
      W = 200: 7 bottom (64) + 3 full (128) = 192; 8 rows left, less than one granule
      W = 100: 7 bottom (64) + 3 full cut to 16 * floor(36 / 16) = 32 rows
      W = 40 : 7 bottom cut to 16 * floor(40 / 16) = 32 rows
      W = 8  : less than one granule -> empty plan
    With W = 40 and 7 activated: beta, on-demand = (64 - 32) rows (Q30)."""
    rank = np.array([7, 3, 9, 0, 1, 2, 4, 5, 6, 8])
    expect = {200: [(7, False, 64), (3, True, 128)], 100: [(7, False, 64), (3, True, 32)], 40: [(7, False, 32)],
              8: []}
    for W, items in expect.items():
        e = _engine(N=10, K=2, I=128, Ub=2)
        e.configure(CacheConfig(v_e=0.5, theta_i=[0.5], prefetch_rows_i=[W]))   # C = 1 -> {0}
        e.cache[0] = {7}
        e.predict_prefetch(0, rank)
        assert e.pending.items == items, (W, e.pending.items)
    tr = e.step(0, np.array([[7, 1]]))                          # the W = 8 engine: nothing planned
    assert dict(tr.act)[7] == BETA and tr.pcie_ondemand == (64 + 128) * 6 * 64
    e = _engine(N=10, K=2, I=128, Ub=2)
    e.configure(CacheConfig(v_e=0.5, theta_i=[0.5], prefetch_rows_i=[40]))
    e.cache[0] = {7}
    e.predict_prefetch(0, rank)
    tr = e.step(0, np.array([[7, 1]]))
    assert dict(tr.act) == {7: BETA, 1: GAMMA}
    assert tr.pcie_ondemand == ((64 - 32) + 128) * 6 * 64
    # a whole bottom inside the window is alpha, as without a window; expert 3 with a 32-row
    # prefix of the full expert is gamma, loads 96 rows, is admitted (victim 0 -- 7 is in A)
    # and fills its slot's top rows on the device: d2d = 2 * I_top rows
    e = _engine(N=10, K=2, I=128, Ub=2)
    e.configure(CacheConfig(v_e=1.0, theta_i=[0.5], prefetch_rows_i=[100]))   # C = 2 -> {0, 1}
    e.cache[0] = {7, 0}
    e.predict_prefetch(0, rank)
    tr = e.step(0, np.array([[7, 3]]))
    assert dict(tr.act) == {7: ALPHA, 3: GAMMA} and tr.adm == [(3, 0)]
    assert tr.pcie_ondemand == (128 - 32) * 6 * 64


def test_window_rows_cross_pcie_once():
    """Conservation (any window, any policy): every non-resident row of an activated expert
    crosses PCIe exactly once -- on-demand bytes + the prefetched rows of activated experts
    = sum over A of (I - I_top if the top was cached else I) rows; and the plan never exceeds
    min(U_b I, W) rows."""
    rng = np.random.default_rng(17)
    N, K, I, g = 12, 3, 128, 16
    for W in (0, 16, 40, 100, 200, 1000):
        e = OracleEngine(2, N, K, 64, I, row_granule=g, buffer_experts=K)
        e.configure(CacheConfig(v_e=4.0, theta_i=[0.5, 0.75], prefetch_rows_i=[W, W], seed=3))
        for t in range(60):
            for i in range(2):
                ids = rng.choice(N, size=K, replace=False)[None]
                plan = e.pending if e.pending is not None and e.pending.target == i else None
                cached_before = set(e.cache[i]) if e.cache_on(i) else set()
                planned = {x: (f, r) for (x, f, r) in plan.items} if plan else {}
                tr = e.step(i, ids, (i + 1) % 2, rng.permutation(N))
                assert sum(r for (_, _, r) in e.pending.items) <= min(K * I, W)
                need = sum((I - e.I_top[i]) if x in cached_before else I for (x, _) in tr.act)
                pre = sum(planned[x][1] for (x, c) in tr.act if x in planned)
                assert tr.pcie_ondemand == (need - pre) * 6 * 64, (W, t, i)
