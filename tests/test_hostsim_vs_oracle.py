"""T1: the library's C++ host control plane (through the C ABI, include/moepic_hostsim.h) vs
the oracle's state machine on random routing traces — bit-exact classes, admissions, plans,
byte counts, configurations (incl. Alg. 1) and cached sets.  No GPU needed."""
import numpy as np
import pytest

from oracle.replay import OracleEngine, CacheConfig
from oracle import policy as P

api = pytest.importorskip("paper_2509_08342_b200.api")


def _trace(rng, T, L, N, K, B, zipf=1.0, repeat=0.6):
    """Skewed, temporally local routing + noisy predicted rankings (SPEC S:105 style)."""
    pops = [rng.permutation(N) for _ in range(L)]
    w = 1.0 / np.arange(1, N + 1) ** zipf
    prev = [None] * L
    out = []
    for t in range(T):
        step = []
        for i in range(L):
            p = np.empty(N)
            p[pops[i]] = w
            p /= p.sum()
            ids = np.zeros((B, K), np.int32)
            for b in range(B):
                keep = [e for e in (prev[i][b] if prev[i] is not None else []) if rng.random() < repeat]
                rest = [e for e in rng.choice(N, size=N, replace=False, p=p) if e not in keep]
                ids[b] = (keep + rest)[:K]
            prev[i] = ids.copy()
            rank = np.argsort(-(np.log(p) + rng.gumbel(size=N) * 0.7), kind="stable").astype(np.int32)
            step.append((ids, rank))
        out.append(step)
    return out


def _run_pair(L, N, K, d, I, g, Ub, B, cfg_kw, T=40, seed=0, solver_at=None, solver_kw=None, n_shared=0):
    rng = np.random.default_rng(seed)
    desc = api.model_desc(L, N, K, d, I, n_shared=n_shared, row_granule=g, buffer_experts=Ub, max_batch=B,
                          v_e_max=L * N)
    hs = api.HostSim(desc)
    orc = OracleEngine(L, N, K, d, I, row_granule=g, buffer_experts=Ub, n_shared=n_shared)
    r1 = hs.configure(**cfg_kw)
    C, It, th, V = orc.configure(CacheConfig(**cfg_kw))
    assert r1["C_i"] == C and r1["I_top_i"] == It and r1["V_i"] == V
    tr = _trace(rng, T, L, N, K, B)
    predict = cfg_kw.get("prefetch", True)
    for t, step in enumerate(tr):
        if t == solver_at:
            kw = dict(cfg_kw, **solver_kw)
            a = hs.configure(**kw)
            C, It, th, V = orc.configure(CacheConfig(**kw))
            assert a["C_i"] == C and a["I_top_i"] == It and a["V_i"] == V, (a, C, It, V)
            for i in range(L):
                assert hs.cached(i) == orc.cache[i]
        for i, (ids, rank) in enumerate(step):
            nxt = (i + 1) % L
            x = hs.step(i, ids, nxt, rank) if predict else hs.step(i, ids)
            o = orc.step(i, ids, nxt, rank) if predict else orc.step(i, ids)
            assert x.act == o.act, (t, i)
            assert x.adm == o.adm, (t, i)
            assert x.plan == o.plan, (t, i)
            assert (x.pcie_ondemand, x.pcie_prefetch, x.hbm) == (o.pcie_ondemand, o.pcie_prefetch, o.hbm)
            assert hs.cached(i) == orc.cache[i]


@pytest.mark.parametrize("policy", [P.LCP, P.LRU, P.LFU, P.RND])
def test_toy_policies(policy):
    _run_pair(2, 8, 2, 64, 128, 16, 2, 1, dict(v_e=4.0, policy=policy, seed=3), T=80)


@pytest.mark.parametrize("theta", [0.25, 0.5, 1.0])
def test_theta_and_batch(theta):
    _run_pair(3, 16, 4, 64, 128, 16, 4, 4, dict(v_e=6.0, theta_i=[theta] * 3, seed=5), T=50, seed=1)


def test_prefetch_off_cache_only_and_prefetch_only():
    _run_pair(2, 8, 2, 64, 128, 16, 2, 1, dict(v_e=4.0, theta_i=[1.0, 1.0], prefetch=False), T=60, seed=2)
    _run_pair(2, 8, 2, 64, 128, 16, 2, 1, dict(v_e=0.0), T=60, seed=3)


def test_shared_experts_bytes():
    _run_pair(2, 16, 3, 64, 128, 16, 3, 2, dict(v_e=8.0, seed=9), T=30, seed=4, n_shared=2)


def test_solver_reconfigure_bit_exact():
    kw = dict(v_e=10.0, t_att=20.0, t_moe=40.0, t_head=10.0, t_load_exp=35.0, zeta=0.02)
    _run_pair(4, 16, 2, 64, 128, 16, 2, 1, kw, T=120, seed=6, solver_at=60,
              solver_kw=dict(use_solver=True))


def test_solver_qwen_like_shape():
    kw = dict(v_e=48.0, t_att=30.0, t_moe=25.0, t_head=10.0, t_load_exp=170.0, zeta=0.01, seed=11)
    _run_pair(6, 32, 4, 64, 192, 64, 4, 2, kw, T=60, seed=7, solver_at=40, solver_kw=dict(use_solver=True))


def test_invalid_configs_rejected():
    desc = api.model_desc(2, 8, 2, 64, 128, row_granule=16, v_e_max=8)
    hs = api.HostSim(desc)
    for bad in (dict(v_e=-1.0), dict(v_e=4.0, theta_i=[0.0, 0.5]), dict(v_e=4.0, theta_i=[1.5, 0.5]),
                dict(v_e=4.0, v_i=[3.0, 3.0]), dict(v_e=4.0, use_solver=True, t_load_exp=1.0, t_moe=1.0),
                dict(v_e=4.0, rho=1.5), dict(v_e=9.0)):
        with pytest.raises(api.MoEpicError):
            hs.configure(**bad)
    with pytest.raises(api.MoEpicError):
        api.HostSim(api.model_desc(2, 8, 8, 64, 128, row_granule=16))   # K must be < N


# randomised sweep (hypothesis): shapes, budgets, split ratios, policies, prefetch, buffer size,
# batch, shared experts and an Alg. 1 reconfiguration midway — every trace bit-exact
try:
    from hypothesis import given, settings, strategies as st, HealthCheck
except ImportError:   # pragma: no cover
    given = None

if given is not None:
    @settings(max_examples=80, deadline=None, suppress_health_check=[HealthCheck.too_slow])
    @given(L=st.integers(1, 4), N=st.sampled_from([4, 8, 16, 32]), kfrac=st.floats(0.05, 0.6),
           I=st.sampled_from([64, 128, 256]), B=st.integers(1, 4), policy=st.sampled_from([P.LCP, P.LRU, P.LFU, P.RND]),
           prefetch=st.booleans(), vfrac=st.floats(0.0, 1.0), theta=st.sampled_from([None, 0.25, 0.5, 0.75, 1.0]),
           ub_extra=st.integers(0, 2), n_shared=st.integers(0, 2), solver=st.booleans(), seed=st.integers(0, 10 ** 6),
           window=st.sampled_from([None, 0, 16, 80, 300]))
    def test_random_configurations(L, N, kfrac, I, B, policy, prefetch, vfrac, theta, ub_extra, n_shared, solver,
                                   seed, window):
        K = max(1, min(N - 1, int(round(kfrac * N))))
        v_e = round(vfrac * L * N, 2)
        kw = dict(v_e=v_e, policy=policy, prefetch=prefetch, seed=seed % 97)
        if window is not None:
            kw["prefetch_rows_i"] = [window] * L
        if theta is not None:
            kw["theta_i"] = [theta] * L
        skw = dict(use_solver=True, t_att=15.0, t_moe=30.0, t_head=5.0, t_load_exp=45.0, zeta=0.05)
        _run_pair(L, N, K, 64, I, 16, K + ub_extra, B, kw, T=24, seed=seed, n_shared=n_shared,
                  solver_at=8 if solver else None, solver_kw=skw)


def test_stats_checkpoint_round_trip():
    """SURVEY §5 checkpoint row: get_stats -> set_stats into a fresh control plane gives a
    bit-identical Alg. 1 configuration (run on the restored H/P/PH and counters) and
    identical traces afterwards, and both equal the oracle that never restarted."""
    L, N, K, I, g = 3, 16, 2, 128, 16
    rng = np.random.default_rng(31)
    desc = api.model_desc(L, N, K, 64, I, row_granule=g, buffer_experts=K, max_batch=2, v_e_max=L * N)
    a = api.HostSim(desc)
    orc = OracleEngine(L, N, K, 64, I, row_granule=g, buffer_experts=K)
    kw = dict(v_e=9.0, t_att=20.0, t_moe=40.0, t_head=10.0, t_load_exp=35.0, zeta=0.02, seed=4)
    a.configure(**kw)
    orc.configure(CacheConfig(**kw))
    tr = _trace(rng, 70, L, N, K, 2)
    for step in tr[:50]:
        for i, (ids, rank) in enumerate(step):
            a.step(i, ids, (i + 1) % L, rank)
            orc.step(i, ids, (i + 1) % L, rank)
    blob = a.get_stats()
    b = api.HostSim(desc)
    b.configure(**kw)
    b.set_stats(blob)
    assert b.get_stats() == blob
    skw = dict(kw, use_solver=True)
    ra, rb = a.configure(**skw), b.configure(**skw)
    C, It, th, V = orc.configure(CacheConfig(**skw))
    assert ra == rb
    assert ra["C_i"] == C and ra["I_top_i"] == It and ra["V_i"] == V
    for i in range(L):
        assert a.cached(i) == b.cached(i) == orc.cache[i]
    for step in tr[50:]:
        for i, (ids, rank) in enumerate(step):
            x, y = a.step(i, ids, (i + 1) % L, rank), b.step(i, ids, (i + 1) % L, rank)
            o = orc.step(i, ids, (i + 1) % L, rank)
            assert x.act == y.act == o.act and x.adm == y.adm == o.adm and x.plan == y.plan == o.plan
    # a snapshot of another shape is rejected without changing the target
    other = api.HostSim(api.model_desc(L, 8, K, 64, I, row_granule=g, max_batch=2, v_e_max=L * 8))
    with pytest.raises(api.MoEpicError):
        other.set_stats(blob)
    with pytest.raises(api.MoEpicError):
        b.set_stats(blob[:-8])


@pytest.mark.parametrize("W", [0, 16, 48, 200])
def test_window_plan_bit_exact(W):
    """Reading Q30: the window-capped plan (cut bottoms keep their prefix) -- C++ control plane
    equals the oracle, including with an Alg. 1 reconfiguration (the window then replaces Y)."""
    _run_pair(3, 16, 4, 64, 128, 16, 4, 2, dict(v_e=6.0, prefetch_rows_i=[W] * 3, seed=5), T=60, seed=8)
    kw = dict(v_e=10.0, t_att=20.0, t_moe=40.0, t_head=10.0, t_load_exp=35.0, zeta=0.02, prefetch_rows_i=[W] * 4)
    _run_pair(4, 16, 2, 64, 128, 16, 2, 1, kw, T=80, seed=6, solver_at=40, solver_kw=dict(use_solver=True))
