"""GPU parity of the gated K2 launch (MOEPIC_K2_GATE).

With the gate (default on steps with >= 256 MB of K2 rows, MOEPIC_K2_GATE=2 on every step, as
here on small shapes) a decode step issues ONE K2 launch: the resident, prefetched and landed
on-demand rows now, and the tail of the step's last on-demand copy once the copy stream's flag
(written after that copy) arrives.  The gate changes when rows are streamed, never which rows or
how they are summed per (segment, CTA) partial -- so the traces are the oracle's bit for bit and y
is within the north_star bar, in every configuration that exercises it:
  * tiny auto tails (fewer tail rows than CTAs: CTAs with no gated rows),
  * a step whose only on-demand copy is small (toy shape),
  * a whole last copy as the tail (MOEPIC_OD_TAIL_KB), more rows than CTAs,
  * shared experts (DeepSeek), token masks with B > 1, Q4G64 rows, poison mode.
The gated and ungated runs must also agree with each other within fp32 rounding, and the gated
run must issue fewer kernel launches per step.
"""
import numpy as np
import pytest
import torch

import synth
from oracle.replay import OracleEngine, CacheConfig
from gpu_model import Model, rel_err, TOL

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    from paper_2509_08342_b200 import build
    build.build()


def _api():
    from paper_2509_08342_b200 import api
    return api


def _run(m, B, cfg, toks, q4=False, env=None, monkeypatch=None, g=64):
    """Replay toks through a fresh context; returns (ys, launches per step, oracle-checked)."""
    api = _api()
    for k, v in (env or {}).items():
        monkeypatch.setenv(k, v)
    desc = api.model_desc(m.L, m.N, m.K, m.d, m.I, n_shared=m.n_shared, row_granule=g, max_batch=B,
                          renorm_topk=1 if m.n_shared == 0 else 0, L_host=m.L_host, v_e_max=m.L * m.N,
                          weight_format=api.M.Q4G64 if q4 else api.M.BF16)
    ctx = api.MoEpic(desc)
    m.load_into(ctx)
    ctx.configure(**cfg)
    orc = OracleEngine(m.L, m.N, m.K, m.d, m.I, n_shared=m.n_shared, row_granule=g)
    if q4:
        from oracle import quant as Q
        orc.row_bytes = Q.packed_row_bytes(m.d)
    orc.configure(CacheConfig(**{k: v for k, v in cfg.items() if k in ("v_e", "theta_i", "seed")}))
    ys, launches = [], []
    stream = torch.cuda.Stream()
    for hl in toks:
        for i in range(m.L):
            h_bits = synth.bf16_bits(hl[i])
            y = torch.empty(hl[i].shape[0], m.d, dtype=torch.float32, device="cuda")
            tr = ctx.layer_forward(i, hl[i].to("cuda"), y, stream=stream, flags=api.M.FUSE_PREDICT)
            stream.synchronize()
            y_ref, ids, _, _ = m.oracle_layer(i, h_bits, renorm=m.n_shared == 0)
            assert np.array_equal(tr.ids, ids)
            from oracle import numeric as ON
            nxt = (i + 1) % m.L
            rank = ON.predicted_ranking(ON.router_logits(h_bits, m.routers[nxt]), m.K)
            o = orc.step(i, ids, nxt, rank)
            assert (tr.act, tr.adm, tr.plan) == (o.act, o.adm, o.plan)
            assert (tr.pcie_ondemand, tr.pcie_prefetch, tr.hbm) == (o.pcie_ondemand, o.pcie_prefetch, o.hbm)
            e = rel_err(y.cpu().numpy(), y_ref)
            assert e <= TOL, (i, e)
            ys.append(y.cpu().numpy())
            launches.append((tr.launches, tr.pcie_ondemand))
    for k in (env or {}):
        monkeypatch.delenv(k)
    ctx.close()
    return ys, launches


QWEN3 = (2, 128, 8, 2048, 768, 0)
CASES = [
    # (L, N, K, d, I, shared), B, budget (experts), q4, extra env
    (QWEN3, 1, 64.0, False, {}),                                  # auto tail < 148 rows
    (QWEN3, 4, 40.0, False, {}),                                  # token masks, K2's full block
    (QWEN3, 1, 64.0, False, {"MOEPIC_OD_TAIL_KB": "3000"}),       # whole last copy as tail: > 1 row per CTA
    ((2, 64, 6, 2048, 1408, 2), 2, 32.0, False, {}),              # DeepSeek: shared experts in phase 0
    ((2, 16, 4, 2048, 768, 0), 1, 8.0, True, {}),                 # Q4G64 rows
    ((2, 8, 2, 4096, 1024, 0), 1, 4.0, True, {}),                 # Q4G64, Mixtral-like hidden size
    (QWEN3, 1, 64.0, False, {"MOEPIC_POISON": "1"}),              # stale reads would turn y into NaN
    (QWEN3, 1, 0.0, False, {}),                                   # V = 0: every expert streamed
]


@pytest.mark.parametrize("dims,B,v_e,q4,env", CASES)
def test_gate_parity_vs_oracle_and_ungated(dims, B, v_e, q4, env, monkeypatch):
    L, N, K, d, I, ns = dims
    if q4:
        from test_gpu_q4 import Q4Model
        m = Q4Model(L, N, K, d, I, n_shared=ns, seed=7, gen_device="cuda")
    else:
        m = Model(L, N, K, d, I, n_shared=ns, seed=7, gen_device="cuda")
    H = synth.hidden_states(12, 4 * B, L, d)
    toks = [[H[t * B:(t + 1) * B, i] for i in range(L)] for t in range(4)]
    cfg = dict(v_e=v_e, seed=3)
    y_g, l_g = _run(m, B, cfg, toks, q4=q4, env={**env, "MOEPIC_K2_GATE": "2"}, monkeypatch=monkeypatch)
    y_u, l_u = _run(m, B, cfg, toks, q4=q4, env={**env, "MOEPIC_K2_GATE": "0"}, monkeypatch=monkeypatch)
    for a, b in zip(y_g, y_u):
        assert rel_err(a, b) <= 1e-5
    # the gate folds the tail launch into the step's single K2 launch
    assert sum(n for n, _ in l_g) < sum(n for n, _ in l_u), (l_g, l_u)


def test_gate_single_small_copy_is_the_tail(monkeypatch):
    """Toy shape, theta = 1, 4 of 8 experts cached: a missed expert is ONE small full-expert copy
    (the tail, whole): every step with an on-demand copy is the router and ONE K2 launch."""
    S = synth.SHAPES["toy"]
    m = Model(2, S.N, S.K, S.d, S.I, seed=2)
    H = synth.hidden_states(5, 8, 2, S.d)
    toks = [[H[t, i][None] for i in range(2)] for t in range(8)]
    cfg = dict(v_e=4.0, theta_i=[1.0, 1.0], seed=0)
    y_g, l_g = _run(m, 1, cfg, toks, env={"MOEPIC_K2_GATE": "2"}, monkeypatch=monkeypatch, g=16)
    y_u, l_u = _run(m, 1, cfg, toks, env={"MOEPIC_K2_GATE": "0"}, monkeypatch=monkeypatch, g=16)
    for a, b in zip(y_g, y_u):
        assert rel_err(a, b) <= 1e-5
    od = [n for n, b in l_g if b > 0]
    assert od and max(od) == 2, l_g   # router + one K2 launch
