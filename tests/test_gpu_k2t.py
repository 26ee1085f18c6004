"""K2T (kernels/expert_tc.cu): decode steps whose experts take more tokens than K2's 4-token block
run on the tcgen05 tensor cores, each weight row read once (SURVEY §8(a) A6/A7, §8(d) "each
weight read once").  Same bar as every decode parity test: routing / traces bit-exact against
the oracle replay, y within 2e-3 of the fp64 oracle layer (north_star)."""
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


def _run(monkeypatch, k2t, L, N, K, d, I, B, tokens, v_e, theta=0.5, n_shared=0, kappa=2.0, seed=0,
         renorm=1):
    from paper_2509_08342_b200 import api
    monkeypatch.setenv("MOEPIC_K2T", "1" if k2t else "0")
    m = Model(L, N, K, d, I, n_shared=n_shared, seed=seed, kappa=kappa, gen_device="cuda")
    desc = api.model_desc(L, N, K, d, I, n_shared=n_shared, row_granule=64, max_batch=B, renorm_topk=renorm,
                          v_e_max=float(L * N))
    ctx = api.MoEpic(desc)
    m.load_into(ctx)
    orc = OracleEngine(L, N, K, d, I, n_shared=n_shared)
    cfg = dict(v_e=v_e, theta_i=[theta] * L, seed=1)
    ctx.configure(**cfg)
    orc.configure(CacheConfig(**cfg))
    H = synth.hidden_states(seed + 3, tokens * B, L, d)
    stream = torch.cuda.Stream()
    ctx.profile(True)
    worst, ys, hot = 0.0, [], 0
    from oracle import numeric as ON
    for t in range(tokens):
        for i in range(L):
            hl = H[t * B:(t + 1) * B, i]
            hb = synth.bf16_bits(hl)
            y = torch.empty(B, d, dtype=torch.float32, device="cuda")
            tr = ctx.layer_forward(i, hl.to("cuda"), y, stream=stream, flags=api.M.FUSE_PREDICT)
            stream.synchronize()
            y_ref, ids, w, _ = m.oracle_layer(i, hb, renorm=bool(renorm))
            assert np.array_equal(tr.ids, ids)
            nxt = (i + 1) % L
            rank = ON.predicted_ranking(ON.router_logits(hb, m.routers[nxt]), K)
            o = orc.step(i, ids, nxt, rank)
            assert (tr.act, tr.adm, tr.plan) == (o.act, o.adm, o.plan)
            assert (tr.pcie_ondemand, tr.pcie_prefetch, tr.hbm) == (o.pcie_ondemand, o.pcie_prefetch, o.hbm)
            e = rel_err(y.cpu().numpy(), y_ref)
            worst = max(worst, e)
            assert e <= TOL, (t, i, e)
            ys.append(y.cpu().numpy())
            hot += int(np.bincount(ids.ravel(), minlength=N).max() > 4)
    k2 = ctx.profile_read(api.M.KERNEL_EXPERT)
    ctx.close()
    return worst, ys, k2, hot


@pytest.mark.parametrize("B", [8, 12, 16])
def test_k2t_parity_and_single_read(monkeypatch, B):
    """d 256, I 512, 16 experts top-4 with concentrated routing: hot experts get > 4 tokens.
    K2T and K2 both match the oracle; K2T streams fewer algorithmic bytes (no per-group re-read)."""
    args = dict(L=2, N=16, K=4, d=256, I=512, B=B, tokens=3, v_e=16.0, kappa=4.0)
    w_t, y_t, k_t, hot = _run(monkeypatch, True, **args)
    w_k, y_k, k_k, _ = _run(monkeypatch, False, **args)
    assert hot > 0, "the inputs must route more than 4 tokens to some expert"
    assert w_t <= TOL and w_k <= TOL
    for a, b in zip(y_t, y_k):   # the two kernels sum in different orders: within the parity bar
        assert float(np.abs(a - b).max() / np.abs(b).max()) <= TOL
    assert k_t["bytes"] < k_k["bytes"], (k_t, k_k)


@pytest.mark.parametrize("theta,v_e", [(0.5, 64.0), (1.0, 24.0), (0.25, 96.0)])
def test_k2t_qwen3_batch16(monkeypatch, theta, v_e):
    """BJ config 2 at B = 16: tops, bottoms, on-demand experts and odd unit counts per CTA."""
    S = synth.SHAPES["qwen3"]
    w, _, k, hot = _run(monkeypatch, True, L=2, N=S.N, K=S.K, d=S.d, I=S.I, B=16, tokens=2, v_e=v_e, theta=theta,
                        kappa=1.0)
    assert hot > 0 and w <= TOL


def test_k2t_deepseek_shared_experts(monkeypatch):
    """Shared experts (weight 1, every token) go through K2T's expert < 0 path; renorm off (Q4)."""
    S = synth.SHAPES["deepseek"]
    w, _, _, _ = _run(monkeypatch, True, L=2, N=S.N, K=S.K, d=S.d, I=S.I, B=8, tokens=2, v_e=32.0, n_shared=2,
                      renorm=0, kappa=1.0)
    assert w <= TOL


def test_k2t_poison_mode(monkeypatch):
    """A stale or unlanded segment read under MOEPIC_POISON would turn y into NaN."""
    monkeypatch.setenv("MOEPIC_POISON", "1")
    w, ys, _, _ = _run(monkeypatch, True, L=2, N=16, K=4, d=256, I=512, B=12, tokens=3, v_e=8.0)
    assert w <= TOL and all(np.isfinite(y).all() for y in ys)
