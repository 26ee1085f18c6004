"""GPU parity of the prefill path (B > 32 tokens: permute + tcgen05 grouped GEMMs + combine,
SURVEY §8(a) A12) against the fp64 oracle, through moepic_layer_forward.

Outputs: max|gpu - ref| / max|ref| <= 2e-3 (BASELINE north_star); routing and cache traces
bit-exact.  The intermediate SwiGLU activations are rounded to bf16 between the two GEMMs
(DESIGN.md §6), which the tolerance covers."""
import numpy as np
import pytest
import torch

import synth
from oracle import numeric as ON
from oracle.replay import OracleEngine, CacheConfig
from gpu_model import Model, rel_err, TOL

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    from paper_2509_08342_b200 import build
    build.build()


def _ctx(model, max_batch, v_e_max, renorm=1):
    from paper_2509_08342_b200 import api
    desc = api.model_desc(model.L, model.N, model.K, model.d, model.I, n_shared=model.n_shared, row_granule=64,
                          max_batch=max_batch, renorm_topk=renorm, L_host=model.L_host, v_e_max=v_e_max)
    ctx = api.MoEpic(desc)
    model.load_into(ctx)
    return ctx


@pytest.mark.parametrize("T,theta,v_e,n_shared", [(300, 0.5, 8.0, 0), (129, 0.25, 4.0, 0), (77, 1.0, 6.0, 0),
                                                  (200, 0.5, 0.0, 0), (160, 0.5, 8.0, 1)])
def test_prefill_small_shapes(T, theta, v_e, n_shared):
    from paper_2509_08342_b200 import api
    L, N, K, d, I = 2, 8, 2, 256, 512
    m = Model(L, N, K, d, I, n_shared=n_shared, seed=T)
    ctx = _ctx(m, max_batch=512, v_e_max=16.0)
    orc = OracleEngine(L, N, K, d, I, row_granule=64, n_shared=n_shared)
    cfg = dict(v_e=v_e, theta_i=[theta] * L, seed=3)
    ctx.configure(**cfg)
    orc.configure(CacheConfig(**cfg))
    H = synth.hidden_states(T, 2 * T, L, d)
    for step in range(2):
        for i in range(L):
            hb = synth.bf16_bits(H[step * T:(step + 1) * T, i])
            y = torch.empty(T, d, dtype=torch.float32, device="cuda")
            tr = ctx.layer_forward(i, H[step * T:(step + 1) * T, i].cuda(), y, flags=api.M.FUSE_PREDICT)
            torch.cuda.synchronize()
            y_ref, ids, w, _ = m.oracle_layer(i, hb)
            assert np.array_equal(tr.ids, ids)
            nxt = (i + 1) % L
            rank = ON.predicted_ranking(ON.router_logits(hb, m.routers[nxt]), K)
            o = orc.step(i, ids, nxt, rank)
            assert tr.act == o.act and tr.adm == o.adm and tr.plan == o.plan
            e = rel_err(y.cpu().numpy(), y_ref)
            assert e <= TOL, (step, i, e)
    ctx.close()


def test_prefill_mixtral_full_size_sampled():
    """BJ config 4 shape: Mixtral-shaped prefill, T = 2048, 50 % budget; the oracle evaluates a
    sample of 48 tokens (per-row GEMMs are independent, so every sampled row is exact)."""
    from paper_2509_08342_b200 import api
    S = synth.SHAPES["mixtral"]
    T = 2048
    m = Model(1, S.N, S.K, S.d, S.I, seed=0, gen_device="cuda")
    ctx = _ctx(m, max_batch=T, v_e_max=4.0)
    ctx.configure(v_e=4.0, seed=0)
    Hs = synth.batch_hidden(9, T, S.d)
    y = torch.empty(T, S.d, dtype=torch.float32, device="cuda")
    tr = ctx.layer_forward(0, Hs.cuda(), y, flags=0)
    torch.cuda.synchronize()
    sample = np.random.default_rng(0).choice(T, 48, replace=False)
    hb = synth.bf16_bits(Hs[sample])
    y_ref, ids, _, _ = m.oracle_layer(0, hb)
    assert np.array_equal(tr.ids[sample], ids)
    assert rel_err(y.cpu().numpy()[sample], y_ref) <= TOL
    ctx.close()
