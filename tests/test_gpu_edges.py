"""GPU edge cases through the C ABI: decode at the largest batch (32 tokens, token masks full),
the smallest prefill batch (33), prefill of a DeepSeek-shaped layer with shared experts and
no renormalisation, a ragged expert tail (I not a multiple of the 128-row GEMM tile), and a
pending prefetch invalidated by configure."""
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


def _run(m, ctx, orc, H, B, steps, renorm=True, flags=None):
    from paper_2509_08342_b200 import api
    flags = api.M.FUSE_PREDICT if flags is None else flags
    for t in range(steps):
        for i in range(m.L):
            h = H[t * B:(t + 1) * B, i]
            hb = synth.bf16_bits(h)
            y = torch.empty(B, m.d, dtype=torch.float32, device="cuda")
            tr = ctx.layer_forward(i, h.cuda(), y, flags=flags)
            torch.cuda.synchronize()
            y_ref, ids, _, _ = m.oracle_layer(i, hb, renorm=renorm)
            assert np.array_equal(tr.ids, ids)
            nxt = (i + 1) % m.L
            rank = ON.predicted_ranking(ON.router_logits(hb, m.routers[nxt]), m.K) if flags else None
            o = orc.step(i, ids, nxt if flags else None, rank)
            assert tr.act == o.act and tr.adm == o.adm and tr.plan == o.plan
            assert rel_err(y.cpu().numpy(), y_ref) <= TOL


def _ctx(m, max_batch, v_e_max, renorm=1, g=64):
    from paper_2509_08342_b200 import api
    desc = api.model_desc(m.L, m.N, m.K, m.d, m.I, n_shared=m.n_shared, row_granule=g, max_batch=max_batch,
                          renorm_topk=renorm, L_host=m.L_host, v_e_max=v_e_max)
    ctx = api.MoEpic(desc)
    m.load_into(ctx)
    return ctx


def test_decode_max_batch_32():
    m = Model(2, 16, 4, 256, 256, seed=12)
    ctx = _ctx(m, 32, 8.0)
    orc = OracleEngine(2, 16, 4, 256, 256)
    cfg = dict(v_e=8.0, seed=3)
    ctx.configure(**cfg)
    orc.configure(CacheConfig(**cfg))
    _run(m, ctx, orc, synth.hidden_states(5, 64, 2, 256), 32, 2)


@pytest.mark.parametrize("T", [33, 130])
def test_prefill_smallest_batches(T):
    m = Model(2, 8, 2, 256, 512, seed=T)
    ctx = _ctx(m, 256, 8.0)
    orc = OracleEngine(2, 8, 2, 256, 512)
    cfg = dict(v_e=6.0, theta_i=[0.5, 0.75], seed=2)
    ctx.configure(**cfg)
    orc.configure(CacheConfig(**cfg))
    _run(m, ctx, orc, synth.hidden_states(T, 2 * T, 2, 256), T, 2)


def test_prefill_deepseek_shape_shared():
    """DeepSeek-V2-Lite-shaped prefill (d 2048, I 1408 -> 11 row tiles of 128: a ragged last
    tile), 2 shared experts, renormalisation off, 256 tokens."""
    S = synth.SHAPES["deepseek"]
    m = Model(1, S.N, S.K, S.d, S.I, n_shared=2, seed=1, gen_device="cuda")
    ctx = _ctx(m, 256, 32.0, renorm=0)
    orc = OracleEngine(1, S.N, S.K, S.d, S.I, n_shared=2)
    cfg = dict(v_e=32.0, seed=5)
    ctx.configure(**cfg)
    orc.configure(CacheConfig(**cfg))
    _run(m, ctx, orc, synth.hidden_states(8, 256, 1, S.d), 256, 1, renorm=False)


def test_configure_drops_pending_prefetch():
    from paper_2509_08342_b200 import api
    m = Model(2, 8, 2, 128, 256, seed=4)
    ctx = _ctx(m, 1, 8.0)
    orc = OracleEngine(2, 8, 2, 128, 256)
    cfg = dict(v_e=2.0, seed=0)
    ctx.configure(**cfg)
    orc.configure(CacheConfig(**cfg))
    H = synth.hidden_states(3, 4, 2, 128)
    hp = H[0, 1][None]
    ctx.predict_prefetch(0, hp.cuda())
    rank = ON.predicted_ranking(ON.router_logits(synth.bf16_bits(hp), m.routers[0]), 2)
    orc.predict_prefetch(0, rank)
    cfg2 = dict(v_e=4.0, theta_i=[0.25, 0.25], seed=0)   # re-layout: the plan must be dropped
    ctx.configure(**cfg2)
    orc.configure(CacheConfig(**cfg2))
    _run(m, ctx, orc, H[1:], 1, 3)


def test_prefill_qwen3_shape_two_chunks():
    """Qwen3-shaped prefill (N = 128, K = 8, d 2048, I 768): the large-batch router selection
    (k1_select, one warp per token, kMaxN = 128 experts), 128 segment tensor maps in one GEMM
    launch, single-CTA tiles (one 128-row tile per expert), partial cache (C < N)."""
    S = synth.SHAPES["qwen3"]
    m = Model(1, S.N, S.K, S.d, S.I, seed=9, gen_device="cuda")
    ctx = _ctx(m, 512, 128.0)
    orc = OracleEngine(1, S.N, S.K, S.d, S.I)
    cfg = dict(v_e=48.0, seed=4)
    ctx.configure(**cfg)
    orc.configure(CacheConfig(**cfg))
    _run(m, ctx, orc, synth.hidden_states(21, 2 * 384, 1, S.d), 384, 2)
