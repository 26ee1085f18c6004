"""Q4G64 low-bit experts on the GPU (reading Q28).

The library quantises at load_expert (host, bit-identical to oracle/quant.py, pinned in
test_oracle_quant.py) and K2 dequantises on the fly.  Against the oracle layer over the SAME
dequantised weights: routing / rankings / cache traces bit-exact, byte counters with the packed
row size, outputs within 2e-3."""
import numpy as np
import pytest
import torch

import synth
from oracle import quant as Q
from oracle.replay import OracleEngine, CacheConfig
from gpu_model import Model, TOL
from test_gpu_parity import _replay

pytestmark = pytest.mark.gpu


class Q4Model(Model):
    """Same synthetic weights; the oracle sees the dequantised Q4G64 experts."""

    def __init__(self, *a, **kw):
        super().__init__(*a, **kw)
        self.deq = {k: Q.dequantize_expert(Q.quantize_expert(*w)) for k, w in self.experts.items()}
        self.deq_shared = {k: Q.dequantize_expert(Q.quantize_expert(*w)) for k, w in self.shared.items()}

    def oracle_layer(self, layer, h_bits, renorm=True):
        from oracle import numeric as ON
        shared = [self.deq_shared[(layer, s)] for s in range(self.n_shared)]
        return ON.moe_layer(h_bits, self.routers[layer], lambda e: self.deq[(layer % self.L_host, e)], self.K,
                            shared=shared, renorm=renorm)


@pytest.mark.parametrize("L,N,K,d,I,ns,B,theta,v_e", [
    (2, 8, 2, 256, 512, 1, 1, 0.5, 4.0),      # CW 4, RS 16; shared expert; beta / gamma / prefetch
    (2, 8, 2, 256, 512, 1, 3, 0.75, 6.0),     # token groups
    (2, 16, 4, 2048, 768, 0, 1, 0.5, 8.0),    # Qwen3-like hidden size: CW 4, RS 8
    (2, 16, 4, 2048, 768, 0, 4, 0.5, 8.0),
    (2, 8, 2, 4096, 1024, 0, 1, 0.5, 8.0),    # Mixtral-like hidden size: CW 8, RS 4
])
def test_q4_decode_parity(L, N, K, d, I, ns, B, theta, v_e):
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    from paper_2509_08342_b200 import api
    m = Q4Model(L, N, K, d, I, n_shared=ns, seed=d + B, gen_device="cuda")
    desc = api.model_desc(L, N, K, d, I, n_shared=ns, row_granule=64, max_batch=B, v_e_max=float(L * N),
                          weight_format=api.M.Q4G64)
    ctx = api.MoEpic(desc)
    m.load_into(ctx)
    orc = OracleEngine(L, N, K, d, I, row_granule=64, n_shared=ns)
    orc.row_bytes = Q.packed_row_bytes(d)
    cfg = dict(v_e=v_e, theta_i=[theta] * L, seed=3)
    assert ctx.configure(**cfg)["C_i"] == list(orc.configure(CacheConfig(**cfg))[0])
    H = synth.hidden_states(d + B, 4 * B, L, d)
    toks = [[H[t * B:(t + 1) * B, i] for i in range(L)] for t in range(4)]
    worst = _replay(m, ctx, orc, toks, api.M.FUSE_PREDICT)
    assert worst <= TOL
    ctx.close()


@pytest.mark.parametrize("T,theta,v_e,ns", [(64, 0.5, 8.0, 0), (129, 0.25, 4.0, 1), (300, 1.0, 6.0, 0),
                                            (200, 0.5, 0.0, 0)])
def test_q4_prefill_parity(T, theta, v_e, ns):
    """NEXT-3 on the prefill path (reading Q32): Q4G64 segments dequantised to fp16 rows, X in fp16,
    the tcgen05 GEMMs in kind::f16.  Against the oracle layer over the dequantised weights:
    routing and cache traces bit-exact, outputs within 2e-3; tops, bottoms, prefetched and
    on-demand groups, ragged expert blocks, a shared expert."""
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    from paper_2509_08342_b200 import api
    from oracle import numeric as ON
    from gpu_model import rel_err
    L, N, K, d, I = 2, 8, 2, 256, 512
    m = Q4Model(L, N, K, d, I, n_shared=ns, seed=T, gen_device="cuda")
    desc = api.model_desc(L, N, K, d, I, n_shared=ns, row_granule=64, max_batch=512, v_e_max=16.0,
                          weight_format=api.M.Q4G64)
    ctx = api.MoEpic(desc)
    m.load_into(ctx)
    orc = OracleEngine(L, N, K, d, I, row_granule=64, n_shared=ns)
    orc.row_bytes = Q.packed_row_bytes(d)
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
            y_ref, ids, _, _ = m.oracle_layer(i, hb)
            assert np.array_equal(tr.ids, ids)
            nxt = (i + 1) % L
            rank = ON.predicted_ranking(ON.router_logits(hb, m.routers[nxt]), K)
            o = orc.step(i, ids, nxt, rank)
            assert tr.act == o.act and tr.adm == o.adm and tr.plan == o.plan
            assert (tr.pcie_ondemand, tr.pcie_prefetch) == (o.pcie_ondemand, o.pcie_prefetch)
            e = rel_err(y.cpu().numpy(), y_ref)
            assert e <= TOL, (step, i, e)
    ctx.close()


def test_q4_prefill_mixtral_hidden_sampled():
    """BJ config 4 (Mixtral hidden size 4096, 8 experts top-2, T = 2048) with Q4G64 experts of
    I = 2048 rows (the oracle quantises in numpy), 25 % budget, 32 sampled rows against the oracle
    over the dequantised weights."""
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    from paper_2509_08342_b200 import api
    from gpu_model import rel_err
    S = synth.SHAPES["mixtral"]
    T = 2048
    I = 2048
    m = Q4Model(1, S.N, S.K, S.d, I, seed=0, gen_device="cuda")
    desc = api.model_desc(1, S.N, S.K, S.d, I, row_granule=64, max_batch=T, v_e_max=2.0,
                          weight_format=api.M.Q4G64)
    ctx = api.MoEpic(desc)
    m.load_into(ctx)
    ctx.configure(v_e=2.0, seed=0)
    Hs = synth.batch_hidden(9, T, S.d)
    y = torch.empty(T, S.d, dtype=torch.float32, device="cuda")
    tr = ctx.layer_forward(0, Hs.cuda(), y, flags=0)
    torch.cuda.synchronize()
    sample = np.random.default_rng(1).choice(T, 32, replace=False)
    hb = synth.bf16_bits(Hs[sample])
    y_ref, ids, _, _ = m.oracle_layer(0, hb)
    assert np.array_equal(tr.ids[sample], ids)
    assert rel_err(y.cpu().numpy()[sample], y_ref) <= TOL
    ctx.close()
