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


def test_q4_rejects_prefill_batches():
    from paper_2509_08342_b200 import api
    import ctypes
    d = api.model_desc(2, 8, 2, 256, 512, max_batch=64, weight_format=api.M.Q4G64)
    n = ctypes.c_size_t()
    assert api.M.moepic_arena_bytes(ctypes.byref(d), ctypes.byref(n)) == api.M.EINVAL
