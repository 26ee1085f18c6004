"""Attention stand-in: oracle pins on CPU, GPU parity through the C ABI.

Pins of oracle/numeric.attention_decode: S = 1 returns v_0 exactly; equal keys give the mean of
the values; the general case equals torch's scaled_dot_product_attention (fp64, KV heads
repeated for the query groups)."""
import numpy as np
import pytest
import torch

import synth
from oracle import numeric as ON


def _rand(shape, seed, scale=1.0):
    g = torch.Generator().manual_seed(seed)
    return synth.bf16_bits((torch.randn(*shape, generator=g) * scale).to(torch.bfloat16))


def test_single_position_returns_value():
    q, k, v = _rand((2, 8, 128), 1), _rand((2, 4, 2, 128), 2), _rand((2, 4, 2, 128), 3)
    out = ON.attention_decode(q, k, v, 1)
    for h in range(8):
        np.testing.assert_array_equal(out[:, h], ON.bf16_to_f64(v)[:, 0, h // 4])


def test_equal_keys_average_values():
    q, v = _rand((1, 4, 128), 4), _rand((1, 9, 2, 128), 5)
    k = np.tile(_rand((1, 1, 2, 128), 6), (1, 9, 1, 1))
    out = ON.attention_decode(q, k, v, 9)
    ref = ON.bf16_to_f64(v)[0].mean(axis=0)          # [Hkv][dh]
    for h in range(4):
        np.testing.assert_allclose(out[0, h], ref[h // 2], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("B,S,Hq,Hkv", [(1, 37, 8, 2), (3, 300, 4, 4), (2, 513, 16, 1)])
def test_matches_torch_sdpa(B, S, Hq, Hkv):
    q, k, v = _rand((B, Hq, 128), 7), _rand((B, S + 5, Hkv, 128), 8), _rand((B, S + 5, Hkv, 128), 9)
    out = ON.attention_decode(q, k, v, S)
    f = lambda a: torch.from_numpy(ON.bf16_to_f64(a))
    G = Hq // Hkv
    kk = f(k)[:, :S].permute(0, 2, 1, 3).repeat_interleave(G, dim=1)    # [B][Hq][S][dh]
    vv = f(v)[:, :S].permute(0, 2, 1, 3).repeat_interleave(G, dim=1)
    ref = torch.nn.functional.scaled_dot_product_attention(f(q)[:, :, None], kk, vv)[:, :, 0]
    np.testing.assert_allclose(out, ref.numpy(), rtol=1e-10, atol=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("B,S,S_max,Hq,Hkv", [(1, 1, 64, 32, 8), (1, 4096, 4096, 32, 8), (4, 1000, 1024, 32, 4),
                                             (2, 257, 300, 16, 16), (16, 511, 512, 32, 8)])
def test_gpu_attention_parity(B, S, S_max, Hq, Hkv):
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    from paper_2509_08342_b200 import api
    q, k, v = _rand((B, Hq, 128), 11, 0.5), _rand((B, S_max, Hkv, 128), 12), _rand((B, S_max, Hkv, 128), 13)
    dev = lambda a: synth.bits_to_bf16(a).cuda()
    out = torch.empty(B, Hq, 128, dtype=torch.float32, device="cuda")
    att = api.Attention(B, S_max, Hq, Hkv)
    att(dev(q), dev(k), dev(v), S, out)
    torch.cuda.synchronize()
    ref = ON.attention_decode(q, k, v, S)
    err = float(np.abs(out.cpu().numpy() - ref).max() / np.abs(ref).max())
    assert err <= 2e-3, err
