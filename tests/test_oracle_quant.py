"""Pins for oracle/quant.py (Q4G64 low-bit experts; reading Q28)
against things other than itself: a closed-form group, brute-force nearest-level search, the
round-down / round-up definitions of lo_b and s_b checked against bf16 neighbours, the
error bound, and the byte layout (unpacked by hand)."""
import numpy as np
import pytest
import torch

import synth
from oracle import numeric as ON
from oracle import quant as Q


def _f(bits):
    return ON.bf16_to_f64(bits)


def _bits_of(vals):
    return synth.bf16_bits(torch.tensor(vals, dtype=torch.float32).to(torch.bfloat16))


def test_equally_spaced_group_is_exact():
    """x_k = k/16 for k = 0..15 repeated: lo = 0, hi = 15/16, s = 1/16 exactly; codes = k."""
    vals = np.tile(np.arange(16) / 16.0, 4)
    q, s, lo = Q.quantize_vector(_bits_of(vals))
    assert list(q) == list(np.tile(np.arange(16), 4))
    assert _f(s)[0] == 1 / 16 and _f(lo)[0] == 0.0
    np.testing.assert_array_equal(Q.dequantize_vector(q, s, lo), vals)


def test_constant_group_scale_one():
    q, s, lo = Q.quantize_vector(_bits_of([0.375] * 64))
    assert np.all(q == 0) and _f(s)[0] == 1.0 and _f(lo)[0] == 0.375


@pytest.mark.parametrize("seed", range(4))
def test_bf16_rounding_directions_and_brute_force_levels(seed):
    g = torch.Generator().manual_seed(seed)
    x = (torch.randn(64 * 32, generator=g) * (0.02 if seed % 2 else 3.0)).to(torch.bfloat16)
    bits = synth.bf16_bits(x)
    q, s, lo = Q.quantize_vector(bits)
    xv = _f(bits).reshape(-1, 64)
    sv, lov = _f(s), _f(lo)
    for gi in range(xv.shape[0]):
        mn, mx = xv[gi].min(), xv[gi].max()
        # lo_b: a bf16 value <= min whose upper bf16 neighbour is > min
        assert lov[gi] <= mn
        b = int(lo[gi])
        nb = b + 1 if (lov[gi] > 0 or b == 0) else (1 if b == 0x8000 else b - 1)
        assert _f(np.array([nb], np.uint16))[0] > mn
        # s_b >= (max - lo_b) / 15 (up to the fp32 division), and the next bf16 below is not
        t = (mx - lov[gi]) / 15
        assert sv[gi] >= t * (1 - 2 ** -22)
        below = _f(np.array([int(s[gi]) - 1], np.uint16))[0]
        assert below < t * (1 + 2 ** -22)
        # every code is the nearest of the 16 levels (brute force), except fp32 near-ties
        levels = lov[gi] + np.arange(16) * sv[gi]
        for k in range(64):
            dist = np.abs(levels - xv[gi, k])
            best = int(np.argmin(dist))
            qk = int(q[gi * 64 + k])
            if qk != best:
                assert abs(dist[qk] - dist[best]) <= 2 ** -20 * sv[gi], (gi, k, qk, best)
        err = np.abs(Q.dequantize_vector(q[gi * 64:(gi + 1) * 64], s[gi:gi + 1], lo[gi:gi + 1]) - xv[gi])
        assert err.max() <= sv[gi] / 2 * (1 + 2 ** -20)


def test_packed_layout_by_hand():
    g = torch.Generator().manual_seed(9)
    d, I = 128, 3
    gate, up = (synth.bf16_bits(torch.randn(I, d, generator=g).to(torch.bfloat16)) for _ in range(2))
    down = synth.bf16_bits(torch.randn(d, I, generator=g).to(torch.bfloat16))
    qe = Q.quantize_expert(gate, up, down)
    img = Q.pack_expert(qe)
    assert img.shape == (I, Q.packed_row_bytes(d)) and Q.packed_row_bytes(d) % 16 == 0
    for r in range(I):
        for part in range(3):
            codes = img[r, part * 64:(part + 1) * 64]
            un = np.empty(d, np.uint8)
            un[0::2], un[1::2] = codes & 15, codes >> 4
            assert np.array_equal(un, qe["q"][r, part])
            pr = img[r, 192 + part * 8:192 + (part + 1) * 8].view(np.uint16)
            assert np.array_equal(pr[0::2], qe["s"][r, part]) and np.array_equal(pr[1::2], qe["lo"][r, part])
        assert np.all(img[r, 192 + 24:] == 0)


def test_dequantised_layer_is_close_to_bf16_layer():
    """Context (not a parity pin): the Q4G64 layer stays within a few percent of the bf16 one
    on the synthetic recipe, so the format is a usable low-bit mode."""
    N, d, I, K = 8, 128, 64, 2
    router = synth.bf16_bits(synth.router_weights(2, 0, N, d))
    experts = [tuple(synth.bf16_bits(x) for x in synth.expert_weights(2, 0, e, d, I)) for e in range(N)]
    deq = [Q.dequantize_expert(Q.quantize_expert(*w)) for w in experts]
    h = synth.bf16_bits(synth.batch_hidden(2, 5, d))
    y, _, _, _ = ON.moe_layer(h, router, experts, K)
    yq, _, _, _ = ON.moe_layer(h, router, deq, K)
    rel = np.abs(yq - y).max() / np.abs(y).max()
    assert 1e-4 < rel < 0.2, rel


@pytest.mark.parametrize("d,I,tp", [(128, 64, 1), (256, 128, 2), (4096, 16, 1)])
def test_library_packer_matches_oracle_bit_for_bit(d, I, tp):
    """moepic_pack_expert (host C++, the path load_expert uses) against oracle/quant.py: every
    code and every group parameter identical, for each tensor-parallel slice."""
    from paper_2509_08342_b200 import api
    g = torch.Generator().manual_seed(d + I)
    gate = synth.bf16_bits((torch.randn(I, d, generator=g) * 0.05).to(torch.bfloat16))
    up = synth.bf16_bits((torch.randn(I, d, generator=g) * 0.05).to(torch.bfloat16))
    down = synth.bf16_bits((torch.randn(d, I, generator=g) * 0.1).to(torch.bfloat16))
    qe = Q.quantize_expert(gate, up, down)
    ref = Q.pack_expert(qe)
    for r in range(tp):
        desc = api.model_desc(1, 4, 2, d, I, row_granule=16, tp_rank=r, tp_size=tp, weight_format=api.M.Q4G64)
        img = api.pack_expert(desc, gate, up, down).reshape(I // tp, -1)
        assert np.array_equal(img, ref[r * I // tp:(r + 1) * I // tp])
    # bf16 format: the interleaved rows [gate_r | up_r | down[:, r]], the down column as fp16
    # (reading Q31): numpy's IEEE round-to-nearest-even float16 conversion of the bf16 values
    desc = api.model_desc(1, 4, 2, d, I, row_granule=16)
    img = api.pack_expert(desc, gate, up, down).view(np.uint16).reshape(I, 3, d)
    down_f16 = synth.bits_to_bf16(np.ascontiguousarray(down.T)).float().numpy().astype(np.float16).view(np.uint16)
    assert np.array_equal(img[:, 0], gate) and np.array_equal(img[:, 1], up) and np.array_equal(img[:, 2], down_f16)


def test_down_column_fp16_reencoding():
    """Reading Q31: the stored down column is fp16.  Pins of the host packer's bf16 -> fp16
    conversion: exact (round trip) over the whole bf16 range [2^-14, 65280] of both signs;
    round-to-nearest-even subnormals below 2^-14 against numpy; +-0 kept; |x| >= 65536 rejected."""
    from paper_2509_08342_b200 import api
    allb = np.arange(1 << 16, dtype=np.uint32).astype(np.uint16)
    fin = allb[(allb & 0x7FFF) < 0x4780]                                # every bf16 fp16 can hold
    d, I = 64, len(fin) // 64 // 16 * 16
    fin = fin[:d * I]
    down = np.ascontiguousarray(fin.reshape(I, d).T)                    # [d][I]: column r = row r
    z = np.zeros((I, d), np.uint16)
    desc = api.model_desc(1, 4, 2, d, I, row_granule=16)
    img = api.pack_expert(desc, z, z, down).view(np.uint16).reshape(I, 3, d)[:, 2].ravel()
    x = synth.bits_to_bf16(fin).float().numpy()
    ref = x.astype(np.float16)
    assert np.array_equal(img, ref.view(np.uint16))
    normal = np.abs(x) >= 2.0 ** -14
    assert np.array_equal(ref[normal].astype(np.float32), x[normal])     # exact where fp16 is normal
    assert np.abs(ref.astype(np.float64) - x)[~normal].max() <= 2.0 ** -25
    bad = down.copy()
    bad[0, 0] = 0x4780                                                   # 65536: does not fit
    with pytest.raises(Exception):
        api.pack_expert(desc, z, z, bad)
