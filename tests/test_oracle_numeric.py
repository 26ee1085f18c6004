"""Pins for oracle/numeric.py against things other than itself.

C-P1 split identity (linearity over I)     C-P2 Eq. 2 renormalisation
C-P3 brute-force top-K                            C-P4 exact rational router logits
C-P5 special cases that reduce to library MoE blocks (HF transformers Mixtral / Qwen3-MoE
     / DeepSeek-V2) and a closed-form SwiGLU example.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest
import torch

import synth
from oracle import numeric as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _bits(t):
    return synth.bf16_bits(t)


def _toy_layer(seed=0, N=8, d=64, I=128, B=16):
    router = _bits(synth.router_weights(seed, 0, N, d))
    experts = [tuple(_bits(x) for x in synth.expert_weights(seed, 0, e, d, I)) for e in range(N)]
    h = _bits(synth.hidden_states(seed, B, 1, d)[:, 0, :])
    return h, router, experts


# ----------------------------------------------------------------- C-P4 router logits
def test_router_logits_exact_rational_toy():
    h, router, _ = _toy_layer()
    lg = O.router_logits(h, router)
    hf = O.bf16_to_f64(h)
    wf = O.bf16_to_f64(router)
    for b in range(4):
        exact = []
        for j in range(router.shape[0]):
            s = sum(Fraction(float(x)) * Fraction(float(y)) for x, y in zip(hf[b], wf[j]))
            exact.append(s)
            absmax = sum(abs(Fraction(float(x)) * Fraction(float(y))) for x, y in zip(hf[b], wf[j]))
            # error bound of any fp64 summation order of d exact terms: (d-1) u sum|p|
            assert abs(Fraction(lg[b, j]) - s) <= Fraction(h.shape[1]) * Fraction(2.0 ** -53) * absmax
        # the canonical top-K equals the exact top-K (gaps are >> 1e-12 here)
        ex_order = sorted(range(len(exact)), key=lambda j: (-exact[j], j))
        assert list(O.topk_ids(lg[b], 2)) == ex_order[:2]


def test_router_canonical_order_golden():
    g = json.load(open(os.path.join(GOLD, "router_canonical_order.json")))
    d = g["d"]
    h = np.zeros((1, d), dtype=np.float32)
    w = np.zeros((1, d), dtype=np.float32)
    h[0, 0], w[0, 0] = 2.0 ** 27, 2.0 ** 26
    h[0, 8], w[0, 8] = -(2.0 ** 27), 2.0 ** 26
    h[0, 16], w[0, 16] = 1.0, 1.0
    hb = (h.view(np.uint32) >> 16).astype(np.uint16)
    wb = (w.view(np.uint32) >> 16).astype(np.uint16)
    assert O.router_logits(hb, wb)[0, 0] == g["canonical_logit"]
    assert math.fsum((h[0].astype(np.float64) * w[0].astype(np.float64)).tolist()) == g["exact_sum"]


# ----------------------------------------------------------------- C-P3 / C-P2
def test_topk_brute_force():
    rng = np.random.default_rng(1)
    for _ in range(200):
        N = int(rng.integers(2, 40))
        K = int(rng.integers(1, N))
        l = rng.integers(-5, 5, size=N).astype(np.float64)   # many ties -> id tie-break
        ids = O.topk_ids(l, K)
        keys = np.lexsort((np.arange(N), -l))               # primary -l, secondary id
        assert list(ids) == list(keys[:K])


def test_gate_weights_eq2():
    rng = np.random.default_rng(2)
    for _ in range(100):
        N = 16
        l = rng.normal(size=N) * 3
        ids = O.topk_ids(l, 4)
        w = O.gate_weights(l, ids, True)
        assert abs(w.sum() - 1.0) < 1e-15
        s = np.exp(l) / np.exp(l).sum()                       # softmax over all N
        ref = s[ids] / s[ids].sum()                           # Eq. 2 literal form
        np.testing.assert_allclose(w, ref, rtol=1e-13)
        np.testing.assert_allclose(O.gate_weights(l, ids, False), s[ids], rtol=1e-13)


# ----------------------------------------------------------------- C-P5 SwiGLU
def test_swiglu_closed_form_golden():
    g = json.load(open(os.path.join(GOLD, "swiglu_closed_form.json")))
    h = np.array([g["h"]])
    y = O.expert_forward(h, np.array(g["gate"]), np.array(g["up"]), np.array(g["down"]))
    np.testing.assert_allclose(y[0], g["y"], rtol=1e-15)


def test_split_identity_every_granule():
    """C-P1: y_top(I_top) + y_bot(I_top) == unsplit for every I_top in {0, g, ..., I}."""
    _, _, experts = _toy_layer()
    h = O.bf16_to_f64(_bits(synth.batch_hidden(3, 5, 64)))
    gate, up, down = (O.bf16_to_f64(x) for x in experts[3])
    full = O.expert_forward(h, gate, up, down)
    for i_top in range(0, 128 + 1, 16):
        yt, yb = O.expert_forward_split(h, gate, up, down, i_top)
        np.testing.assert_allclose(yt + yb, full, rtol=1e-12, atol=1e-14)
        if i_top == 0:
            assert np.all(yt == 0)
        if i_top == 128:
            assert np.all(yb == 0)


def _hf_experts_from(experts):
    gu = torch.stack([torch.cat([torch.from_numpy(O.bf16_to_f64(g)), torch.from_numpy(O.bf16_to_f64(u))], 0)
                      for g, u, _ in experts])
    dn = torch.stack([torch.from_numpy(O.bf16_to_f64(dd)) for _, _, dd in experts])
    return gu, dn


def test_moe_layer_matches_hf_mixtral_block():
    from transformers import MixtralConfig
    from transformers.models.mixtral.modeling_mixtral import MixtralSparseMoeBlock
    h, router, experts = _toy_layer()
    cfg = MixtralConfig(hidden_size=64, intermediate_size=128, num_local_experts=8,
                        num_experts_per_tok=2, hidden_act="silu")
    blk = MixtralSparseMoeBlock(cfg).double().eval()
    gu, dn = _hf_experts_from(experts)
    with torch.no_grad():
        blk.gate.weight.copy_(torch.from_numpy(O.bf16_to_f64(router)))
        blk.experts.gate_up_proj.copy_(gu)
        blk.experts.down_proj.copy_(dn)
        ref = blk(torch.from_numpy(O.bf16_to_f64(h))[None]).squeeze(0).numpy()
    y, ids, w, _ = O.moe_layer(h, router, experts, K=2)
    # HF takes the softmax in fp32 (router_logits.float()); tolerance covers that rounding
    np.testing.assert_allclose(y, ref, rtol=1e-5, atol=1e-6 * np.abs(ref).max())


@pytest.mark.parametrize("norm", [True, False])
def test_moe_layer_matches_hf_qwen3_block(norm):
    from transformers import Qwen3MoeConfig
    from transformers.models.qwen3_moe.modeling_qwen3_moe import Qwen3MoeSparseMoeBlock
    N, d, I, K = 16, 64, 32, 4
    router = _bits(synth.router_weights(5, 0, N, d))
    experts = [tuple(_bits(x) for x in synth.expert_weights(5, 0, e, d, I)) for e in range(N)]
    h = _bits(synth.batch_hidden(5, 9, d))
    cfg = Qwen3MoeConfig(hidden_size=d, moe_intermediate_size=I, num_experts=N, num_experts_per_tok=K,
                         norm_topk_prob=norm, hidden_act="silu")
    blk = Qwen3MoeSparseMoeBlock(cfg).double().eval()
    gu, dn = _hf_experts_from(experts)
    with torch.no_grad():
        blk.gate.weight.copy_(torch.from_numpy(O.bf16_to_f64(router)))
        blk.experts.gate_up_proj.copy_(gu)
        blk.experts.down_proj.copy_(dn)
        out = blk(torch.from_numpy(O.bf16_to_f64(h))[None])
        ref = (out[0] if isinstance(out, tuple) else out).squeeze(0).numpy()
    y, _, _, _ = O.moe_layer(h, router, experts, K=K, renorm=norm)
    np.testing.assert_allclose(y, ref, rtol=1e-5, atol=1e-6 * np.abs(ref).max())


def _deepseek_hf_case():
    """Renorm off + 2 shared experts through HF's DeepseekV2Moe in fp64; HF's single shared MLP
    of 2I rows equals our two shared experts of I rows by the split identity (reading Q6)."""
    from transformers import DeepseekV2Config
    from transformers.models.deepseek_v2.modeling_deepseek_v2 import DeepseekV2Moe
    N, d, I, K = 16, 64, 32, 3
    router = _bits(synth.router_weights(6, 0, N, d))
    experts = [tuple(_bits(x) for x in synth.expert_weights(6, 0, e, d, I)) for e in range(N)]
    shared = [tuple(_bits(x) for x in synth.shared_expert_weights(6, 0, s, d, I)) for s in range(2)]
    h = _bits(synth.batch_hidden(6, 7, d))
    cfg = DeepseekV2Config(hidden_size=d, moe_intermediate_size=I, n_routed_experts=N, num_experts_per_tok=K,
                           n_shared_experts=2, routed_scaling_factor=1.0, topk_method="greedy",
                           n_group=1, topk_group=1, hidden_act="silu", intermediate_size=4 * d)
    blk = DeepseekV2Moe(cfg).double().eval()
    gu, dn = _hf_experts_from(experts)
    f = lambda a: torch.from_numpy(O.bf16_to_f64(a))
    with torch.no_grad():
        blk.gate.weight.copy_(f(router))
        blk.experts.gate_up_proj.copy_(gu)
        blk.experts.down_proj.copy_(dn)
        blk.shared_experts.gate_proj.weight.copy_(torch.cat([f(shared[0][0]), f(shared[1][0])], 0))
        blk.shared_experts.up_proj.weight.copy_(torch.cat([f(shared[0][1]), f(shared[1][1])], 0))
        blk.shared_experts.down_proj.weight.copy_(torch.cat([f(shared[0][2]), f(shared[1][2])], 1))
        ref = blk(f(h)[None]).squeeze(0).numpy()
    return h, router, experts, shared, K, ref


def test_moe_layer_matches_hf_deepseek_v2_block():
    h, router, experts, shared, K, ref = _deepseek_hf_case()
    y, _, _, _ = O.moe_layer(h, router, experts, K=K, shared=shared, renorm=False)
    np.testing.assert_allclose(y, ref, rtol=1e-5, atol=1e-6 * np.abs(ref).max())


@pytest.mark.parametrize("G", [2, 4])
def test_tp_partials_sum_to_hf_block(G):
    """C-P16 for tensor parallelism along I: the per-rank shares over the
    row partition {[rI/G, (r+1)I/G)} of every routed and shared expert sum to HF's
    DeepseekV2Moe output; each share alone is NOT the full output (a dropped slice would show)."""
    h, router, experts, shared, K, ref = _deepseek_hf_case()
    parts = [O.moe_layer_tp_partial(h, router, experts, K, r, G, shared=shared, renorm=False) for r in range(G)]
    y = np.sum(parts, axis=0)
    np.testing.assert_allclose(y, ref, rtol=1e-5, atol=1e-6 * np.abs(ref).max())
    for p in parts:
        assert np.abs(p - ref).max() > 1e-3 * np.abs(ref).max()


def test_single_expert_reduces_to_plain_mlp():
    """K=1 with renormalisation gives w = 1 exactly: the layer is one SwiGLU MLP
    (torch.nn.functional textbook form)."""
    h, router, experts = _toy_layer(B=6)
    y, ids, w, _ = O.moe_layer(h, router, experts, K=1)
    assert np.all(w == 1.0)
    hf = torch.from_numpy(O.bf16_to_f64(h))
    for b in range(6):
        g, u, dn = (torch.from_numpy(O.bf16_to_f64(x)) for x in experts[ids[b, 0]])
        ref = torch.nn.functional.linear(torch.nn.functional.silu(hf[b] @ g.T) * (hf[b] @ u.T), dn)
        np.testing.assert_allclose(y[b], ref.numpy(), rtol=1e-12, atol=1e-14)


def test_predicted_ranking_batch1_and_batch():
    rng = np.random.default_rng(7)
    l = rng.normal(size=(1, 12))
    r = O.predicted_ranking(l, 3)
    assert list(r) == list(np.argsort(-l[0], kind="stable"))
    # hand example B=2, N=4, K=1: token0 top=2, token1 top=2 -> c=[0,0,2,0];
    # remaining by max logit desc: expert 1 (0.9), 3 (0.5), 0 (0.1)
    l2 = np.array([[0.1, 0.9, 1.0, 0.2], [0.0, -1.0, 2.0, 0.5]])
    assert list(O.predicted_ranking(l2, 1)) == [2, 1, 3, 0]
