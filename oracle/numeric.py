"""C-N: the numeric part of the MoE layer, as its plain definition (TEST INFRASTRUCTURE).

The method (cache, split, offload, prefetch) reaches exactly the plain MoE output
("the cached top segment and the buffered bottom segment are concatenated"), so
the oracle is a dense MoE layer with all weights in memory, evaluated in fp64.

Citations:
  router scores / top-K          P:143-145  (s_{i,j} = softmax[R^i(h^i)]_j, top-K)
  MoE output, Eq. 2              P:146-149  (renormalised weights s_j / sum_o s_o)
  speculative prediction, Eq. 3  P:287-290  (s^pred_{i+1} = softmax[R^{i+1}(h^i)])
  vertical split                 P:12-13, P:196, P:230 (reading Q1: along I)
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "bf16_to_f64", "router_logits", "topk_ids", "gate_weights", "silu",
    "expert_forward", "expert_forward_split", "moe_layer", "predicted_ranking",
]


def weights_f64(w: np.ndarray) -> np.ndarray:
    """Expert weights as fp64: uint16 arrays are bf16 bit patterns; float64 arrays (dequantised
    low-bit experts, oracle/quant.py) are taken as they are."""
    if np.asarray(w).dtype == np.float64:
        return np.asarray(w)
    return bf16_to_f64(w)


def bf16_to_f64(bits: np.ndarray) -> np.ndarray:
    """uint16 bf16 bit patterns -> exact fp64 values."""
    b = np.ascontiguousarray(bits, dtype=np.uint16)
    return (b.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def router_logits(h_bits: np.ndarray, w_bits: np.ndarray) -> np.ndarray:
    """l[b, j] = sum_k h[b,k] * W_r[j,k] in fp64, canonical order C.R.

    R^i is a bias-free linear map R^d -> R^N.  Every bf16*bf16 product is exact
    in fp64, so only the summation order matters; C.R fixes it:
      1. index k in [0, d) is cut into chunks of 8; chunk c belongs to lane c mod 32;
      2. lane l adds its products in increasing k, starting from +0.0;
      3. lanes combine by xor-butterfly o = 16, 8, 4, 2, 1: acc_l <- acc_l + acc_{l^o};
      4. the logit is acc_0.
    Written with elementwise numpy adds only (no np.sum / dot, which block or pair).
    """
    h = bf16_to_f64(h_bits)             # [B][d]
    w = bf16_to_f64(w_bits)             # [N][d]
    B, d = h.shape
    N = w.shape[0]
    assert d % 8 == 0, "canonical router order needs d % 8 == 0"
    n_chunks = d // 8
    acc = np.zeros((B, N, 32), dtype=np.float64)
    lanes = np.arange(32)
    for j in range((n_chunks + 31) // 32):
        chunk = lanes + 32 * j
        valid = chunk < n_chunks
        for e in range(8):
            k = chunk[valid] * 8 + e
            prod = h[:, None, k] * w[None, :, k]          # exact products [B][N][lanes]
            acc[:, :, valid] = acc[:, :, valid] + prod
    for o in (16, 8, 4, 2, 1):
        acc = acc + acc[:, :, lanes ^ o]
    return acc[:, :, 0].copy()


def topk_ids(logits_row: np.ndarray, K: int) -> np.ndarray:
    """The K largest experts by key (l desc, id asc), returned in key order."""
    N = logits_row.shape[0]
    order = sorted(range(N), key=lambda j: (-logits_row[j], j))
    return np.array(order[:K], dtype=np.int32)


def gate_weights(logits_row: np.ndarray, ids: np.ndarray, renorm: bool = True) -> np.ndarray:
    """Eq. 2: w_k = s_{j_k} / sum_{o in S} s_o with s = softmax(l).

    With renormalisation the softmax denominator over all N cancels, leaving the
    softmax over the selected logits: w_k = exp(l_k - l_max) / sum_{k'} exp(l_k' - l_max).
    renorm=False (reading Q4, DeepSeek-V2 style) returns the raw s_{j_k}.
    """
    l = logits_row.astype(np.float64)
    if renorm:
        sel = l[ids]
        m = sel.max()
        e = np.exp(sel - m)
        return e / e.sum()
    m = l.max()
    e = np.exp(l - m)
    return e[ids] / e.sum()


def silu(x: np.ndarray) -> np.ndarray:
    return x / (1.0 + np.exp(-x))


def expert_forward(h: np.ndarray, gate: np.ndarray, up: np.ndarray, down: np.ndarray) -> np.ndarray:
    """SwiGLU FFN expert (reading Q3): E(h) = W_down (silu(W_gate h) * (W_up h)).

    h [B][d] fp64, gate/up [I][d], down [d][I] (HF layout), all fp64.  -> [B][d].
    """
    g = h @ gate.T
    u = h @ up.T
    a = silu(g) * u
    return a @ down.T


def expert_forward_split(h, gate, up, down, i_top: int):
    """Top + bottom partial down-projections at split row i_top (reading Q1).

    Returns (y_top, y_bottom); y_top + y_bottom == expert_forward(...) by linearity.
    """
    g = h @ gate.T
    u = h @ up.T
    a = silu(g) * u
    y_top = a[:, :i_top] @ down[:, :i_top].T
    y_bot = a[:, i_top:] @ down[:, i_top:].T
    return y_top, y_bot


def moe_layer(h_bits, router_bits, experts, K, shared=(), renorm=True):
    """The dense MoE layer (Eq. 2 inner sum; reading Q5: no Norm / residual).

    experts: sequence of N (gate, up, down) uint16 bf16 bit arrays in HF layout
             (or a callable e -> triple, so large layers can be evaluated lazily).
    shared:  shared experts, always active with weight 1 (reading Q6).
    Returns (y fp64 [B][d], ids int32 [B][K], w fp64 [B][K], logits fp64 [B][N]).
    """
    h = bf16_to_f64(h_bits)
    logits = router_logits(h_bits, router_bits)
    B, d = h.shape
    get = experts if callable(experts) else (lambda e: experts[e])
    ids = np.stack([topk_ids(logits[b], K) for b in range(B)])
    w = np.stack([gate_weights(logits[b], ids[b], renorm) for b in range(B)])
    y = np.zeros((B, d), dtype=np.float64)
    for e in sorted(set(ids.ravel().tolist())):
        gate, up, down = (weights_f64(x) for x in get(e))
        rows = [b for b in range(B) if e in ids[b]]
        out = expert_forward(h[rows], gate, up, down)
        for r, b in enumerate(rows):
            k = int(np.where(ids[b] == e)[0][0])
            y[b] += w[b, k] * out[r]
    for (gate, up, down) in shared:
        y += expert_forward(h, weights_f64(gate), weights_f64(up), weights_f64(down))
    return y, ids, w, logits


def moe_layer_ep_partial(h_bits, router_bits, experts, K, ep_rank, ep_size, shared=(), renorm=True):
    """Rank ep_rank's share of the layer output under expert parallelism:
    the routed experts it owns (e * ep_size // N == ep_rank) plus rows
    [r I / G, (r+1) I / G) of every shared expert (split identity).  Summing the shares
    of all ranks gives moe_layer(...)[0]."""
    h = bf16_to_f64(h_bits)
    logits = router_logits(h_bits, router_bits)
    B, d = h.shape
    N = logits.shape[1]
    get = experts if callable(experts) else (lambda e: experts[e])
    y = np.zeros((B, d), dtype=np.float64)
    for b in range(B):
        ids = topk_ids(logits[b], K)
        w = gate_weights(logits[b], ids, renorm)
        for k, e in enumerate(ids):
            if e * ep_size // N != ep_rank:
                continue
            gate, up, down = (bf16_to_f64(x) for x in get(int(e)))
            y[b] += w[k] * expert_forward(h[b:b + 1], gate, up, down)[0]
    for (gate, up, down) in shared:
        g, u, dn = bf16_to_f64(gate), bf16_to_f64(up), bf16_to_f64(down)
        I = g.shape[0]
        lo, hi = ep_rank * I // ep_size, (ep_rank + 1) * I // ep_size
        y += expert_forward(h, g[lo:hi], u[lo:hi], dn[:, lo:hi])
    return y


def moe_layer_tp_partial(h_bits, router_bits, experts, K, tp_rank, tp_size, shared=(), renorm=True):
    """Rank tp_rank's share of the layer output under tensor parallelism along I (SURVEY 8(f)
    NEXT-4): every routed and shared expert restricted to its intermediate rows
    [r I / G, (r+1) I / G) (gate/up rows, down columns), weighted by the full layer's gate
    weights.  The split identity of P:254 (a sum of partial down-projections over a partition
    of I) makes the sum of all ranks' shares equal to moe_layer(...)[0]."""
    h = bf16_to_f64(h_bits)
    logits = router_logits(h_bits, router_bits)
    B, d = h.shape
    get = experts if callable(experts) else (lambda e: experts[e])
    y = np.zeros((B, d), dtype=np.float64)
    for b in range(B):
        ids = topk_ids(logits[b], K)
        w = gate_weights(logits[b], ids, renorm)
        for k, e in enumerate(ids):
            g, u, dn = (weights_f64(x) for x in get(int(e)))
            I = g.shape[0]
            lo, hi = tp_rank * I // tp_size, (tp_rank + 1) * I // tp_size
            y[b] += w[k] * expert_forward(h[b:b + 1], g[lo:hi], u[lo:hi], dn[:, lo:hi])[0]
    for (gate, up, down) in shared:
        g, u, dn = weights_f64(gate), weights_f64(up), weights_f64(down)
        I = g.shape[0]
        lo, hi = tp_rank * I // tp_size, (tp_rank + 1) * I // tp_size
        y += expert_forward(h, g[lo:hi], u[lo:hi], dn[:, lo:hi])
    return y


def predicted_ranking(pred_logits: np.ndarray, K: int) -> np.ndarray:
    """Next-layer ranking R' of all N experts (Eq. 3; reading Q9).

    key(j) = (c_j desc, max_b l'[b,j] desc, j asc), c_j = #tokens whose predicted top-K
    (by l' desc, id asc) contains j.  For B = 1 this is "descending order of their
    predicted scores" since softmax is monotone.
    """
    B, N = pred_logits.shape
    c = np.zeros(N, dtype=np.int64)
    for b in range(B):
        for j in topk_ids(pred_logits[b], K):
            c[j] += 1
    mx = pred_logits.max(axis=0)
    order = sorted(range(N), key=lambda j: (-c[j], -mx[j], j))
    return np.array(order, dtype=np.int32)


def attention_decode(q_bits, k_bits, v_bits, S):
    """Attention stand-in (Att^i of Eq. 1): grouped-query attention
    of B decode tokens over the first S positions of a KV cache, fp64.
    q [B][Hq][dh], k / v [B][S_max][Hkv][dh] (bf16 bits); head h reads kv head h // (Hq / Hkv).
    out[b][h] = sum_s softmax_s(q . k_s / sqrt(dh)) v_s."""
    q, k, v = bf16_to_f64(q_bits), bf16_to_f64(k_bits), bf16_to_f64(v_bits)
    B, Hq, dh = q.shape
    Hkv = k.shape[2]
    G = Hq // Hkv
    out = np.zeros((B, Hq, dh))
    for b in range(B):
        for h in range(Hq):
            kk, vv = k[b, :S, h // G], v[b, :S, h // G]
            sc = kk @ q[b, h] / np.sqrt(dh)
            p = np.exp(sc - sc.max())
            out[b, h] = (p / p.sum()) @ vv
    return out
