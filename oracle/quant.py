"""Low-bit expert weights, format Q4G64 — TEST INFRASTRUCTURE.

The paper runs Mixtral with HQQ low-bit experts and leaves the format to the
quantiser; this build fixes one plain asymmetric 4-bit group format (reading Q28) so
the PCIe-bound path moves ~3.5x fewer bytes per expert.  Definition, per stored row vector
(gate row r, up row r, down column r, each d values) and per group of 64 consecutive entries
x_0..x_63 (bf16 values, exact in fp32):

    lo   = min_k x_k,   hi = max_k x_k                                   (fp32, exact)
    lo_b = the largest bf16 value <= lo                                   (round down)
    t    = fp32((hi - lo_b) / 15)        (the subtraction and the division each rounded)
    s_b  = the smallest bf16 value >= t, or 1.0 if that is 0               (round up)
    q_k  = clamp(rint(fp32(fp32(x_k - lo_b) / s_b)), 0, 15)  (rint: ties to even)
    x'_k = lo_b + q_k * s_b                                               (dequantised)

Rounding lo down and s up keeps every (x - lo_b) / s_b inside [0, 15] up to the fp32 rounding
of t, so |x'_k - x_k| <= s_b / 2 (+ the clamp at 15 within one fp32 ulp).  The integer codes
are decided in fp32 in this exact operation order on both sides (C++ host packer and this
oracle), so they are compared bit for bit; the layer output is then the plain MoE layer
(numeric.moe_layer) over the dequantised weights x'.
"""
from __future__ import annotations

import numpy as np

GROUP = 64


def _bf16_bits_to_f32(bits):
    return (np.ascontiguousarray(bits, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def bf16_round_down(v: np.ndarray) -> np.ndarray:
    """Largest bf16 value <= v (fp32 in, bf16 bit patterns out); v finite."""
    v = np.asarray(v, dtype=np.float32)
    u = v.view(np.uint32)
    t = (u >> 16).astype(np.uint16)                     # truncation = round toward zero
    back = _bf16_bits_to_f32(t)
    # negative values whose truncation is above v need one step further from zero
    bump = (v < 0) & (back > v)
    t = np.where(bump, t + 1, t).astype(np.uint16)
    return t


def bf16_round_up(v: np.ndarray) -> np.ndarray:
    """Smallest bf16 value >= v for v >= 0 (fp32 in, bf16 bit patterns out)."""
    v = np.asarray(v, dtype=np.float32)
    u = v.view(np.uint32)
    t = (u >> 16).astype(np.uint16)
    back = _bf16_bits_to_f32(t)
    bump = back < v
    return np.where(bump, t + 1, t).astype(np.uint16)


def quantize_vector(x_bits: np.ndarray):
    """One stored row vector (bf16 bits, length d, d % 64 == 0) ->
    (codes uint8 [d] in 0..15, s_b bits uint16 [d/64], lo_b bits uint16 [d/64])."""
    x = _bf16_bits_to_f32(x_bits).reshape(-1, GROUP)
    lo = x.min(axis=1)
    hi = x.max(axis=1)
    lo_b = bf16_round_down(lo)
    lo_f = _bf16_bits_to_f32(lo_b)
    t = (np.float32(hi - lo_f) / np.float32(15.0)).astype(np.float32)
    s_b = bf16_round_up(t)
    s_b = np.where(s_b == 0, np.uint16(0x3F80), s_b).astype(np.uint16)      # 0 -> 1.0
    s_f = _bf16_bits_to_f32(s_b)
    diff = (x - lo_f[:, None]).astype(np.float32)
    r = (diff / s_f[:, None]).astype(np.float32)
    q = np.clip(np.rint(r), 0, 15).astype(np.uint8)
    return q.reshape(-1), s_b, lo_b


def dequantize_vector(q, s_b, lo_b) -> np.ndarray:
    """fp64 x' = lo_b + q * s_b per group (exact in fp64)."""
    s = _bf16_bits_to_f32(s_b).astype(np.float64)
    lo = _bf16_bits_to_f32(lo_b).astype(np.float64)
    qq = np.asarray(q, dtype=np.float64).reshape(-1, GROUP)
    return (lo[:, None] + qq * s[:, None]).reshape(-1)


def quantize_expert(gate_bits, up_bits, down_bits):
    """HF-layout expert (gate/up [I][d], down [d][I], bf16 bits) -> per intermediate row r the
    codes and group parameters of gate_r, up_r and down[:, r]:
    dict(q=[I][3][d] uint8, s=[I][3][d/64] uint16, lo=[I][3][d/64] uint16)."""
    g = np.asarray(gate_bits, dtype=np.uint16)
    u = np.asarray(up_bits, dtype=np.uint16)
    dn = np.asarray(down_bits, dtype=np.uint16)
    I, d = g.shape
    # the row vectors of part p are rows of a [I][d] matrix; d % 64 == 0, so quantising the
    # flattened matrix groups exactly the 64-entry groups of each row vector
    parts = [quantize_vector(m.reshape(-1)) for m in (g, u, np.ascontiguousarray(dn.T))]
    q = np.stack([p[0].reshape(I, d) for p in parts], axis=1)
    s = np.stack([p[1].reshape(I, d // GROUP) for p in parts], axis=1)
    lo = np.stack([p[2].reshape(I, d // GROUP) for p in parts], axis=1)
    return dict(q=q, s=s, lo=lo)


def dequantize_expert(qe):
    """-> (gate [I][d], up [I][d], down [d][I]) fp64 dequantised weights."""
    q, s, lo = qe["q"], qe["s"], qe["lo"]
    I, _, d = q.shape
    w = dequantize_vector(q.reshape(-1), s.reshape(-1), lo.reshape(-1)).reshape(I, 3, d)
    return w[:, 0, :].copy(), w[:, 1, :].copy(), w[:, 2, :].T.copy()


def packed_row_bytes(d: int) -> int:
    """Bytes of one interleaved Q4G64 row: 3 x d/2 code bytes then 3 x d/64 (s, lo) bf16 pairs,
    padded to 16 bytes."""
    raw = 3 * (d // 2) + 3 * (d // GROUP) * 4
    return (raw + 15) // 16 * 16


def pack_expert(qe) -> np.ndarray:
    """The library's pinned-arena image of a Q4G64 expert ([I][packed_row_bytes] uint8):
    row r = [gate codes | up codes | down codes] (two codes per byte, low nibble = even column)
    then [gate (s, lo) | up (s, lo) | down (s, lo)] per group, then zero padding."""
    q, s, lo = qe["q"], qe["s"], qe["lo"]
    I, _, d = q.shape
    rb = packed_row_bytes(d)
    out = np.zeros((I, rb), np.uint8)
    for r in range(I):
        for part in range(3):
            c = q[r, part]
            out[r, part * (d // 2):(part + 1) * (d // 2)] = (c[0::2] | (c[1::2] << 4)).astype(np.uint8)
        base = 3 * (d // 2)
        for part in range(3):
            pr = np.empty(2 * (d // GROUP), np.uint16)
            pr[0::2] = s[r, part]
            pr[1::2] = lo[r, part]
            off = base + part * (d // GROUP) * 4
            out[r, off:off + (d // GROUP) * 4] = pr.view(np.uint8)
    return out
