// Combine of the step's partials, shared by the fused tail of the
// final K2 launch and by the stand-alone K3.
//
// y[b][c] = (h[b][c] if residual) + sum over the partial vectors serving token b.  The partials
// of token b are enumerated in a fixed order (segments in step order, chunks in CTA order) and
// numbered k = 0, 1, ...  A block covers CB consecutive float4 columns of one token; lane l of
// warp w takes column l % CB and the partials k = w * P + l / CB (mod 16 P), P = 32 / CB, in
// increasing k (loads issued four at a time); the P lane phases are added by a butterfly, then
// the 16 warp sums in warp order.
// CB (32, 16, 8 or 4) is chosen from the output size only (combine_cb), so small outputs still
// spread over the whole grid; the order depends only on the step's segment table and the
// output shape, so the result is deterministic.
#pragma once

#include "kernels.hpp"
#include "device_utils.cuh"

namespace moepic {

constexpr int kCombineWarps = 16;

// float4 columns per block: the widest that still yields >= 128 blocks (all SMs busy)
__host__ __device__ inline int combine_cb(int B, int d) {
  const int d4 = d >> 2;
  int cb = 32;
  while (cb > 4 && (int64_t)B * ((d4 + cb - 1) / cb) < 128) cb >>= 1;
  return cb;
}
__host__ __device__ inline int combine_blocks(int B, int d) {
  const int cb = combine_cb(B, d);
  return B * (((d >> 2) + cb - 1) / cb);
}

// Must be called by all kCombineWarps * 32 threads of the block; `red` is 16 * 32 float4 of smem.
__device__ __forceinline__ void combine_block(int blk, const CombineSeg* segs, int nsegs, const float* ws,
                                              const uint16_t* h, float* y, int B, int d, int residual,
                                              float4* red, unsigned long long* dbg = nullptr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int d4 = d >> 2;
  const int CB = combine_cb(B, d);
  const int P = 32 / CB;                        // lane phases over the partials
  const int S = kCombineWarps * P;              // partial stride of one lane
  const int ncb = (d4 + CB - 1) / CB;
  const int b = blk / ncb;
  const int c4 = (blk - b * ncb) * CB + (lane % CB);
  const int phase = warp * P + lane / CB;       // this lane's residue class mod S
  const bool active = c4 < d4;
  const uint32_t bit = 1u << b;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  // flattened walk over token b's partials: a cursor (segment s, its first index k0) moves
  // forward as k grows, so four addresses are formed before their loads are issued together
  // (one memory latency per four partials instead of one per segment)
  int total = 0;
  for (int s = 0; s < nsegs; ++s)
    if (segs[s].tok_mask & bit) total += segs[s].nchunks;
  if (dbg && threadIdx.x == 0) dbg[5] = gtimer();
  int cs = 0, ck0 = 0;
  auto addr = [&](int k) -> const float4* {   // k < total, k non-decreasing across calls
    for (;;) {
      const CombineSeg& sg = segs[cs];
      if ((sg.tok_mask & bit) && k < ck0 + sg.nchunks) {
        const int ntok = __popc(sg.tok_mask);
        const int t = __popc(sg.tok_mask & (bit - 1u));
        return reinterpret_cast<const float4*>(ws + sg.ws_off + (int64_t)t * d) + c4 +
               (int64_t)(k - ck0) * ntok * d4;
      }
      if (sg.tok_mask & bit) ck0 += sg.nchunks;
      ++cs;
    }
  };
  if (active) {
    int k = phase;
    for (; k + 3 * S < total; k += 4 * S) {
      const float4* p0 = addr(k);
      const float4* p1 = addr(k + S);
      const float4* p2 = addr(k + 2 * S);
      const float4* p3 = addr(k + 3 * S);
      const float4 v0 = *p0, v1 = *p1, v2 = *p2, v3 = *p3;
      acc.x += v0.x; acc.y += v0.y; acc.z += v0.z; acc.w += v0.w;
      acc.x += v1.x; acc.y += v1.y; acc.z += v1.z; acc.w += v1.w;
      acc.x += v2.x; acc.y += v2.y; acc.z += v2.z; acc.w += v2.w;
      acc.x += v3.x; acc.y += v3.y; acc.z += v3.z; acc.w += v3.w;
    }
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    const float4* q0 = k < total ? addr(k) : nullptr;
    const float4* q1 = k + S < total ? addr(k + S) : nullptr;
    const float4* q2 = k + 2 * S < total ? addr(k + 2 * S) : nullptr;
    const float4 v0 = q0 ? *q0 : z, v1 = q1 ? *q1 : z, v2 = q2 ? *q2 : z;
    if (q0) { acc.x += v0.x; acc.y += v0.y; acc.z += v0.z; acc.w += v0.w; }
    if (q1) { acc.x += v1.x; acc.y += v1.y; acc.z += v1.z; acc.w += v1.w; }
    if (q2) { acc.x += v2.x; acc.y += v2.y; acc.z += v2.z; acc.w += v2.w; }
  }
  if (dbg && threadIdx.x == 0) dbg[6] = gtimer();
  // lane phases (lanes CB apart) by a butterfly
  for (int o = CB; o < 32; o <<= 1) {
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    acc.z += __shfl_xor_sync(0xffffffffu, acc.z, o);
    acc.w += __shfl_xor_sync(0xffffffffu, acc.w, o);
  }
  red[warp * 32 + lane] = acc;
  __syncthreads();
  if (dbg && threadIdx.x == 0) dbg[7] = gtimer();
  if (warp == 0 && lane < CB && active) {
    float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
    if (residual) {
      const uint2 hv = reinterpret_cast<const uint2*>(h + (size_t)b * d)[c4];
      r = make_float4(bf16lo(hv.x), bf16hi(hv.x), bf16lo(hv.y), bf16hi(hv.y));
    }
#pragma unroll
    for (int w = 0; w < kCombineWarps; ++w) {
      const float4 v = red[w * 32 + lane];
      r.x += v.x; r.y += v.y; r.z += v.z; r.w += v.w;
    }
    reinterpret_cast<float4*>(y + (size_t)b * d)[c4] = r;
  }
  __syncthreads();   // `red` is reused by the next block
}

// Flattened variant: the CTA first lists, per token, the float offsets of its partial vectors in
// the same fixed order (segments in step order, chunks in CTA order) in shared memory, so the
// lanes index their partials directly instead of walking the segment table.
// Called by all kCombineWarps * 32 threads; tstart: B + 1 ints; offs: sum over tokens of their
// partial counts (the host checks it fits).
__device__ __forceinline__ void combine_build_table(const CombineSeg* segs, int nsegs, int B, int d, int* tstart,
                                                    uint32_t* offs) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // 1. partial count per token (one warp per token; lanes over segments)
  for (int b = warp; b < B; b += kCombineWarps) {
    int tot = 0;
    for (int s0 = 0; s0 < nsegs; s0 += 32) {
      const int s = s0 + lane;
      int c = (s < nsegs && (segs[s].tok_mask >> b & 1u)) ? segs[s].nchunks : 0;
#pragma unroll
      for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
      tot += c;
    }
    if (lane == 0) tstart[b + 1] = tot;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    tstart[0] = 0;
    for (int b = 0; b < B; ++b) tstart[b + 1] += tstart[b];
  }
  __syncthreads();
  // 2. offsets: a segment's chunks at its exclusive prefix within the token
  for (int b = warp; b < B; b += kCombineWarps) {
    int base = tstart[b];
    for (int s0 = 0; s0 < nsegs; s0 += 32) {
      const int s = s0 + lane;
      const bool has = s < nsegs && (segs[s].tok_mask >> b & 1u);
      const int c = has ? segs[s].nchunks : 0;
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      if (has) {
        const uint32_t m = segs[s].tok_mask;
        const int ntok = __popc(m), t = __popc(m & ((1u << b) - 1u));
        const int64_t o0 = segs[s].ws_off + (int64_t)t * d;
        for (int k = 0; k < c; ++k) offs[base + incl - c + k] = (uint32_t)(o0 + (int64_t)k * ntok * d);
      }
      base += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void combine_block_flat(int blk, const int* tstart, const uint32_t* offs, const float* ws,
                                                   const uint16_t* h, float* y, int B, int d, int residual,
                                                   float4* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int d4 = d >> 2;
  const int CB = combine_cb(B, d);
  const int P = 32 / CB;
  const int S = kCombineWarps * P;
  const int ncb = (d4 + CB - 1) / CB;
  const int b = blk / ncb;
  const int c4 = (blk - b * ncb) * CB + (lane % CB);
  const int phase = warp * P + lane / CB;
  const bool active = c4 < d4;
  const uint32_t* ob = offs + tstart[b];
  const int total = tstart[b + 1] - tstart[b];
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (active) {
    const float4* w4 = reinterpret_cast<const float4*>(ws) + c4;
    int k = phase;
    for (; k + 3 * S < total; k += 4 * S) {
      const float4 v0 = w4[ob[k] >> 2], v1 = w4[ob[k + S] >> 2], v2 = w4[ob[k + 2 * S] >> 2], v3 = w4[ob[k + 3 * S] >> 2];
      acc.x += v0.x; acc.y += v0.y; acc.z += v0.z; acc.w += v0.w;
      acc.x += v1.x; acc.y += v1.y; acc.z += v1.z; acc.w += v1.w;
      acc.x += v2.x; acc.y += v2.y; acc.z += v2.z; acc.w += v2.w;
      acc.x += v3.x; acc.y += v3.y; acc.z += v3.z; acc.w += v3.w;
    }
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 v0 = k < total ? w4[ob[k] >> 2] : z;
    const float4 v1 = k + S < total ? w4[ob[k + S] >> 2] : z;
    const float4 v2 = k + 2 * S < total ? w4[ob[k + 2 * S] >> 2] : z;
    if (k < total) { acc.x += v0.x; acc.y += v0.y; acc.z += v0.z; acc.w += v0.w; }
    if (k + S < total) { acc.x += v1.x; acc.y += v1.y; acc.z += v1.z; acc.w += v1.w; }
    if (k + 2 * S < total) { acc.x += v2.x; acc.y += v2.y; acc.z += v2.z; acc.w += v2.w; }
  }
  for (int o = CB; o < 32; o <<= 1) {
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    acc.z += __shfl_xor_sync(0xffffffffu, acc.z, o);
    acc.w += __shfl_xor_sync(0xffffffffu, acc.w, o);
  }
  red[warp * 32 + lane] = acc;
  __syncthreads();
  if (warp == 0 && lane < CB && active) {
    float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
    if (residual) {
      const uint2 hv = reinterpret_cast<const uint2*>(h + (size_t)b * d)[c4];
      r = make_float4(bf16lo(hv.x), bf16hi(hv.x), bf16lo(hv.y), bf16hi(hv.y));
    }
#pragma unroll
    for (int w = 0; w < kCombineWarps; ++w) {
      const float4 v = red[w * 32 + lane];
      r.x += v.x; r.y += v.y; r.z += v.z; r.w += v.w;
    }
    reinterpret_cast<float4*>(y + (size_t)b * d)[c4] = r;
  }
  __syncthreads();
}

}  // namespace moepic
