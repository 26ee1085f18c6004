// Attention stand-in for the decode step (the paper's Att^i of Eq. 1, P:97-104,
// whose duration T_att opens the prefetch window): grouped-query attention of B new
// tokens over a KV cache of S positions, flash-decoding style.
//
//   o[b][h] = sum_s softmax_s(q[b][h] . k[b][s][h/G] / sqrt(dh)) v[b][s][h/G],   G = Hq / Hkv
//
// K_A1: grid (splits, Hkv, B), 4 warps; a CTA streams positions [s0, s1) of one kv head once and
// serves all G query heads of its group.  A warp takes tiles of 32 positions: lane j scores
// position j against the G queries (staged in shared memory), one max / sum butterfly per tile
// and head updates the online softmax (running max m, sum l), then p_j is broadcast while the
// lanes (4 dims each) accumulate p_j * v_j; the 4 warps merge in shared memory and write one
// partial (m, l, acc[dh]) per (split, head).  K_A2 merges the splits of every (b, h) in split
// order.  HBM-bound: the cache is read once (2 * S * Hkv * dh * 2 bytes per token); fp32 math.
#include "kernels.hpp"
#include "device_utils.cuh"

#include <cmath>

namespace moepic {

namespace {
constexpr int kAttnWarps = 4;
constexpr int kAttnDh = 128;
}  // namespace

int attn_splits(int S) { return (S + kAttnChunk - 1) / kAttnChunk; }

template <int G>
__global__ void __launch_bounds__(kAttnWarps * 32) k_attn_split(AttnParams p) {
  const int split = blockIdx.x, kh = blockIdx.y, b = blockIdx.z;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int s0 = split * kAttnChunk, s1 = min(p.S, s0 + kAttnChunk);
  __shared__ float sq[G][kAttnDh];   // the group's G queries, pre-scaled by 1/sqrt(dh)
  const float scale = rsqrtf((float)kAttnDh);
  for (int i = threadIdx.x; i < G * kAttnDh; i += blockDim.x)
    sq[i / kAttnDh][i % kAttnDh] =
        __uint_as_float((uint32_t)p.q[((size_t)b * p.Hq + kh * G) * kAttnDh + i] << 16) * scale;
  __syncthreads();
  float m[G], l[G], acc[G][4];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    m[g] = -INFINITY;
    l[g] = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[g][i] = 0.f;
  }
  const size_t rowstride = (size_t)p.Hkv * kAttnDh;
  const uint16_t* kb = p.k + (size_t)b * p.S_max * rowstride + (size_t)kh * kAttnDh;
  const uint16_t* vb = p.v + (size_t)b * p.S_max * rowstride + (size_t)kh * kAttnDh;
  // tiles of 32 positions: lane j scores position j of the tile (no per-position reduction),
  // one max / sum butterfly per tile and head, then p_j is broadcast to accumulate v_j
  for (int t0 = s0 + warp * 32; t0 < s1; t0 += kAttnWarps * 32) {
    const int pos = t0 + lane;
    const bool valid = pos < s1;
    float sc[G];
#pragma unroll
    for (int g = 0; g < G; ++g) sc[g] = 0.f;
    if (valid) {
      const uint4* kr = reinterpret_cast<const uint4*>(kb + (size_t)pos * rowstride);
#pragma unroll
      for (int c = 0; c < kAttnDh / 8; ++c) {
        float kv[8];
        unpack8(__ldg(kr + c), kv);
#pragma unroll
        for (int g = 0; g < G; ++g)
#pragma unroll
          for (int e = 0; e < 8; ++e) sc[g] = fmaf(kv[e], sq[g][8 * c + e], sc[g]);
      }
    }
    float pj[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float mx = valid ? sc[g] : -INFINITY;
#pragma unroll
      for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      const float mn = fmaxf(m[g], mx);
      pj[g] = valid ? __expf(sc[g] - mn) : 0.f;
      float sum = pj[g];
#pragma unroll
      for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      const float corr = __expf(m[g] - mn);
      l[g] = l[g] * corr + sum;
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[g][i] *= corr;
      m[g] = mn;
    }
    const int nj = min(32, s1 - t0);
#pragma unroll 8
    for (int j = 0; j < nj; ++j) {
      float vv[4];
      unpack4(__ldg(reinterpret_cast<const uint2*>(vb + (size_t)(t0 + j) * rowstride) + lane), vv);
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float pg = __shfl_sync(0xffffffffu, pj[g], j);
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[g][i] = fmaf(pg, vv[i], acc[g][i]);
      }
    }
  }
  // merge the warps: warp w's (m, l, acc) in smem, warp 0 combines in warp order
  __shared__ float sm[kAttnWarps][G], sl[kAttnWarps][G], sacc[kAttnWarps][G][kAttnDh];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    if (lane == 0) {
      sm[warp][g] = m[g];
      sl[warp][g] = l[g];
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) sacc[warp][g][lane * 4 + i] = acc[g][i];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float M = -INFINITY;
      for (int w = 0; w < kAttnWarps; ++w) M = fmaxf(M, sm[w][g]);
      float L = 0.f, a[4] = {0.f, 0.f, 0.f, 0.f};
      for (int w = 0; w < kAttnWarps; ++w) {
        const float c = sm[w][g] == -INFINITY ? 0.f : __expf(sm[w][g] - M);
        L += sl[w][g] * c;
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] += sacc[w][g][lane * 4 + i] * c;
      }
      const int h = kh * G + g;
      float* part = p.ws + (((size_t)b * p.Hq + h) * p.splits + split) * (kAttnDh + 2);
      if (lane == 0) {
        part[0] = M;
        part[1] = L;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) part[2 + lane * 4 + i] = a[i];
    }
  }
}

__global__ void __launch_bounds__(kAttnDh) k_attn_merge(AttnParams p) {
  // the splits' (m, l) are read in parallel (one thread each) and turned into weights once; then
  // every thread (one dim) sums its column with independent loads
  constexpr int kMaxSplits = 1024;   // S <= 131072 positions
  __shared__ float sc[kMaxSplits];
  __shared__ float sL;
  const int h = blockIdx.x, b = blockIdx.y, i = threadIdx.x;
  const float* part = p.ws + ((size_t)b * p.Hq + h) * p.splits * (kAttnDh + 2);
  float mloc = -INFINITY;
  for (int sp = i; sp < p.splits; sp += kAttnDh) mloc = fmaxf(mloc, part[(size_t)sp * (kAttnDh + 2)]);
#pragma unroll
  for (int o = 16; o; o >>= 1) mloc = fmaxf(mloc, __shfl_xor_sync(0xffffffffu, mloc, o));
  __shared__ float swm[kAttnDh / 32];
  if ((i & 31) == 0) swm[i >> 5] = mloc;
  __syncthreads();
  float M = swm[0];
#pragma unroll
  for (int w = 1; w < kAttnDh / 32; ++w) M = fmaxf(M, swm[w]);
  for (int sp = i; sp < p.splits; sp += kAttnDh) {
    const float m0 = part[(size_t)sp * (kAttnDh + 2)];
    sc[sp] = m0 == -INFINITY ? 0.f : __expf(m0 - M);
  }
  __syncthreads();
  if (i == 0) {   // sum of l in split order (fixed order)
    float L = 0.f;
    for (int sp = 0; sp < p.splits; ++sp) L += part[(size_t)sp * (kAttnDh + 2) + 1] * sc[sp];
    sL = L;
  }
  float a = 0.f;
#pragma unroll 8
  for (int sp = 0; sp < p.splits; ++sp) a += part[(size_t)sp * (kAttnDh + 2) + 2 + i] * sc[sp];
  __syncthreads();
  p.out[((size_t)b * p.Hq + h) * kAttnDh + i] = a / sL;
}

template <int G>
static void launch_g(const AttnParams& p, cudaStream_t s) {
  k_attn_split<G><<<dim3(p.splits, p.Hkv, p.B), kAttnWarps * 32, 0, s>>>(p);
}

// the decode step alternates these kernels with K2 (~200 KB of shared memory): asking for the
// maximum carveout keeps the SM's L1 / shared split unchanged between them
cudaError_t attention_init() {
  cudaError_t e = cudaSuccess, r;
  const void* fns[] = {(const void*)k_attn_split<1>, (const void*)k_attn_split<2>, (const void*)k_attn_split<4>,
                       (const void*)k_attn_split<8>, (const void*)k_attn_split<16>, (const void*)k_attn_merge};
  for (const void* f : fns)
    if ((r = cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100)) != cudaSuccess) e = r;
  return e;
}

bool launch_attention(const AttnParams& p, cudaStream_t s) {
  const int G = p.Hq / p.Hkv;
  switch (G) {
    case 1: launch_g<1>(p, s); break;
    case 2: launch_g<2>(p, s); break;
    case 4: launch_g<4>(p, s); break;
    case 8: launch_g<8>(p, s); break;
    case 16: launch_g<16>(p, s); break;
    default: return false;
  }
  k_attn_merge<<<dim3(p.Hq, p.B), kAttnDh, 0, s>>>(p);
  return true;
}

}  // namespace moepic
