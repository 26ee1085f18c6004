// K3 combine: y[b] = (h[b] if residual) + sum over the step's segments and
// their per-CTA partials, in a fixed order (deterministic).
#include "kernels.hpp"
#include "device_utils.cuh"

namespace moepic {

// CTA (x, b): 32 float4 columns of token b; warp w sums chunks w, w+8, ... of every segment
// serving b (lane = column), then the 8 warp partials are added in warp order.  Fixed order
// everywhere -> deterministic.
template <int CAP>
struct CombineParamsCap {
  float* y;
  const uint16_t* h;
  const float* ws;
  int B, d, residual, nsegs;
  CombineSeg segs[CAP];
};

template <class P>
__global__ void __launch_bounds__(256) k3_combine(const __grid_constant__ P p) {
  __shared__ float4 red[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int b = blockIdx.y;
  const int c4 = blockIdx.x * 32 + lane;
  const int d4 = p.d >> 2;
  const bool active = c4 < d4;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const uint32_t bit = 1u << b;
  if (active) {
    for (int s = 0; s < p.nsegs; ++s) {
      const CombineSeg sg = p.segs[s];
      if (!(sg.tok_mask & bit)) continue;
      const int ntok = __popc(sg.tok_mask);
      const int t = __popc(sg.tok_mask & (bit - 1u));
      const float4* base = reinterpret_cast<const float4*>(p.ws + sg.ws_off + (int64_t)t * p.d) + c4;
      const int64_t stride4 = (int64_t)ntok * d4;
      int ci = warp;
      for (; ci + 24 < sg.nchunks; ci += 32) {   // 4 independent loads in flight per lane
        const float4 v0 = base[(int64_t)ci * stride4];
        const float4 v1 = base[(int64_t)(ci + 8) * stride4];
        const float4 v2 = base[(int64_t)(ci + 16) * stride4];
        const float4 v3 = base[(int64_t)(ci + 24) * stride4];
        acc.x += v0.x; acc.y += v0.y; acc.z += v0.z; acc.w += v0.w;
        acc.x += v1.x; acc.y += v1.y; acc.z += v1.z; acc.w += v1.w;
        acc.x += v2.x; acc.y += v2.y; acc.z += v2.z; acc.w += v2.w;
        acc.x += v3.x; acc.y += v3.y; acc.z += v3.z; acc.w += v3.w;
      }
      for (; ci < sg.nchunks; ci += 8) {
        const float4 v = base[(int64_t)ci * stride4];
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
    }
  }
  red[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && active) {
    float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
    if (p.residual) {
      const uint2 hv = reinterpret_cast<const uint2*>(p.h + (size_t)b * p.d)[c4];
      r = make_float4(bf16lo(hv.x), bf16hi(hv.x), bf16lo(hv.y), bf16hi(hv.y));
    }
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      const float4 v = red[w][lane];
      r.x += v.x; r.y += v.y; r.z += v.z; r.w += v.w;
    }
    reinterpret_cast<float4*>(p.y + (size_t)b * p.d)[c4] = r;
  }
}

// parameter block sized to the step (see expert.cu: launch commands cross the busy PCIe link)
template <int CAP>
static void launch_cap(const CombineParams& p, cudaStream_t s) {
  CombineParamsCap<CAP> q;
  q.y = p.y; q.h = p.h; q.ws = p.ws;
  q.B = p.B; q.d = p.d; q.residual = p.residual; q.nsegs = p.nsegs;
  for (int i = 0; i < p.nsegs; ++i) q.segs[i] = p.segs[i];
  dim3 grid((unsigned)((p.d / 4 + 31) / 32), (unsigned)p.B);
  k3_combine<CombineParamsCap<CAP>><<<grid, 256, 0, s>>>(q);
}

void launch_combine(const CombineParams& p, cudaStream_t s) {
  if (p.nsegs <= 16) launch_cap<16>(p, s);
  else if (p.nsegs <= 128) launch_cap<128>(p, s);
  else launch_cap<kMaxStepSegs>(p, s);
}

}  // namespace moepic
