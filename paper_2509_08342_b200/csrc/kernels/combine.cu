// K3 combine: y[b] = (h[b] if residual) + sum over the step's segments and
// their per-CTA partials, in a fixed order (deterministic).  Used when no K2 launch of the step
// could fuse the combine.
#include "kernels.hpp"

#include <algorithm>
#include "device_utils.cuh"
#include "combine_dev.cuh"

namespace moepic {

// One CTA of 16 warps per (token, column block): combine_dev.cuh, the same order as
// the fused combine at the end of the final K2 launch.
template <int CAP>
struct CombineParamsCap {
  float* y;
  const uint16_t* h;
  const float* ws;
  int B, d, residual, nsegs;
  unsigned long long* tstamp;
  CombineSeg segs[CAP];
};

template <class P>
__global__ void __launch_bounds__(kCombineWarps * 32) k3_combine(const __grid_constant__ P p) {
  __shared__ float4 red[kCombineWarps * 32];
  extern __shared__ CombineSeg cs[];   // the segment table, walked per lane (see expert.cu)
  stamp_start(p.tstamp);
  asm volatile("griddepcontrol.launch_dependents;");   // a PDL-launched router may get ready now
  for (int i = threadIdx.x; i < p.nsegs; i += blockDim.x) cs[i] = p.segs[i];
  __syncthreads();
  combine_block(blockIdx.x, cs, p.nsegs, p.ws, p.h, p.y, p.B, p.d, p.residual, red);
  stamp_end(p.tstamp);
}

// parameter block sized to the step (see expert.cu: launch commands cross the busy PCIe link)
template <int CAP>
static void launch_cap(const CombineParams& p, cudaStream_t s) {
  CombineParamsCap<CAP> q;
  q.y = p.y; q.h = p.h; q.ws = p.ws;
  q.B = p.B; q.d = p.d; q.residual = p.residual; q.nsegs = p.nsegs; q.tstamp = p.tstamp;
  for (int i = 0; i < p.nsegs; ++i) q.segs[i] = p.segs[i];
  const int nblk = combine_blocks(p.B, p.d);
  k3_combine<CombineParamsCap<CAP>><<<nblk, kCombineWarps * 32, (size_t)p.nsegs * sizeof(CombineSeg), s>>>(q);
}

__global__ void __launch_bounds__(256) k0_stage_in(uint4* __restrict__ dst, const uint4* __restrict__ src,
                                                   size_t n16) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

void launch_stage_in(void* dst, const void* src_mapped, size_t bytes, cudaStream_t s) {
  const size_t n16 = bytes / 16;
  const int grid = (int)std::min<size_t>((n16 + 255) / 256, 64);
  k0_stage_in<<<grid, 256, 0, s>>>(static_cast<uint4*>(dst), static_cast<const uint4*>(src_mapped), n16);
}

__global__ void k0_trap() { __trap(); }

void launch_trap(cudaStream_t s) { k0_trap<<<1, 1, 0, s>>>(); }

__global__ void k0_stamp(unsigned long long* p) { *p = gtimer(); }
void launch_stamp(unsigned long long* p, cudaStream_t s) { k0_stamp<<<1, 1, 0, s>>>(p); }
// clock handshake (mapped host memory m): m[0] = 1 once running; waits for m[2] != 0 (written by
// the host right after it read its own clock); m[1] = %globaltimer when it saw it
__global__ void k0_clock_sync(volatile unsigned long long* m) {
  m[0] = 1;
  __threadfence_system();
  while (m[2] == 0) {
  }
  m[1] = gtimer();
  __threadfence_system();
}
void launch_clock_sync(unsigned long long* m, cudaStream_t s) { k0_clock_sync<<<1, 1, 0, s>>>(m); }

cudaError_t combine_init() {
  cudaError_t e = cudaSuccess, r;
  if ((r = cudaFuncSetAttribute(k3_combine<CombineParamsCap<16>>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                100)) != cudaSuccess) e = r;
  if ((r = cudaFuncSetAttribute(k3_combine<CombineParamsCap<128>>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                100)) != cudaSuccess) e = r;
  if ((r = cudaFuncSetAttribute(k3_combine<CombineParamsCap<kMaxStepSegs>>,
                                cudaFuncAttributePreferredSharedMemoryCarveout, 100)) != cudaSuccess) e = r;
  return e;
}

void launch_combine(const CombineParams& p, cudaStream_t s) {
  if (p.nsegs <= 16) launch_cap<16>(p, s);
  else if (p.nsegs <= 128) launch_cap<128>(p, s);
  else launch_cap<kMaxStepSegs>(p, s);
}

}  // namespace moepic
