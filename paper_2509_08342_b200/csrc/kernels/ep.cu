// Expert / tensor parallel data plane over peer device memory.
//
// Every rank owns one exchange region (cudaMalloc, exported with CUDA IPC and mapped by every
// peer, over NVLink / NVSwitch between GPUs).  Producers store straight into the consumer's
// region (P2P stores fused with the gather / combine that produces the rows), then publish a
// per-(phase, source) epoch counter with a system-scope release; consumers spin on their own
// counters with acquire loads.  Buffers are double-buffered by epoch parity: a peer can be at
// most one epoch ahead in any phase, because every phase of every layer waits for every rank.
//
// Phases (kernels below, launched on the caller's compute stream):
//   ids       each rank's routed ids / gate weights of its own tokens -> every rank (all-gather),
//             then published to the host mailbox (the control plane needs the whole batch)
//   dispatch  token rows -> the ranks owning their experts (one copy per (token, rank) pair)
//   combine   each rank's weighted partial rows -> the token's owner
//   reduce    owner sums its partial rows in rank order (+ residual)
//   allreduce replicated-token decode: y = sum over ranks of the partial outputs, rank order
// The NCCL transport (moepic_api.cpp) reuses the same index lists and the reduce / publish
// kernels; its data movement is ncclAllGather / grouped ncclSend-ncclRecv / ncclAllReduce.
#include <cstdint>

#include "ep.hpp"

namespace moepic {

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long* sig_of(uint8_t* base, const EpOffsets& of, int phase, int src) {
  return reinterpret_cast<unsigned long long*>(base + of.sig) + phase * kEpMaxRanks + src;
}

// threads 0..G-1 of the CTA each wait for one source, then the CTA proceeds.  A peer that never
// signals (its process died) must not hang the GPU: after ~10 s of %globaltimer the wait traps,
// the launch fails and the context is poisoned (ERUNTIME, then ESTATE).
__device__ __forceinline__ void wait_all(const EpPeers& pr, const EpOffsets& of, int phase, unsigned long long epoch) {
  if (threadIdx.x < (unsigned)pr.G) {
    const unsigned long long* f = sig_of(pr.base[pr.me], of, phase, threadIdx.x);
    unsigned long long t0 = 0;
    for (unsigned n = 0; ld_acquire_sys(f) < epoch; ++n) {
      __nanosleep(64);
      if ((n & 0xFFFF) == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (!t0) t0 = t;
        else if (t - t0 > 10000000000ull) __trap();
      }
    }
  }
  __syncthreads();
  __threadfence_system();
}

// every CTA's stores are fenced system-wide before the last CTA to finish signals all peers
__device__ __forceinline__ void signal_when_done(const EpPeers& pr, const EpOffsets& of, int phase,
                                                 unsigned long long epoch) {
  __threadfence_system();
  __syncthreads();
  __shared__ unsigned int last;
  if (threadIdx.x == 0) {
    unsigned int* ctr = reinterpret_cast<unsigned int*>(pr.base[pr.me] + of.ctr) + phase;
    last = atomicAdd(ctr, 1u) == gridDim.x - 1;
    if (last) *ctr = 0;   // every CTA has arrived: reset for the next epoch
  }
  __syncthreads();
  if (last && threadIdx.x < (unsigned)pr.G) {
    __threadfence_system();
    st_release_sys(sig_of(pr.base[threadIdx.x], of, phase, pr.me), epoch);
  }
}

__device__ __forceinline__ void copy_row16(uint4* __restrict__ dst, const uint4* __restrict__ src, int n16, int lane) {
  for (int k = lane; k < n16; k += 32) dst[k] = __ldcg(src + k);
}

// ---------------------------------------------------------------- ids all-gather + publish
__global__ void __launch_bounds__(256) ep_ids_kernel(EpIdsParams p) {
  const int half = (int)(p.epoch & 1);
  if (p.push) {
    // my tokens' ids and weights into every rank's ids_all[half] at my offset
    for (int q = 0; q < p.pr.G; ++q) {
      int32_t* di = reinterpret_cast<int32_t*>(p.pr.base[q] + p.of.ids_all[half]) + (size_t)p.pr.me * p.BlK;
      float* dw = reinterpret_cast<float*>(p.pr.base[q] + p.of.w_all[half]) + (size_t)p.pr.me * p.BlK;
      for (int i = threadIdx.x; i < p.BlK; i += blockDim.x) {
        di[i] = p.ids[i];
        dw[i] = p.w[i];
      }
    }
    signal_when_done(p.pr, p.of, kEpPhIds, p.epoch);
    wait_all(p.pr, p.of, kEpPhIds, p.epoch);
  }
  // publish the whole batch's routing to the host (tagged mailbox words, see RouterParams)
  const int32_t* ia = reinterpret_cast<const int32_t*>(p.pr.base[p.pr.me] + p.of.ids_all[half]);
  const float* wa = reinterpret_cast<const float*>(p.pr.base[p.pr.me] + p.of.w_all[half]);
  const unsigned long long tag = (unsigned long long)p.seq << 32;
  for (int i = threadIdx.x; i < p.TK; i += blockDim.x) {
    p.mb_ids[i] = tag | (uint32_t)__ldcg(ia + i);
    p.mb_w[i] = tag | __float_as_uint(__ldcg(wa + i));
  }
}

void launch_ep_ids(const EpIdsParams& p, cudaStream_t s) { ep_ids_kernel<<<1, 256, 0, s>>>(p); }

// ---------------------------------------------------------------- dispatch
// Warp per entry: my local token d_tok[e] -> rank d_dst[e] at row d_row[e] of its recv[half]
// (peer mode) or row e of the NCCL send buffer (entries are grouped by destination).  Then the
// sub-batch routing this rank computes is gathered from ids_all into ids_out / w_out.
__global__ void __launch_bounds__(256) ep_dispatch_kernel(EpDispatchParams p) {
  const int half = (int)(p.epoch & 1);
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int n16 = p.d / 8;   // bf16 row in 16-byte units
  for (int e = warp; e < p.n_disp; e += nwarps) {
    const int tok = p.d_tok[e];
    const uint4* src = reinterpret_cast<const uint4*>(p.h + (size_t)tok * p.d);
    uint4* dst = p.push ? reinterpret_cast<uint4*>(p.pr.base[p.d_dst[e]] + p.of.recv[half]) + (size_t)p.d_row[e] * n16
                        : reinterpret_cast<uint4*>(p.sendbuf) + (size_t)e * n16;
    copy_row16(dst, src, n16, lane);
  }
  const int32_t* ia = reinterpret_cast<const int32_t*>(p.pr.base[p.pr.me] + p.of.ids_all[half]);
  const float* wa = reinterpret_cast<const float*>(p.pr.base[p.pr.me] + p.of.w_all[half]);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < p.n_sub * p.K; i += gridDim.x * blockDim.x) {
    const int j = i / p.K, k = i - j * p.K;
    const int t = p.sub[j];
    p.ids_out[i] = __ldcg(ia + (size_t)t * p.K + k);
    p.w_out[i] = __ldcg(wa + (size_t)t * p.K + k);
  }
  if (p.push) signal_when_done(p.pr, p.of, kEpPhDispatch, p.epoch);
}

void launch_ep_dispatch(const EpDispatchParams& p, int grid, cudaStream_t s) {
  ep_dispatch_kernel<<<grid, 256, 0, s>>>(p);
}

// ---------------------------------------------------------------- wait (before the expert kernels)
__global__ void ep_wait_kernel(EpPeers pr, EpOffsets of, int phase, unsigned long long epoch) {
  wait_all(pr, of, phase, epoch);
}

void launch_ep_wait(const EpPeers& pr, const EpOffsets& of, int phase, unsigned long long epoch, cudaStream_t s) {
  ep_wait_kernel<<<1, 32, 0, s>>>(pr, of, phase, epoch);
}

// ---------------------------------------------------------------- combine send
// Warp per computed row j of the sub-batch output: -> rank c_dst[j], row c_row[j] of comb[half].
__global__ void __launch_bounds__(256) ep_combine_kernel(EpCombineParams p) {
  const int half = (int)(p.epoch & 1);
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int n16 = p.d / 4;   // fp32 row
  for (int j = warp; j < p.n_sub; j += nwarps) {
    const uint4* src = reinterpret_cast<const uint4*>(p.ysub + (size_t)j * p.d);
    uint4* dst = reinterpret_cast<uint4*>(p.pr.base[p.c_dst[j]] + p.of.comb[half]) + (size_t)p.c_row[j] * n16;
    copy_row16(dst, src, n16, lane);
  }
  signal_when_done(p.pr, p.of, kEpPhCombine, p.epoch);
}

void launch_ep_combine(const EpCombineParams& p, int grid, cudaStream_t s) {
  ep_combine_kernel<<<grid, 256, 0, s>>>(p);
}

// ---------------------------------------------------------------- reduce at the token owner
// y[i] = (h[i] if residual) + sum of my comb[half] rows r_row[r_off[i] .. r_off[i+1]) in list
// order (expert-owner rank ascending): a fixed order, so results are bitwise repeatable.
__global__ void __launch_bounds__(256) ep_reduce_kernel(EpReduceParams p) {
  if (p.wait) wait_all(p.pr, p.of, kEpPhCombine, p.epoch);
  const int half = (int)(p.epoch & 1);
  const float4* comb = reinterpret_cast<const float4*>(p.pr.base[p.pr.me] + p.of.comb[half]);
  const int n4 = p.d / 4;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < p.Bl * n4; idx += gridDim.x * blockDim.x) {
    const int i = idx / n4, c = idx - i * n4;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (p.residual) {
      const uint2 hv = *reinterpret_cast<const uint2*>(p.h + (size_t)i * p.d + 4 * c);
      acc.x = __uint_as_float(hv.x << 16);
      acc.y = __uint_as_float(hv.x & 0xFFFF0000u);
      acc.z = __uint_as_float(hv.y << 16);
      acc.w = __uint_as_float(hv.y & 0xFFFF0000u);
    }
    const int r1 = p.r_off[i + 1];
    for (int r = p.r_off[i]; r < r1; ++r) {
      const float4 v = __ldcg(comb + (size_t)p.r_row[r] * n4 + c);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    reinterpret_cast<float4*>(p.y)[(size_t)i * n4 + c] = acc;
  }
}

void launch_ep_reduce(const EpReduceParams& p, int grid, cudaStream_t s) {
  ep_reduce_kernel<<<grid, 256, 0, s>>>(p);
}

// ---------------------------------------------------------------- replicated-token all-reduce
// Each rank stores its partial y into slot [me] of every rank's red[half]; once all G slots of
// its own region are published, every rank sums them in rank order (identical bits everywhere).
__global__ void __launch_bounds__(256) ep_allreduce_kernel(EpAllreduceParams p) {
  const int half = (int)(p.epoch & 1);
  const size_t n4 = (size_t)p.n / 4;
  const size_t slot4 = (size_t)p.slot_floats / 4;
  const float4* y4 = reinterpret_cast<const float4*>(p.y);
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    const float4 v = y4[i];
    for (int q = 0; q < p.pr.G; ++q)
      reinterpret_cast<float4*>(p.pr.base[q] + p.of.red[half])[(size_t)p.pr.me * slot4 + i] = v;
  }
  signal_when_done(p.pr, p.of, kEpPhReduce, p.epoch);
  wait_all(p.pr, p.of, kEpPhReduce, p.epoch);
  const float4* red = reinterpret_cast<const float4*>(p.pr.base[p.pr.me] + p.of.red[half]);
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    float4 acc = __ldcg(red + i);
    for (int q = 1; q < p.pr.G; ++q) {
      const float4 v = __ldcg(red + (size_t)q * slot4 + i);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    reinterpret_cast<float4*>(p.y)[i] = acc;
  }
}

void launch_ep_allreduce(const EpAllreduceParams& p, int grid, cudaStream_t s) {
  ep_allreduce_kernel<<<grid, 256, 0, s>>>(p);
}

}  // namespace moepic
