// K1 router + next-layer predictor (Eq. 2; Eq. 3).
//
// Phase 1: one warp per (matrix, token, expert) logit in fp64 canonical order C.R (DESIGN.md
// R1): chunk c of 8 consecutive k is lane c%32's; lanes add exact bf16*bf16 products in
// increasing k; xor-butterfly 16,8,4,2,1.
// Phase 2 (last CTA, ticket): top-K per token by (logit desc, id asc) with warp-shuffle argmax
// rounds; Eq. 2 weights (one exp per lane); ids / weights published to device memory and to the
// mapped-pinned mailbox, system fence, then `seq_route` — the host starts planning copies now.
// Phase 3 (same CTA): batch ranking of the next layer's experts (reading Q9) by warp ballots
// (rank_j = #experts whose key precedes j's), published with `seq_rank`.
// Batches above kRouterSplitB (prefill) run phases 2-3 in k1_select instead: one warp per token,
// so the selection is spread over the whole GPU rather than one CTA.
#include "kernels.hpp"
#include "device_utils.cuh"

#include <cstdio>

namespace moepic {

__device__ __forceinline__ bool key_better(double av, int aid, double bv, int bid) {
  return av > bv || (av == bv && aid < bid);
}

// top-K of row[0..N) by (value desc, id asc) using one warp; writes ids_out[0..K) on lane 0
// and returns on every lane the selection bitmap of this lane's experts.
__device__ void warp_topk(const double* row, int N, int K, int* ids_out, unsigned* taken_bits) {
  const int lane = threadIdx.x & 31;
  unsigned taken = 0;  // bit q <-> expert lane + 32 q
  double vals[kMaxN / 32];
  for (int q = 0, j = lane; j < N; ++q, j += 32) vals[q] = row[j];
  for (int r = 0; r < K; ++r) {
    double bv = -INFINITY;
    int bid = 0x7fffffff;
#pragma unroll
    for (int q = 0; q < kMaxN / 32; ++q) {
      const int j = lane + 32 * q;
      if (j < N && !(taken & (1u << q)) && key_better(vals[q], j, bv, bid)) { bv = vals[q]; bid = j; }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oid = __shfl_xor_sync(0xffffffffu, bid, o);
      if (key_better(ov, oid, bv, bid)) { bv = ov; bid = oid; }
    }
    if ((bid & 31) == lane) taken |= 1u << (bid >> 5);
    if (lane == 0) ids_out[r] = bid;
  }
  *taken_bits = taken;
}

__global__ void __launch_bounds__(256) k1_router(RouterParams p) {
  __shared__ int s_last;
  __shared__ int s_cnt[kMaxN];
  __shared__ double s_max[kMaxN];
  __shared__ int s_topk[8][64];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const int BN = p.B * p.N;
  const int total = BN * 2;
  const int n_chunks = p.d >> 3;
  stamp_start(p.tstamp);

  // ---- phase 1: one warp per (matrix, token, expert) logit
  const int gw = blockIdx.x * nwarps + warp;
  if (gw < total) {
    const int m = gw / BN;
    const int rem = gw - m * BN;
    const int b = rem / p.N;
    const int j = rem - b * p.N;
    const uint16_t* W = m == 0 ? p.W0 : p.W1;
    if (W != nullptr) {
      const uint4* hv = reinterpret_cast<const uint4*>(p.h + (size_t)b * p.d);
      const uint4* wv = reinterpret_cast<const uint4*>(W + (size_t)j * p.d);
      double acc = 0.0;
#pragma unroll 4
      for (int c = lane; c < n_chunks; c += 32) {
        const uint4 a = __ldg(hv + c), w = __ldg(wv + c);
        float fa[8], fw[8];
        unpack8(a, fa);
        unpack8(w, fw);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc += (double)fa[e] * (double)fw[e];  // exact product
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) acc = acc + __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) p.logits[(size_t)m * BN + rem] = acc;
    }
  }
  if (p.B > kRouterSplitB) {   // large batch: k1_select does phases 2 and 3
    stamp_end(p.tstamp);
    return;
  }
  // ---- the last CTA to finish phase 1 does the selection
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(p.ticket, 1u);
    s_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) {
    stamp_end(p.tstamp);
    return;
  }
  __threadfence();
  const double* L0 = p.logits;
  const double* L1 = p.logits + BN;

  // ---- phase 2: routing
  if (p.W0 != nullptr) {
    for (int b = warp; b < p.B; b += nwarps) {
      unsigned bits;
      const double* row = L0 + (size_t)b * p.N;
      warp_topk(row, p.N, p.K, s_topk[warp], &bits);
      __syncwarp();
      const double mx = row[s_topk[warp][0]];
      double ek = 0.0, part = 0.0;
      if (lane < p.K) ek = exp(row[s_topk[warp][lane]] - mx);
      if (p.renorm) {
        part = ek;
      } else {
        for (int j = lane; j < p.N; j += 32) part += exp(row[j] - mx);
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      if (lane < p.K) {
        p.ids[b * p.K + lane] = s_topk[warp][lane];
        p.w[b * p.K + lane] = (float)(ek / part);
      }
      __syncwarp();
    }
    __syncthreads();
    const unsigned long long tag = (unsigned long long)p.seq << 32;
    for (int i = threadIdx.x; i < p.B * p.K; i += blockDim.x) {   // coalesced PCIe bursts
      p.mb_ids[i] = tag | (uint32_t)p.ids[i];
      p.mb_w[i] = tag | __float_as_uint(p.w[i]);
    }
  }

  // ---- phase 3: next-layer ranking, key = (count desc, max logit desc, id asc)
  if (p.W1 != nullptr) {
    for (int j = threadIdx.x; j < p.N; j += blockDim.x) {
      s_cnt[j] = 0;
      double mx = -INFINITY;
      for (int b = 0; b < p.B; ++b) mx = fmax(mx, L1[(size_t)b * p.N + j]);
      s_max[j] = mx;
    }
    __syncthreads();
    for (int b = warp; b < p.B; b += nwarps) {
      unsigned bits;
      warp_topk(L1 + (size_t)b * p.N, p.N, p.K, s_topk[warp], &bits);
      for (int q = 0, j = lane; j < p.N; ++q, j += 32)
        if (bits & (1u << q)) atomicAdd(&s_cnt[j], 1);
    }
    __syncthreads();
    for (int j = warp; j < p.N; j += nwarps) {
      const int cj = s_cnt[j];
      const double mj = s_max[j];
      int r = 0;
      for (int o0 = 0; o0 < p.N; o0 += 32) {
        const int o = o0 + lane;
        bool before = false;
        if (o < p.N) {
          const int co = s_cnt[o];
          const double mo = s_max[o];
          before = (co > cj) || (co == cj && (mo > mj || (mo == mj && o < j)));
        }
        r += __popc(__ballot_sync(0xffffffffu, before));
      }
      if (lane == 0) p.ranking[r] = j;
    }
    __syncthreads();
    const unsigned long long tag = (unsigned long long)p.seq << 32;
    for (int i = threadIdx.x; i < p.N; i += blockDim.x) p.mb_rank[i] = tag | (uint32_t)p.ranking[i];
  }
  if (threadIdx.x == 0) *p.ticket = 0u;
  stamp_end(p.tstamp);
}

// order-preserving map double -> u64 (larger double <-> larger key; 0 is below every logit)
__device__ __forceinline__ unsigned long long order_key(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double order_val(unsigned long long k) {
  return __longlong_as_double((long long)((k & 0x8000000000000000ull) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k));
}

// Large-batch selection (prefill): one warp per token for the routing top-K / Eq. 2 weights and
// the predicted top-K (Eq. 3 counts and max logits, reading Q9); the last CTA ranks the next
// layer's experts.  Same keys and arithmetic as phases 2-3 of k1_router.
__global__ void __launch_bounds__(256) k1_select(RouterParams p) {
  __shared__ int s_last;
  __shared__ int s_topk[8][64];
  __shared__ int s_cnt[kMaxN];
  __shared__ unsigned long long s_max[kMaxN];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int BN = p.B * p.N;
  const double* L0 = p.logits;
  const double* L1 = p.logits + BN;
  const unsigned long long tag = (unsigned long long)p.seq << 32;
  const int b = blockIdx.x * 8 + warp;
  stamp_start(p.tstamp);
  for (int j = threadIdx.x; j < p.N; j += blockDim.x) {
    s_cnt[j] = 0;
    s_max[j] = 0ull;
  }
  __syncthreads();
  if (b < p.B) {
    if (p.W0 != nullptr) {
      unsigned bits;
      const double* row = L0 + (size_t)b * p.N;
      warp_topk(row, p.N, p.K, s_topk[warp], &bits);
      __syncwarp();
      const double mx = row[s_topk[warp][0]];
      double ek = 0.0, part = 0.0;
      if (lane < p.K) ek = exp(row[s_topk[warp][lane]] - mx);
      if (p.renorm) {
        part = ek;
      } else {
        for (int j = lane; j < p.N; j += 32) part += exp(row[j] - mx);
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      if (lane < p.K) {
        const int id = s_topk[warp][lane];
        const float wv = (float)(ek / part);
        p.ids[b * p.K + lane] = id;
        p.w[b * p.K + lane] = wv;
        p.mb_ids[b * p.K + lane] = tag | (uint32_t)id;
        p.mb_w[b * p.K + lane] = tag | __float_as_uint(wv);
      }
      __syncwarp();
    }
    if (p.W1 != nullptr) {
      unsigned bits;
      const double* row = L1 + (size_t)b * p.N;
      warp_topk(row, p.N, p.K, s_topk[warp], &bits);
      for (int q = 0, j = lane; j < p.N; ++q, j += 32) {
        if (bits & (1u << q)) atomicAdd(&s_cnt[j], 1);
        atomicMax(&s_max[j], order_key(row[j]));
      }
    }
  }
  if (p.W1 == nullptr) {
    stamp_end(p.tstamp);
    return;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < p.N; j += blockDim.x) {   // one global atomic per expert per CTA
    if (s_cnt[j]) atomicAdd(&p.sel_cnt[j], s_cnt[j]);
    if (s_max[j]) atomicMax(&p.sel_max[j], s_max[j]);
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(p.ticket2, 1u);
    s_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) {
    stamp_end(p.tstamp);
    return;
  }
  __threadfence();
  // ranking: key = (count desc, max logit desc, id asc)
  const int nwarps = blockDim.x >> 5;
  for (int j = warp; j < p.N; j += nwarps) {
    const int cj = *((volatile int*)&p.sel_cnt[j]);
    const double mj = order_val(*((volatile unsigned long long*)&p.sel_max[j]));
    int r = 0;
    for (int o0 = 0; o0 < p.N; o0 += 32) {
      const int o = o0 + lane;
      bool before = false;
      if (o < p.N) {
        const int co = *((volatile int*)&p.sel_cnt[o]);
        const double mo = order_val(*((volatile unsigned long long*)&p.sel_max[o]));
        before = (co > cj) || (co == cj && (mo > mj || (mo == mj && o < j)));
      }
      r += __popc(__ballot_sync(0xffffffffu, before));
    }
    if (lane == 0) p.ranking[r] = j;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < p.N; i += blockDim.x) {
    p.mb_rank[i] = tag | (uint32_t)p.ranking[i];
    p.sel_cnt[i] = 0;
    p.sel_max[i] = 0ull;
  }
  if (threadIdx.x == 0) *p.ticket2 = 0u;
  stamp_end(p.tstamp);
}

// Small kernels run between K2 launches that need ~200 KB of shared memory: asking for the
// maximum shared-memory carveout keeps the SM's L1/shared split unchanged between them.
cudaError_t router_init() {
  cudaError_t e = cudaFuncSetAttribute(k1_router, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaError_t f = cudaFuncSetAttribute(k1_select, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  return e != cudaSuccess ? e : f;
}

void launch_router(const RouterParams& p, cudaStream_t s) {
  const int warps = 2 * p.B * p.N;
  const int grid = (warps + 7) / 8;
  k1_router<<<grid, 256, 0, s>>>(p);
  if (p.B > kRouterSplitB) k1_select<<<(p.B + 7) / 8, 256, 0, s>>>(p);
}

}  // namespace moepic
