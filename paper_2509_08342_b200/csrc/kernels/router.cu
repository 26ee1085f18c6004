// K1 router + next-layer predictor (Eq. 2; Eq. 3).
//
// Phase 1: one warp per (matrix, token, expert) logit in fp64 canonical order C.R (DESIGN.md
// R1): chunk c of 8 consecutive k is lane c%32's; lanes add exact bf16*bf16 products in
// increasing k; xor-butterfly 16,8,4,2,1.
// Phase 2 (last CTA, ticket): top-K per token by (logit desc, id asc): every (token, expert) pair
// counts the experts whose key precedes its own in shared memory (all pairs in parallel; the
// single-warp argmax rounds this replaced cost 5.6 us for N = 128, K = 8); Eq. 2 weights (one
// exp per lane); ids / weights published to device memory and to the mapped-pinned mailbox as
// self-validating words — the host starts planning copies now.
// Phase 3 (same CTA): batch ranking of the next layer's experts (reading Q9): predicted top-K
// counts by the same rank counting, then rank_j = #experts whose key precedes j's.
// Batches above kRouterSplitB (prefill) run phases 2-3 in k1_select instead: one warp per token,
// so the selection is spread over the whole GPU rather than one CTA.
#include "kernels.hpp"
#include "device_utils.cuh"

#include <cstdio>

namespace moepic {

// Mailbox words go to mapped pinned host memory with write-through stores: a plain store may sit
// in L2 as a dirty system-memory line until later traffic evicts it (the host then saw the
// routing hundreds of microseconds late, in proportion to the layer's HBM traffic; measured with
// MOEPIC_TIMELINE), and a system-scope fence waits behind the saturated host->device link.
__device__ __forceinline__ void st_wt(unsigned long long* p, unsigned long long v) {
  asm volatile("st.global.wt.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

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

// order-preserving map double -> u64 (larger double <-> larger key; 0 is below every logit)
__device__ __forceinline__ unsigned long long order_key(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double order_val(unsigned long long k) {
  return __longlong_as_double((long long)((k & 0x8000000000000000ull) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k));
}

// key order of the routing / prediction top-K: (logit desc, id asc) — a strict total order
__device__ __forceinline__ bool logit_before(double lo, int o, double lj, int j) {
  return lo > lj || (lo == lj && o < j);
}

// Rank counting (phases 2-3): the rank of item j among N under a strict total order is the number
// of items that precede it.  Each warp holds NQ = N/32 items per lane in registers and walks a
// slice of the N comparands (shared-memory broadcasts), so one load feeds NQ comparisons; a
// batch of nb rows spreads over the warps (nb < warps: the warps of a row split its comparands
// and add their counts in shared memory).  fn(t, j, r) receives every rank.
struct RowLogits {   // key of (row t, item j): (logit desc, id asc)
  const double* rows;
  int N;
  __device__ double key(int t, int j) const { return rows[t * N + j]; }
  __device__ static bool before(double ko, int o, double kj, int j) { return logit_before(ko, o, kj, j); }
};
struct RankKey {     // (count desc, order-preserving max-logit key desc, id asc), one row
  const int* cnt;
  const unsigned long long* mx;
  struct K { int c; unsigned long long m; };
  __device__ K key(int, int j) const { return K{cnt[j], mx[j]}; }
  __device__ static bool before(const K& ko, int o, const K& kj, int j) {
    return ko.c > kj.c || (ko.c == kj.c && (ko.m > kj.m || (ko.m == kj.m && o < j)));
  }
};

template <int NQ, class R, class Fn>
__device__ void rank_rows_t(const R& keys, int nb, int N, int* s_rank, Fn& fn) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int wpt = nb >= nw ? 1 : nw / nb;
  if (wpt > 1) {
    for (int i = threadIdx.x; i < nb * N; i += blockDim.x) s_rank[i] = 0;
    __syncthreads();
  }
  using KT = decltype(keys.key(0, 0));
  for (int t = warp / wpt; t < nb; t += nw / wpt) {
    const int sl = warp % wpt;
    const int o0 = sl * N / wpt, o1 = (sl + 1) * N / wpt;
    KT kj[NQ];
    int r[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int j = lane + 32 * q;
      kj[q] = keys.key(t, j < N ? j : 0);
      r[q] = 0;
    }
#pragma unroll 4
    for (int o = o0; o < o1; ++o) {
      const KT ko = keys.key(t, o);
#pragma unroll
      for (int q = 0; q < NQ; ++q) r[q] += R::before(ko, o, kj[q], lane + 32 * q) ? 1 : 0;
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int j = lane + 32 * q;
      if (j >= N) continue;
      if (wpt > 1) atomicAdd(&s_rank[t * N + j], r[q]);
      else fn(t, j, r[q]);
    }
  }
  if (wpt > 1) {
    __syncthreads();
    for (int i = threadIdx.x; i < nb * N; i += blockDim.x) fn(i / N, i % N, s_rank[i]);
  }
}

template <class R, class Fn>
__device__ void rank_rows(const R& keys, int nb, int N, int* s_rank, Fn& fn) {
  if (N <= 32) rank_rows_t<1>(keys, nb, N, s_rank, fn);
  else if (N <= 64) rank_rows_t<2>(keys, nb, N, s_rank, fn);
  else if (N <= 128) rank_rows_t<4>(keys, nb, N, s_rank, fn);
  else if (N <= 256) rank_rows_t<8>(keys, nb, N, s_rank, fn);
  else rank_rows_t<16>(keys, nb, N, s_rank, fn);
}

constexpr int kSelBuf = 2048;   // logits staged in shared memory per selection pass (16 KB)

// CPL = chunks of 8 per lane the phase-1 loads are sized for: 16 covers d <= 4096; 8 (d <= 2048)
// keeps the registers low enough for two CTAs per SM when a batch needs several waves
template <int CPL>
__global__ void __launch_bounds__(256, CPL <= 8 ? 2 : 1) k1_router(RouterParams p) {
  __shared__ int s_last;
  __shared__ double s_l[kSelBuf];
  __shared__ int s_cnt[kMaxN];
  __shared__ double s_max[kMaxN];
  __shared__ unsigned long long s_key[kMaxN];
  __shared__ int s_rank[kSelBuf];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const int BN = p.B * p.N;
  const int total = BN * 2;
  const int n_chunks = p.d >> 3;
  stamp_start(p.tstamp);
  if (p.dbg && threadIdx.x == 0) atomicMin(p.dbg, gtimer());

  // ---- phase 1: one warp per (matrix, token, expert) logit.  Every load of the lane's chunks
  // is issued before the first add (one memory latency), then the lane adds its exact products
  // in increasing k (C.R), then the xor butterfly.
  const int gw = blockIdx.x * nwarps + warp;
  if (gw >= total || (gw < total && (gw / BN == 0 ? p.W0 : p.W1) == nullptr))
    asm volatile("griddepcontrol.wait;" ::: "memory");   // warps without a logit still order after it
  if (gw < total) {
    const int m = gw / BN;
    const int rem = gw - m * BN;
    const int b = rem / p.N;
    const int j = rem - b * p.N;
    const uint16_t* W = m == 0 ? p.W0 : p.W1;
    if (W != nullptr) {
      const uint4* hv = reinterpret_cast<const uint4*>(p.h + (size_t)b * p.d);
      const uint4* wv = reinterpret_cast<const uint4*>(W + (size_t)j * p.d);
      uint4 wr[CPL], hr[CPL];
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        const int c = lane + 32 * q;
        if (c < n_chunks) wr[q] = __ldg(wv + c);
      }
      // programmatic dependent launch: the router weights do not depend on the previous kernel
      // (the layer before's final K2), h does -- wait for that grid only now (no-op otherwise)
      asm volatile("griddepcontrol.wait;" ::: "memory");
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        const int c = lane + 32 * q;
        if (c < n_chunks) hr[q] = __ldg(hv + c);
      }
      double acc = 0.0;
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        if (lane + 32 * q < n_chunks) {
          float fa[8], fw[8];
          unpack8(hr[q], fa);
          unpack8(wr[q], fw);
#pragma unroll
          for (int e = 0; e < 8; ++e) acc += (double)fa[e] * (double)fw[e];  // exact product
        }
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
  if (p.dbg && threadIdx.x == 0) atomicMax(p.dbg + 1, gtimer());
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
  if (p.dbg && threadIdx.x == 0) p.dbg[2] = gtimer();
  const double* L0 = p.logits;
  const double* L1 = p.logits + BN;
  const int tpg = kSelBuf / p.N;   // tokens per staged group

  // ---- phase 2: routing.  Every (token, expert) pair computes its rank under the key
  // (logit desc, id asc) by counting the experts that precede it (a strict total order, so the
  // ranks are a permutation); the K experts with rank < K are the top-K in key order.
  if (p.W0 != nullptr) {
    for (int b0 = 0; b0 < p.B; b0 += tpg) {
      const int nb = min(tpg, p.B - b0);
      __syncthreads();
      for (int i = threadIdx.x; i < nb * p.N; i += blockDim.x) s_l[i] = L0[(size_t)b0 * p.N + i];
      __syncthreads();
      int32_t* ids = p.ids + (size_t)b0 * p.K;
      const int K = p.K;
      auto out = [&](int t, int j, int r) {
        if (r < K) ids[t * K + r] = j;
      };
      rank_rows(RowLogits{s_l, p.N}, nb, p.N, s_rank, out);
    }
    __syncthreads();
    if (p.dbg && threadIdx.x == 0) p.dbg[5] = gtimer();
    // Eq. 2 weights, one warp per token (lane k: exp(l_k - l_max); fixed butterfly sum)
    for (int b = warp; b < p.B; b += nwarps) {
      const double* row = L0 + (size_t)b * p.N;
      const double mx = row[p.ids[b * p.K]];
      double ek[2] = {0.0, 0.0}, part = 0.0;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int k = lane + 32 * q;
        if (k < p.K) ek[q] = exp(row[p.ids[b * p.K + k]] - mx);
      }
      if (p.renorm) {
        part = ek[0] + ek[1];
      } else {
        for (int j = lane; j < p.N; j += 32) part += exp(row[j] - mx);
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int k = lane + 32 * q;
        if (k < p.K) p.w[b * p.K + k] = (float)(ek[q] / part);
      }
    }
    __syncthreads();
    const unsigned long long tag = (unsigned long long)p.seq << 32;
    for (int i = threadIdx.x; i < p.B * p.K; i += blockDim.x) {   // coalesced PCIe bursts
      st_wt(p.mb_ids + i, tag | (uint32_t)p.ids[i]);
      st_wt(p.mb_w + i, tag | __float_as_uint(p.w[i]));
    }
    if (p.dbg && threadIdx.x == 0) p.dbg[3] = gtimer();
  }

  // ---- phase 3: next-layer ranking, key = (count desc, max logit desc, id asc) (Q9): counts of
  // the predicted top-K by the same rank counting, then every expert's rank under the key
  if (p.W1 != nullptr) {
    for (int j = threadIdx.x; j < p.N; j += blockDim.x) {
      s_cnt[j] = 0;
      double mx = -INFINITY;
      for (int b = 0; b < p.B; ++b) mx = fmax(mx, L1[(size_t)b * p.N + j]);
      s_max[j] = mx + 0.0;   // -0 -> +0: the integer key below must tie exactly where doubles do
    }
    for (int b0 = 0; b0 < p.B; b0 += tpg) {
      const int nb = min(tpg, p.B - b0);
      __syncthreads();
      for (int i = threadIdx.x; i < nb * p.N; i += blockDim.x) s_l[i] = L1[(size_t)b0 * p.N + i];
      __syncthreads();
      int32_t* ranking = p.B == 1 ? p.ranking : nullptr;
      const int K = p.K;
      auto out = [&](int, int j, int r) {
        if (ranking) ranking[r] = j;                 // B = 1: the ranking is the predicted order
        else if (r < K) atomicAdd(&s_cnt[j], 1);
      };
      rank_rows(RowLogits{s_l, p.N}, nb, p.N, s_rank, out);
    }
    __syncthreads();
    if (p.dbg && threadIdx.x == 0) p.dbg[6] = gtimer();
    // B = 1: c_j = [rank'_j < K] and max_j = l'_j, so (c desc, max desc, id asc) is the order of
    // (l' desc, id asc) itself, already written above.  B > 1: rank by the full key, with the
    // max logit as an order-preserving integer so one pass compares integers only.
    if (p.B > 1) {
      for (int j = threadIdx.x; j < p.N; j += blockDim.x) s_key[j] = order_key(s_max[j]);
      __syncthreads();
      int32_t* ranking = p.ranking;
      auto out = [&](int, int j, int r) { ranking[r] = j; };
      rank_rows(RankKey{s_cnt, s_key}, 1, p.N, s_rank, out);
    }
    __syncthreads();
    if (p.dbg && threadIdx.x == 0) p.dbg[7] = gtimer();
    const unsigned long long tag = (unsigned long long)p.seq << 32;
    for (int i = threadIdx.x; i < p.N; i += blockDim.x) st_wt(p.mb_rank + i, tag | (uint32_t)p.ranking[i]);
  }
  if (threadIdx.x == 0) *p.ticket = 0u;
  if (p.dbg && threadIdx.x == 0) p.dbg[4] = gtimer();
  stamp_end(p.tstamp);
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
        st_wt(p.mb_ids + b * p.K + lane, tag | (uint32_t)id);
        st_wt(p.mb_w + b * p.K + lane, tag | __float_as_uint(wv));
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
    st_wt(p.mb_rank + i, tag | (uint32_t)p.ranking[i]);
    p.sel_cnt[i] = 0;
    p.sel_max[i] = 0ull;
  }
  if (threadIdx.x == 0) *p.ticket2 = 0u;
  stamp_end(p.tstamp);
}

// Small kernels run between K2 launches that need ~200 KB of shared memory: asking for the
// maximum shared-memory carveout keeps the SM's L1/shared split unchanged between them.
cudaError_t router_init() {
  cudaError_t e = cudaFuncSetAttribute(k1_router<16>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaError_t f = cudaFuncSetAttribute(k1_router<8>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaError_t g = cudaFuncSetAttribute(k1_select, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  return e != cudaSuccess ? e : f != cudaSuccess ? f : g;
}

void launch_router(const RouterParams& p, cudaStream_t s, bool pdl) {
  const int warps = 2 * p.B * p.N;
  const int grid = (warps + 7) / 8;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  if (p.d > 2048) cudaLaunchKernelEx(&cfg, k1_router<16>, p);
  else cudaLaunchKernelEx(&cfg, k1_router<8>, p);
  if (p.B > kRouterSplitB) k1_select<<<(p.B + 7) / 8, 256, 0, s>>>(p);
}

}  // namespace moepic
