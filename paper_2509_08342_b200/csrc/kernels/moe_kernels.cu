// MoEpic sm_100a kernels: K1 router/predictor, K2 split-expert streaming SwiGLU, K3 combine.
//
// K1  (Eq. 2; Eq. 3): one warp per logit, fp64 canonical order C.R
//     (DESIGN.md): chunk c of 8 consecutive k is lane c%32's; lanes add exact bf16*bf16
//     products in increasing k; xor-butterfly 16,8,4,2,1.  The last CTA (ticket) selects the
//     top-K per token by (logit desc, id asc) with warp-shuffle argmax rounds, computes the
//     Eq. 2 weights, ranks the next layer's experts (Q9) and publishes ids / weights / ranking
//     to device memory and to the mapped-pinned mailbox (__threadfence_system, then seq).
// K2: each segment = contiguous rows of the row-interleaved expert
//     layout [gate_r | up_r | down[:,r]] (6d bytes per row).  Persistent grid; CTA c streams
//     its contiguous row range through a 4-stage cp.async.bulk (TMA 1-D) + mbarrier ring in
//     shared memory; per row tile: gate/up dot products (fp32) -> block reduce ->
//     a = silu(g) * u * w_gate -> y_partial += a * down_r.  Partials per (segment, CTA) go to a
//     workspace; there is no atomic, so the result is deterministic.
// K3  combine: y[b] = (h[b] if residual) + sum over segments / chunks in a fixed order.
#include "kernels.hpp"

#include <cuda_bf16.h>
#include <cstdio>

namespace moepic {

// ============================================================== small helpers
__device__ __forceinline__ float bf16lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16hi(uint32_t v) { return __uint_as_float(v & 0xFFFF0000u); }

__device__ __forceinline__ void unpack8(const uint4& v, float* f) {
  f[0] = bf16lo(v.x); f[1] = bf16hi(v.x);
  f[2] = bf16lo(v.y); f[3] = bf16hi(v.y);
  f[4] = bf16lo(v.z); f[5] = bf16hi(v.z);
  f[6] = bf16lo(v.w); f[7] = bf16hi(v.w);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// TMA 1-D bulk copy global -> shared, completion counted on the mbarrier (bytes % 16 == 0).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// ============================================================== K1 router
struct Key {  // (value desc, id asc)
  double v;
  int id;
};
__device__ __forceinline__ bool key_better(double av, int aid, double bv, int bid) {
  return av > bv || (av == bv && aid < bid);
}

// top-K of row[0..N) by (value desc, id asc) using one warp; writes ids_out[0..K) on lane 0
// and returns on every lane the selection bitmap of this lane's experts.
__device__ void warp_topk(const double* row, int N, int K, int* ids_out, unsigned* taken_bits) {
  const int lane = threadIdx.x & 31;
  unsigned taken = 0;  // bit q <-> expert lane + 32 q
  for (int r = 0; r < K; ++r) {
    double bv = -INFINITY;
    int bid = 0x7fffffff;
    for (int q = 0, j = lane; j < N; ++q, j += 32) {
      if (taken & (1u << q)) continue;
      double v = row[j];
      if (key_better(v, j, bv, bid)) { bv = v; bid = j; }
    }
    for (int o = 16; o; o >>= 1) {
      double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      int oid = __shfl_xor_sync(0xffffffffu, bid, o);
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
      for (int c = lane; c < n_chunks; c += 32) {
        uint4 a = __ldg(hv + c), w = __ldg(wv + c);
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
  // ---- last CTA does the selection
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = atomicAdd(p.ticket, 1u);
    s_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const double* L0 = p.logits;
  const double* L1 = p.logits + BN;
  if (p.W0 != nullptr) {
    for (int b = warp; b < p.B; b += nwarps) {
      unsigned bits;
      warp_topk(L0 + (size_t)b * p.N, p.N, p.K, s_topk[warp], &bits);
      __syncwarp();
      if (lane == 0) {
        const double* row = L0 + (size_t)b * p.N;
        double mx = row[s_topk[warp][0]];
        double den = 0.0;
        if (p.renorm) {
          for (int k = 0; k < p.K; ++k) den += exp(row[s_topk[warp][k]] - mx);
        } else {
          for (int j = 0; j < p.N; ++j) den += exp(row[j] - mx);
        }
        for (int k = 0; k < p.K; ++k) {
          int e = s_topk[warp][k];
          float wk = (float)(exp(row[e] - mx) / den);
          p.ids[b * p.K + k] = e;
          p.w[b * p.K + k] = wk;
          p.mb_ids[b * p.K + k] = e;
          p.mb_w[b * p.K + k] = wk;
        }
      }
      __syncwarp();
    }
  }
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
    // rank_j = #{j' : key(j') before key(j)}, key = (count desc, max logit desc, id asc)
    for (int j = threadIdx.x; j < p.N; j += blockDim.x) {
      int r = 0;
      const int cj = s_cnt[j];
      const double mj = s_max[j];
      for (int o = 0; o < p.N; ++o) {
        const int co = s_cnt[o];
        const double mo = s_max[o];
        r += (co > cj) || (co == cj && (mo > mj || (mo == mj && o < j)));
      }
      p.ranking[r] = j;
      p.mb_rank[r] = j;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *p.ticket = 0u;
    __threadfence_system();
    *p.mb_seq = p.seq;
    __threadfence_system();
  }
}

void launch_router(const RouterParams& p, cudaStream_t s) {
  const int warps = 2 * p.B * p.N;
  const int grid = (warps + 7) / 8;
  k1_router<<<grid, 256, 0, s>>>(p);
}

// ============================================================== K2 split-expert decode
int k2_rows_per_tile(int d) {
  if (d > 2048) return 2;
  if (d > 1024) return 4;
  if (d > 512) return 8;
  return 16;
}
static int k2_cpt(int d) { return (d / 8 + kK2Threads - 1) / kK2Threads; }
int k2_max_tokens(int d) { return k2_rows_per_tile(d) == 16 ? 2 : 4; }
size_t k2_smem_bytes(int d) {
  const int RS = k2_rows_per_tile(d);
  const int TBmax = 4;
  size_t stage = (size_t)kK2Stages * RS * 6 * d;
  return stage + kK2Stages * sizeof(uint64_t) + (size_t)(kK2Threads / 32) * 2 * 16 * TBmax * sizeof(float) +
         (size_t)16 * TBmax * sizeof(float) + 128;
}

struct TileIt {
  int s;
  int64_t row;
};

template <int TB, int CPT, int RS>
__global__ void __launch_bounds__(kK2Threads, 1) k2_split_expert(const __grid_constant__ K2Params p) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int NW = kK2Threads / 32;
  const int d = p.d;
  const int rowb = 6 * d;
  const int tileb = RS * rowb;
  uint8_t* stages = smem;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + (size_t)kK2Stages * tileb);
  float* red = reinterpret_cast<float*>(mbar + kK2Stages);   // [NW][2][RS][TB]
  float* act = red + NW * 2 * RS * TB;                        // [RS][TB]
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int64_t R = p.total_rows;
  const int64_t G = gridDim.x;
  const int64_t r0 = k2_row_lo(blockIdx.x, R, G), r1 = k2_row_lo(blockIdx.x + 1, R, G);
  if (r0 >= r1) return;

  if (tid == 0) {
    for (int i = 0; i < kK2Stages; ++i) mbar_init(&mbar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  auto seg_end = [&](int s) -> int64_t { return (int64_t)p.segs[s].row_begin + p.segs[s].nrows; };
  TileIt start;
  start.s = 0;
  while (seg_end(start.s) <= r0) ++start.s;
  start.row = r0;
  // next tile from iterator: [row, e) within one segment
  auto tile_end = [&](const TileIt& it) -> int64_t {
    int64_t e = it.row + RS;
    int64_t se = seg_end(it.s);
    if (e > se) e = se;
    if (e > r1) e = r1;
    return e;
  };
  auto advance = [&](TileIt& it) {
    int64_t e = tile_end(it);
    it.row = e;
    if (e >= seg_end(it.s)) ++it.s;
  };

  // ---- producer prologue (thread 0): fill every stage
  TileIt pit = start;
  uint64_t pol = 0;
  if (tid == 0) {
    pol = evict_first_policy();
    for (int st = 0; st < kK2Stages && pit.row < r1; ++st) {
      const int64_t e = tile_end(pit);
      const Seg& sg = p.segs[pit.s];
      const uint32_t bytes = (uint32_t)((e - pit.row) * rowb);
      mbar_expect_tx(&mbar[st], bytes);
      bulk_g2s(stages + (size_t)st * tileb, sg.base + (pit.row - sg.row_begin) * rowb, bytes, &mbar[st], pol);
      advance(pit);
    }
  }

  float yacc[TB][CPT][8];
  float hreg[TB][CPT][8];
  float wgt[TB];
  int ntok = 0;
  int cur = -1;

  auto flush = [&](int s) {
    const Seg& sg = p.segs[s];
    const int ci = (int)blockIdx.x - sg.cta_first;
    float* dst = p.ws + sg.ws_off + (int64_t)ci * ntok * d;
#pragma unroll
    for (int t = 0; t < TB; ++t) {
      if (t < ntok) {
#pragma unroll
        for (int cc = 0; cc < CPT; ++cc) {
          const int c8 = tid + cc * kK2Threads;
          if (c8 * 8 < d) {
            float4* o = reinterpret_cast<float4*>(dst + (int64_t)t * d + c8 * 8);
            o[0] = make_float4(yacc[t][cc][0], yacc[t][cc][1], yacc[t][cc][2], yacc[t][cc][3]);
            o[1] = make_float4(yacc[t][cc][4], yacc[t][cc][5], yacc[t][cc][6], yacc[t][cc][7]);
          }
        }
      }
    }
  };

  TileIt it = start;
  int stage = 0;
  uint32_t phase = 0;
  int prev_stage = -1;
  while (it.row < r1) {
    const int s = it.s;
    const int64_t ta = it.row, tb = tile_end(it);
    const int nr = (int)(tb - ta);
    if (s != cur) {
      if (cur >= 0) flush(cur);
      cur = s;
      const Seg& sg = p.segs[s];
      ntok = 0;
      uint32_t m = sg.tok_mask;
#pragma unroll
      for (int t = 0; t < TB; ++t) {
        wgt[t] = 0.f;
        int b = 0;
        if (m) {
          b = __ffs(m) - 1;
          m &= m - 1;
          ++ntok;
          if (sg.expert >= 0) {
            for (int k = 0; k < p.K; ++k)
              if (p.ids[b * p.K + k] == sg.expert) wgt[t] = p.w[b * p.K + k];
          } else {
            wgt[t] = 1.f;
          }
        }
#pragma unroll
        for (int cc = 0; cc < CPT; ++cc) {
          const int c8 = tid + cc * kK2Threads;
          if (t < ntok && c8 * 8 < d) {
            uint4 v = __ldg(reinterpret_cast<const uint4*>(p.h + (size_t)b * d) + c8);
            unpack8(v, hreg[t][cc]);
          } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) hreg[t][cc][e] = 0.f;
          }
#pragma unroll
          for (int e = 0; e < 8; ++e) yacc[t][cc][e] = 0.f;
        }
      }
    }
    mbar_wait(&mbar[stage], phase);
    const uint8_t* tile = stages + (size_t)stage * tileb;

    // ---- phase 1: gate / up partial dots for this thread's columns
    float pg[RS][TB], pu[RS][TB];
#pragma unroll
    for (int r = 0; r < RS; ++r)
#pragma unroll
      for (int t = 0; t < TB; ++t) pg[r][t] = pu[r][t] = 0.f;
#pragma unroll
    for (int r = 0; r < RS; ++r) {
      if (r < nr) {
        const uint8_t* rowp = tile + (size_t)r * rowb;
#pragma unroll
        for (int cc = 0; cc < CPT; ++cc) {
          const int c8 = tid + cc * kK2Threads;
          if (c8 * 8 < d) {
            float g8[8], u8[8];
            unpack8(*reinterpret_cast<const uint4*>(rowp + c8 * 16), g8);
            unpack8(*reinterpret_cast<const uint4*>(rowp + 2 * d + c8 * 16), u8);
#pragma unroll
            for (int t = 0; t < TB; ++t) {
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                pg[r][t] = fmaf(g8[e], hreg[t][cc][e], pg[r][t]);
                pu[r][t] = fmaf(u8[e], hreg[t][cc][e], pu[r][t]);
              }
            }
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < RS; ++r)
#pragma unroll
      for (int t = 0; t < TB; ++t) {
        float a = pg[r][t], b = pu[r][t];
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          a += __shfl_xor_sync(0xffffffffu, a, o);
          b += __shfl_xor_sync(0xffffffffu, b, o);
        }
        if (lane == 0) {
          red[((warp * 2 + 0) * RS + r) * TB + t] = a;
          red[((warp * 2 + 1) * RS + r) * TB + t] = b;
        }
      }
    __syncthreads();
    // the previous stage is now free (every thread finished its phase 2): refill it
    if (tid == 0 && prev_stage >= 0 && pit.row < r1) {
      const int64_t e = tile_end(pit);
      const Seg& sg = p.segs[pit.s];
      const uint32_t bytes = (uint32_t)((e - pit.row) * rowb);
      mbar_expect_tx(&mbar[prev_stage], bytes);
      bulk_g2s(stages + (size_t)prev_stage * tileb, sg.base + (pit.row - sg.row_begin) * rowb, bytes,
               &mbar[prev_stage], pol);
      advance(pit);
    }
    if (tid < RS * TB) {
      const int r = tid / TB, t = tid - (tid / TB) * TB;
      float g = 0.f, u = 0.f;
#pragma unroll
      for (int w2 = 0; w2 < NW; ++w2) {
        g += red[((w2 * 2 + 0) * RS + r) * TB + t];
        u += red[((w2 * 2 + 1) * RS + r) * TB + t];
      }
      const float a = (r < nr && t < ntok) ? g / (1.f + __expf(-g)) * u * wgt[t] : 0.f;
      act[r * TB + t] = a;
    }
    __syncthreads();
    // ---- phase 2: y_partial += a * down_r
#pragma unroll
    for (int r = 0; r < RS; ++r) {
      if (r < nr) {
        const uint8_t* rowp = tile + (size_t)r * rowb + 4 * d;
#pragma unroll
        for (int cc = 0; cc < CPT; ++cc) {
          const int c8 = tid + cc * kK2Threads;
          if (c8 * 8 < d) {
            float d8[8];
            unpack8(*reinterpret_cast<const uint4*>(rowp + c8 * 16), d8);
#pragma unroll
            for (int t = 0; t < TB; ++t) {
              const float a = act[r * TB + t];
#pragma unroll
              for (int e = 0; e < 8; ++e) yacc[t][cc][e] = fmaf(a, d8[e], yacc[t][cc][e]);
            }
          }
        }
      }
    }
    prev_stage = stage;
    advance(it);
    if (++stage == kK2Stages) { stage = 0; phase ^= 1u; }
  }
  if (cur >= 0) flush(cur);
}

template <int TB, int CPT, int RS>
static void k2_launch_t(const K2Params& p, int grid, cudaStream_t s) {
  k2_split_expert<TB, CPT, RS><<<grid, kK2Threads, k2_smem_bytes(p.d), s>>>(p);
}

template <int CPT, int RS>
static void k2_dispatch_tb(const K2Params& p, int grid, int tb, cudaStream_t s) {
  switch (tb) {
    case 1: k2_launch_t<1, CPT, RS>(p, grid, s); break;
    case 2: k2_launch_t<2, CPT, RS>(p, grid, s); break;
    default:
      if constexpr (RS <= 8) k2_launch_t<4, CPT, RS>(p, grid, s);
      break;
  }
}

void launch_k2(const K2Params& p, int grid, int tb, cudaStream_t s) {
  const int cpt = k2_cpt(p.d);
  const int rs = k2_rows_per_tile(p.d);
  if (cpt == 2) k2_dispatch_tb<2, 2>(p, grid, tb, s);
  else if (rs == 4) k2_dispatch_tb<1, 4>(p, grid, tb, s);
  else if (rs == 8) k2_dispatch_tb<1, 8>(p, grid, tb, s);
  else k2_dispatch_tb<1, 16>(p, grid, tb, s);
}

template <int TB, int CPT, int RS>
static cudaError_t k2_attr() {
  return cudaFuncSetAttribute(k2_split_expert<TB, CPT, RS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              220 * 1024);
}

// ============================================================== K3 combine
// CTA (x, b): 32 float4 columns of token b; warp w sums chunks w, w+8, ... of every segment
// serving b (lane = column), then the 8 warp partials are added in warp order.  Fixed order
// everywhere -> deterministic.
__global__ void __launch_bounds__(256) k3_combine(const __grid_constant__ CombineParams p) {
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

void launch_combine(const CombineParams& p, cudaStream_t s) {
  dim3 grid((unsigned)((p.d / 4 + 31) / 32), (unsigned)p.B);
  k3_combine<<<grid, 256, 0, s>>>(p);
}

bool kernels_init(char* err, size_t errlen) {
  cudaError_t e = cudaSuccess;
  cudaError_t r;
#define MOEPIC_ATTR(TB, CPT, RS) \
  if ((r = k2_attr<TB, CPT, RS>()) != cudaSuccess) e = r;
  MOEPIC_ATTR(1, 2, 2) MOEPIC_ATTR(2, 2, 2) MOEPIC_ATTR(4, 2, 2)
  MOEPIC_ATTR(1, 1, 4) MOEPIC_ATTR(2, 1, 4) MOEPIC_ATTR(4, 1, 4)
  MOEPIC_ATTR(1, 1, 8) MOEPIC_ATTR(2, 1, 8) MOEPIC_ATTR(4, 1, 8)
  MOEPIC_ATTR(1, 1, 16) MOEPIC_ATTR(2, 1, 16)
#undef MOEPIC_ATTR
  if (e != cudaSuccess) {
    snprintf(err, errlen, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    return false;
  }
  return true;
}

}  // namespace moepic
