// Prefill kernels ("experts ... often fully activated"): permute tokens by expert,
// tcgen05 grouped GEMMs over the split segments, combine.
//
// GEMM kernels are persistent and warp-specialised, one CTA (or cta_group::2 CTA pair) per SM,
// 320 threads:
//   warp 0  TMA producer: ring of 192 KB of stages (A 128x64 bf16 + B), 128-byte swizzle,
//           cp.async.bulk.tensor completing on `full`, waits `empty` before reuse;
//   warp 1  allocates 512 TMEM columns (two 256-column fp32 accumulators); one lane issues
//           tcgen05.mma (M = 128 or 256 for a pair, N = 256, K = 16) and tcgen05.commit's each
//           stage back to `empty`, each finished tile to `tfull`;
//   warps 2-9 epilogue: tcgen05.ld 32 lanes x 16 columns, SwiGLU (gate/up) or fp32 store (down),
//           then arrive on `tempty` so the MMA warp can reuse that accumulator.
// gate/up: [D_g | D_u] = X_e [W_g; W_u]^T as one N = 256 MMA per K step;
//          a = silu(D_g) * D_u -> fp16 A_act[rows][I] at the segment's intermediate columns.
// down:    Y[rows][n0..n0+256) (+)= A_act[rows][seg] * Down[seg][n0..], the down rows are
//          N-contiguous in the row-interleaved layout, so B is an MN-major operand; both are fp16
//          (the stored down columns are fp16, reading Q31), one MMA per K step.
// Weights are read through a 3-D tensor map {d, 3, rows} over the row-interleaved layout
// [gate_r | up_r | down[:, r]] so the same rows serve both GEMMs without any repacking.
#include "prefill.hpp"
#include "kernels.hpp"
#include "device_utils.cuh"
#include "tc_dev.cuh"

#include <algorithm>
#include <cstdio>
#include <cstring>

namespace moepic {

namespace {

constexpr int kEpiWarps = 8;                   // 2 per TMEM lane quarter, each half the columns
constexpr int kThreads = 64 + 32 * kEpiWarps;  // producer warp, MMA warp, epilogue warps
constexpr uint32_t kAccCols = 256;             // one fp32 accumulator tile (N = 256)
constexpr uint32_t kTmemCols = 2 * kAccCols;   // double-buffered: epilogue of tile j || MMA of j+1
constexpr uint32_t kABytes = kPfBM * kPfBK * 2;        // 16 KB
// CG = 1 (one CTA, UMMA M = 128):  gate/up stage A | B_gate | B_up (48 KB) x 4,
//                                   down stage A | B[256 cols] (48 KB) x 4.
// CG = 2 (CTA pair, cta_group::2, UMMA M = 256, each CTA holds half of A and half of B):
//                                   gate/up A | B_gate or B_up (32 KB) x 6,
//                                   down A | B[128 cols] (32 KB) x 6.
template <bool DOWN, int CG> struct Cfg {
  static constexpr uint32_t kBBytes = 32 * 1024 / CG;
  static constexpr uint32_t kBOff = kABytes;
  static constexpr uint32_t kStageBytes = kBOff + kBBytes;
  static constexpr int kStages = (int)((192 * 1024) / kStageBytes);
};

__device__ __forceinline__ uint32_t bf16_rne(float a) {   // round-to-nearest-even to bf16 bits
  const uint32_t u = __float_as_uint(a);
  return (u + 0x7FFFu + ((u >> 16) & 1u)) >> 16;
}
// Tile t of a launch -> (segment, expert, m tile, n tile); both CTAs of a pair decode the same
// tile.  M tiles fastest: the CTAs sharing one weight tile run side by side, so the weights
// cross HBM once and the (L2-resident) token tiles are the ones re-read.
template <bool DOWN, int CG>
__device__ __forceinline__ bool decode_tile(const PfGemmParams& p, int t, int& seg, int& ex, int& mt, int& nt) {
  if (!DOWN) {
    for (int s = 0; s < p.nseg; ++s) {
      const int ntn = (p.seg[s].nrows + kPfBN1 - 1) / kPfBN1;
      const int mtn = (p.ex[p.seg[s].e].mtiles + CG - 1) / CG;
      const int n = mtn * ntn;
      if (t < n) { seg = s; ex = p.seg[s].e; nt = t / mtn; mt = t - nt * mtn; return true; }
      t -= n;
    }
  } else {
    const int ntn = p.d / kPfBN2;
    for (int e = 0; e < p.nexp; ++e) {
      const int mtn = (p.ex[e].mtiles + CG - 1) / CG;
      const int n = mtn * ntn;
      if (t < n) { seg = -1; ex = e; nt = t / mtn; mt = t - nt * mtn; return true; }
      t -= n;
    }
  }
  return false;
}

__device__ __forceinline__ uint32_t map_to_leader(uint32_t saddr) {   // same offset in CTA 0 of the pair
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(saddr));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

// Persistent: CTA (pair) c processes tiles c, c + G, c + 2G, ... (G = grid / CG).  The smem
// ring runs continuously across tiles; the accumulator alternates between two 256-column TMEM
// buffers so the epilogue of tile j overlaps the main loop of tile j + 1.
template <bool DOWN, int CG>
__global__ void __launch_bounds__(kThreads, 1) pf_gemm(const __grid_constant__ PfGemmParams p) {
  constexpr int kStages = Cfg<DOWN, CG>::kStages;
  constexpr uint32_t kStageBytes = Cfg<DOWN, CG>::kStageBytes;
  constexpr uint32_t kBOff = Cfg<DOWN, CG>::kBOff;
  constexpr int kTM = kPfBM * CG;               // output rows per tile (per CTA pair)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;            // [2] accumulator ready (MMA -> epilogue)
  uint64_t* tempty = tfull + 2;                 // [2] accumulator drained (epilogue -> MMA)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = CG == 2 ? (int)cluster_ctarank() : 0;   // 0 = the pair's MMA leader
  const int G = (int)gridDim.x / CG;
  const int c0 = (int)blockIdx.x / CG;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], kEpiWarps * CG);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if constexpr (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                   ::"r"(smem_u32(tmem_slot)), "r"(kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                   ::"r"(smem_u32(tmem_slot)), "r"(kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync_all();    // peer barriers initialised before any TMA
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  auto nkb_of = [&](int ex) {
    if (!DOWN) return p.d / kPfBK;
    const PfExpert& E = p.ex[ex];
    int n = 0;
    for (int s = E.seg_begin; s < E.seg_end; ++s) n += p.seg[s].nrows / kPfBK;
    return n;
  };

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      int it = 0;                                // k blocks issued so far (ring position)
      for (int t = c0; t < p.ntiles; t += G) {
        int seg, ex, mt, nt;
        decode_tile<DOWN, CG>(p, t, seg, ex, mt, nt);
        const PfExpert& E = p.ex[ex];
        const int arow = E.m_off + mt * kTM + rank * kPfBM;
        const int nkb = nkb_of(ex);
        int s = DOWN ? E.seg_begin : seg, kin = 0;   // down: current segment and k block inside it
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int st = it % kStages;
          if (it >= kStages) mbar_wait(&empty[st], ((it / kStages) - 1) & 1);
          uint8_t* sa = smem + st * kStageBytes;
          uint8_t* sb = sa + kBOff;
          const uint32_t fb = smem_u32(&full[st]);
          if (rank == 0) mbar_expect_tx(&full[st], CG * kStageBytes);
          if (!DOWN) {
            tma2d<CG>(sa, &p.tmA, kb * kPfBK, arow, fb);
            if constexpr (CG == 1) {
              tma3d<CG>(sb, &p.tmB[seg], kb * kPfBK, 0, nt * kPfBN1, fb);
              tma3d<CG>(sb + 16384, &p.tmB[seg], kb * kPfBK, 1, nt * kPfBN1, fb);
            } else {
              // the pair's B operand is [W_g; W_u] split by N: the leader holds the gate rows,
              // the peer the up rows
              tma3d<CG>(sb, &p.tmB[seg], kb * kPfBK, rank, nt * kPfBN1, fb);
            }
          } else {
            while (kin >= p.seg[s].nrows / kPfBK) { ++s; kin = 0; }
            tma2d<CG>(sa, &p.tmA, p.seg[s].row0 + kin * kPfBK, arow, fb);
            // B (MN-major down columns): this CTA's 256 / CG output columns
#pragma unroll
            for (int j = 0; j < 4 / CG; ++j)
              tma3d<CG>(sb + j * 8192, &p.tmB[s], nt * kPfBN2 + rank * (kPfBN2 / CG) + j * 64, 2, kin * kPfBK, fb);
            ++kin;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (pair leader)
    if (lane == 0 && rank == 0) {
      // gate/up: B_gate and B_up are adjacent 128-row K-major blocks, i.e. one 256-row operand
      // (CG = 1) or one 128-row half per CTA (CG = 2), so one N = 256 MMA computes [D_g | D_u]
      // down: fp16 a x fp16 down columns (reading Q31); gate/up: bf16 x bf16, or fp16 x fp16 for
      // dequantised Q4G64 rows (reading Q32)
      const uint32_t idesc = DOWN ? make_idesc(kTM, kPfBN2, 1, 0, 1)
                                  : (p.f16 ? make_idesc(kTM, 2 * kPfBN1, 0, 0, 1) : make_idesc(kTM, 2 * kPfBN1, 0));
      int it = 0, j = 0;
      for (int t = c0; t < p.ntiles; t += G, ++j) {
        int seg, ex, mt, nt;
        decode_tile<DOWN, CG>(p, t, seg, ex, mt, nt);
        const int nkb = nkb_of(ex);
        const int acc_buf = j & 1;
        if (j >= 2) mbar_wait(&tempty[acc_buf], ((j >> 1) - 1) & 1);   // epilogue drained it
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)acc_buf * kAccCols;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int st = it % kStages;
          mbar_wait(&full[st], (it / kStages) & 1);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + st * kStageBytes);
          const uint32_t sb = sa + kBOff;
#pragma unroll
          for (int k = 0; k < kPfBK / 16; ++k) {
            const uint64_t da = desc_k_sw128(sa + k * 32);
            const uint32_t acc = (kb | k) ? 1u : 0u;
            if (!DOWN) {
              umma<CG>(d, da, desc_k_sw128(sb + k * 32), idesc, acc);
            } else {
              umma<CG>(d, da, desc_mn_sw128(sb + k * 2048, 8192, 1024), idesc, acc);
            }
          }
          umma_commit<CG>(&empty[st]);
        }
        umma_commit<CG>(&tfull[acc_buf]);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 2..9)
    const int ew = warp - 2;
    const int q = warp & 3;                       // TMEM lane quarter this warp may access
    const int half = ew >> 2;                     // which half of the tile's columns
    const int m = q * 32 + lane;                  // row within this CTA's 128 rows
    const uint32_t tempty_addr0 = CG == 2 ? map_to_leader(smem_u32(&tempty[0])) : smem_u32(&tempty[0]);
    int j = 0;
    for (int t = c0; t < p.ntiles; t += G, ++j) {
      int seg, ex, mt, nt;
      decode_tile<DOWN, CG>(p, t, seg, ex, mt, nt);
      const PfExpert& E = p.ex[ex];
      const int mrow = mt * kTM + rank * kPfBM;
      const int arow = E.m_off + mrow;
      const int acc_buf = j & 1;
      mbar_wait(&tfull[acc_buf], (j >> 1) & 1);
      tc_fence_after();
      const bool row_ok = mrow + m < E.count;
      const uint32_t tbase = tmem + (uint32_t)acc_buf * kAccCols + ((uint32_t)(q * 32) << 16);
      if (!DOWN) {
        const PfSeg S = p.seg[seg];
        const size_t off = (size_t)(arow + m) * p.ld_out + S.row0 + nt * kPfBN1;
        uint16_t* out = reinterpret_cast<uint16_t*>(p.out) + off;
        for (int c = half * (kPfBN1 / 2); c < (half + 1) * (kPfBN1 / 2); c += 16) {
          float g[16], u[16];
          tmem_ld16(tbase + c, g);
          tmem_ld16(tbase + kPfBN1 + c, u);
          if (row_ok && nt * kPfBN1 + c < S.nrows) {
            uint32_t ph[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float a0 = g[2 * i] / (1.f + __expf(-g[2 * i])) * u[2 * i];
              const float a1 = g[2 * i + 1] / (1.f + __expf(-g[2 * i + 1])) * u[2 * i + 1];
              ph[i] = f16_sat(a0) | (f16_sat(a1) << 16);   // fp16 a (reading Q31)
            }
            uint4* o = reinterpret_cast<uint4*>(out + c);
            o[0] = make_uint4(ph[0], ph[1], ph[2], ph[3]);
            o[1] = make_uint4(ph[4], ph[5], ph[6], ph[7]);
          }
        }
      } else {
        float* out = reinterpret_cast<float*>(p.out) + (size_t)(arow + m) * p.ld_out + nt * kPfBN2;
        for (int c = half * (kPfBN2 / 2); c < (half + 1) * (kPfBN2 / 2); c += 16) {
          float v[16];
          tmem_ld16(tbase + c, v);
          if (row_ok) {
            float4* o = reinterpret_cast<float4*>(out + c);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              float4 x = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
              if (p.accumulate) {
                const float4 y = o[i];
                x.x += y.x; x.y += y.y; x.z += y.z; x.w += y.w;
              }
              o[i] = x;
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_addr0 + (uint32_t)acc_buf * 8);   // the leader's barrier
    }
  }
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync_all();    // both CTAs done before the pair frees TMEM
  else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if constexpr (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
  }
}

// ------------------------------------------------------------------ permute / combine
__global__ void pf_permute(const __grid_constant__ PfPermuteParams p) {
  // one warp per (t, k): claim a row of the expert's block, copy h[t] there
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int TK = p.T * p.K;
  const int total = TK + p.n_shared * p.T;
  if (gw >= total) return;
  int row, t;
  if (gw < TK) {
    t = gw / p.K;
    const int e = p.ids[gw];
    if (e < p.e_lo || e >= p.e_hi) {
      if (lane == 0) p.pos[gw] = -1;
      return;
    }
    int r = 0;
    if (lane == 0) r = atomicAdd(&p.cursor[e], 1);
    r = __shfl_sync(0xffffffffu, r, 0);
    row = p.m_off[e] + r;
    if (lane == 0) p.pos[gw] = row;
  } else {
    const int s = (gw - TK) / p.T;
    t = (gw - TK) - s * p.T;
    row = p.shared_off[s] + t;
  }
  const uint4* src = reinterpret_cast<const uint4*>(p.h + (size_t)t * p.d);
  uint4* dst = reinterpret_cast<uint4*>(p.xperm + (size_t)row * p.d);
  if (!p.f16) {
    for (int c = lane; c < p.d / 8; c += 32) dst[c] = src[c];
  } else {   // bf16 -> fp16: exact for |h| in [2^-14, 65504] (saturated beyond)
    for (int c = lane; c < p.d / 8; c += 32) {
      const uint4 v = src[c];
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
      uint32_t o[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) o[i] = f16_sat(bf16lo(w[i])) | (f16_sat(bf16hi(w[i])) << 16);
      dst[c] = make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
}

// Q4G64 rows -> fp16 rows (reading Q32): one warp per row; lane j takes code words j, j + 32, ...
// (8 codes of one 64-column group each: x' = lo_b + code * s_b in fp32, rounded once to fp16)
__global__ void pf_dequant(const __grid_constant__ PfDequantParams p) {
  const int gw = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (gw >= p.total_rows) return;
  int s = 0;
  while (s + 1 < p.nseg && p.seg[s + 1].row_begin <= gw) ++s;
  const int r = gw - p.seg[s].row_begin;
  const uint8_t* row = p.seg[s].src + (size_t)r * p.src_row_bytes;
  uint4* out = reinterpret_cast<uint4*>(p.seg[s].dst + (size_t)r * 3 * p.d);
  const int d = p.d, words = 3 * d / 8, wpp = d / 8;   // code words per row / per part
  const uint32_t* codes = reinterpret_cast<const uint32_t*>(row);
  const uint32_t* prm = reinterpret_cast<const uint32_t*>(row + 3 * (d / 2));
  for (int w = lane; w < words; w += 32) {
    const int part = w / wpp, col = (w - part * wpp) * 8;
    const uint32_t pr = __ldg(prm + part * (d >> 6) + (col >> 6));
    const float sc = __uint_as_float(pr << 16), mn = __uint_as_float(pr & 0xFFFF0000u);
    const uint32_t c = __ldg(codes + w);
    uint32_t o[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float q0 = __uint_as_float(0x4B000000u | ((c >> (8 * i)) & 15u)) - 8388608.0f;
      const float q1 = __uint_as_float(0x4B000000u | ((c >> (8 * i + 4)) & 15u)) - 8388608.0f;
      o[i] = f16_sat(fmaf(q0, sc, mn)) | (f16_sat(fmaf(q1, sc, mn)) << 16);
    }
    out[w] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

__global__ void pf_combine(const __grid_constant__ PfCombineParams p) {
  const int t = blockIdx.y;
  const int c4 = blockIdx.x * blockDim.x + threadIdx.x;
  if (c4 * 4 >= p.d) return;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (p.residual) {
    const uint2 hv = reinterpret_cast<const uint2*>(p.h + (size_t)t * p.d)[c4];
    acc = make_float4(bf16lo(hv.x), bf16hi(hv.x), bf16lo(hv.y), bf16hi(hv.y));
  }
  for (int k = 0; k < p.K; ++k) {
    const int r = p.pos[t * p.K + k];
    if (r < 0) continue;
    const float w = p.w[t * p.K + k];
    const float4 v = reinterpret_cast<const float4*>(p.Y + (size_t)r * p.d)[c4];
    acc.x = fmaf(w, v.x, acc.x); acc.y = fmaf(w, v.y, acc.y);
    acc.z = fmaf(w, v.z, acc.z); acc.w = fmaf(w, v.w, acc.w);
  }
  for (int s = 0; s < p.n_shared; ++s) {
    const int r = p.shared_off[s] + t;
    const float4 v = reinterpret_cast<const float4*>(p.Y + (size_t)r * p.d)[c4];
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
  }
  reinterpret_cast<float4*>(p.y + (size_t)t * p.d)[c4] = acc;
}

// ------------------------------------------------------------------ tensor maps
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn g_encode = nullptr;

bool get_encode() {
  if (g_encode) return true;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !fn)
    return false;
  g_encode = reinterpret_cast<EncodeTiledFn>(fn);
  return true;
}

}  // namespace

size_t pf_gemm_smem_bytes() { return 192 * 1024 + 1024 + 512; }   // stages (192 KB) + align + barriers

bool pf_tmap_2d(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  if (!get_encode()) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t es[2] = {1, 1};
  return g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool pf_tmap_weights(CUtensorMap* m, const void* seg_base, uint64_t rows, int d, uint32_t box_rows) {
  if (!get_encode()) return false;
  cuuint64_t dims[3] = {(cuuint64_t)d, 3, rows};
  cuuint64_t strides[2] = {(cuuint64_t)d * 2, (cuuint64_t)d * 6};
  cuuint32_t box[3] = {64, 1, box_rows};
  cuuint32_t es[3] = {1, 1, 1};
  return g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(seg_base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <bool DOWN, int CG>
static void launch_gemm(const PfGemmParams& p, cudaStream_t s) {
  cudaLaunchConfig_t cfg{};
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int ctas = std::min(p.ntiles, sms / CG) * CG;   // persistent: one CTA (pair) per SM (pair)
  cfg.gridDim = dim3((unsigned)ctas);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = pf_gemm_smem_bytes();
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, pf_gemm<DOWN, CG>, p);
}
void launch_pf_gateup(const PfGemmParams& p, cudaStream_t s) {
  if (p.ntiles <= 0) return;
  if (p.cta_pair) launch_gemm<false, 2>(p, s);
  else launch_gemm<false, 1>(p, s);
}
void launch_pf_down(const PfGemmParams& p, cudaStream_t s) {
  if (p.ntiles <= 0) return;
  if (p.cta_pair) launch_gemm<true, 2>(p, s);
  else launch_gemm<true, 1>(p, s);
}
void launch_pf_permute(const PfPermuteParams& p, cudaStream_t s) {
  const int warps = p.T * p.K + p.n_shared * p.T;
  pf_permute<<<(warps + 7) / 8, 256, 0, s>>>(p);
}
void launch_pf_dequant(const PfDequantParams& p, cudaStream_t s) {
  if (p.total_rows <= 0) return;
  pf_dequant<<<(p.total_rows + 7) / 8, 256, 0, s>>>(p);
}
void launch_pf_combine(const PfCombineParams& p, cudaStream_t s) {
  dim3 grid((unsigned)((p.d / 4 + 127) / 128), (unsigned)p.T);
  pf_combine<<<grid, 128, 0, s>>>(p);
}

bool prefill_init(char* err, size_t errlen) {
  const int sm = (int)pf_gemm_smem_bytes();
  const cudaError_t e[4] = {
      cudaFuncSetAttribute(pf_gemm<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm),
      cudaFuncSetAttribute(pf_gemm<true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm),
      cudaFuncSetAttribute(pf_gemm<false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm),
      cudaFuncSetAttribute(pf_gemm<true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm)};
  for (cudaError_t x : e)
    if (x != cudaSuccess) {
      snprintf(err, errlen, "prefill attributes: %s", cudaGetErrorString(x));
      return false;
    }
  return true;
}

}  // namespace moepic
