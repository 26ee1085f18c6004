// K2T: split-expert decode on the tcgen05 tensor cores for batches where an expert serves more
// tokens than K2's CUDA-core token block (B_e > 4).
//
// K2 keeps one token group's gate/up dots and down-projection partials in registers, so an expert
// with B_e > 4 tokens is streamed once per 4-token group.  K2T reads every weight row ONCE for up
// to 16 tokens: the accumulators live in TMEM.
//
// Work unit = 64 rows of a segment (the row granule; segments are multiples of 64 rows).  CTA c of
// G owns units [c U / G, (c+1) U / G) and processes them in blocks of two units (128 rows):
//   gate/up  D_g, D_u [128 rows][16 tokens] (fp32, TMEM) = W_{g,u}[128 rows][d] . h[16][d]^T:
//            UMMA M = 128 (rows), N = 16 (the whole batch, B <= 16, zero rows past B), K = d;
//            A = weight tile (K-major, TMA 128-byte swizzle), B = h tile (K-major, TMA).
//   epilogue a[r][t] = silu(g) * u * w_{t, e(r)} for t in the segment's token set, else 0
//            (Eq. 2 weight folded in), rounded to fp16 (the stored down columns are fp16,
//            reading Q31) and written to shared memory as the K-major B operand of the down MMA.
//   down     D2[mt] [128 cols][16 tokens] += Down[128 rows][cols mt]^T . a[128 rows][16]:
//            UMMA M = 128 (output columns, MN-major A straight from the row-interleaved rows),
//            N = 16, K = 128 rows, fp16 x fp16.  D2 covers all d columns (d / 128 tiles of 16
//            TMEM columns) and accumulates over EVERY block of the CTA, whatever the segment:
//            the token weight is inside a, so D2[.][t] is this CTA's share of y[t].
//   flush    D2 -> workspace partial [G][B][d] once per launch (combined in fixed order by K3).
// Warp roles (192 threads): warp 0 TMA producer, warp 1 TMEM allocator + MMA issuer (one lane),
// warps 2-5 epilogue (one TMEM lane quarter each).  h stays resident in shared memory (d / 64
// swizzled [16][64] tiles); the ring holds 32 KB stages (4 for d = 2048, up to 6), and EVERY stage
// carries 32 KB of weights: a full block's stage is one 64-column chunk of gate and up for both
// units (or one 128-column M tile of down for both units), a half block's (a CTA's odd last
// unit) is two chunks (two M tiles) of its one unit.  Under a saturated memory system a CTA's
// share of the bandwidth follows its bytes in flight, so half-size stages would make the CTAs
// with an odd unit count the stragglers (measured: 33 % longer tails).  The producer and the MMA
// warp walk the same sequence GU(0), GU(1), DN(0), GU(2), DN(1), ..., DN(last), so the down MMAs
// of block j run while the epilogue of block j+1 computes its activations.
// TMEM: D_gu 2 buffers x 32 columns | D2 (d / 128) x 16 columns  (<= 320 of 512, d <= 2048).
#include "kernels.hpp"
#include "device_utils.cuh"
#include "tc_dev.cuh"

#include <cstdio>

namespace moepic {

namespace {

constexpr int kTcThreads = 192;
constexpr int kTcMaxStages = 6;
constexpr uint32_t kTcStage = 32768;   // always 32 KB of weights (see the stage table above)
constexpr uint32_t kTcB2 = 4096;       // a (fp16): [unit A | unit B] x 16 tokens x 64 rows
constexpr uint32_t kTcSmemMax = 227 * 1024;
constexpr uint32_t kTcTmemCols = 512;
constexpr int kTcN = 16;

// Segment of unit u by a forward-only cursor: each role visits its units in increasing order, so
// the walk over the segment table (kernel parameters, constant cache) is amortised to O(1) per
// lookup -- a linear scan per lookup kept the producer away from the ring for microseconds.
template <class P>
__device__ __forceinline__ int tc_seg_at(const P& p, int u, int& cur) {
  while (cur + 1 < p.nsegs && p.segs[cur + 1].unit_begin <= u) ++cur;
  return cur;
}
template <class P>
__device__ __forceinline__ int tc_seg_first(const P& p, int u) {   // binary search: last s with begin <= u
  int lo = 0, hi = p.nsegs - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (p.segs[mid].unit_begin <= u) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// mbarrier wait that adds the cycles spent to *acc (MOEPIC_K2_TRACE diagnostics) when acc != null
__device__ __forceinline__ void tc_wait(uint64_t* bar, uint32_t parity, unsigned long long* acc) {
  if (!acc) {
    mbar_wait(bar, parity);
    return;
  }
  const unsigned long long t0 = clock64();
  mbar_wait(bar, parity);
  *acc += clock64() - t0;
}

}  // namespace

template <class P>
__global__ void __launch_bounds__(kTcThreads, 1) k2t_split_expert(const __grid_constant__ P p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = p.stages;
  uint8_t* hs = smem + (size_t)S * kTcStage;                       // h: d/64 tiles [16 tokens][64]
  uint8_t* b2 = hs + (size_t)p.d * 32;                             // [2][kTcB2]
  uint64_t* full = reinterpret_cast<uint64_t*>(b2 + 2 * kTcB2);
  uint64_t* empty = full + kTcMaxStages;
  uint64_t* gu_full = empty + kTcMaxStages;    // [2] MMA -> epilogue: D_gu[buf] ready
  uint64_t* epi_done = gu_full + 2;          // [2] epilogue -> MMA: D_gu[buf] read, a[buf] written
  uint64_t* b2_empty = epi_done + 2;         // [2] MMA -> epilogue: down MMAs of a[buf] finished
  uint64_t* d2_full = b2_empty + 2;          // MMA -> epilogue: every down MMA finished
  uint64_t* h_full = d2_full + 1;            // h resident
  float* wt = reinterpret_cast<float*>(h_full + 1);   // [2 bufs][2 units][16 tokens]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(wt + 64);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = (int)gridDim.x, c = (int)blockIdx.x;
  const int u0 = (int)((int64_t)c * p.units / G), u1 = (int)((int64_t)(c + 1) * p.units / G);
  const int nb = (u1 - u0 + 1) / 2;
  const int d = p.d;
  stamp_start(p.tstamp);
  asm volatile("griddepcontrol.launch_dependents;");
  // MOEPIC_K2_TRACE: per CTA [start, MMA issue done, flush start, end (ns)] and wait cycles
  // [producer on empty, MMA on full, MMA issuing stages (+ waits on the epilogue << 40), epilogue on gu_full]
  unsigned long long* dbg = p.dbg ? p.dbg + (size_t)c * 8 : nullptr;
  unsigned long long w_empty = 0, w_full = 0, w_epi = 0, w_gu = 0, w_issue = 0;
  if (dbg && threadIdx.x == 0) dbg[0] = gtimer();

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(h_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&gu_full[i], 1);
      mbar_init(&epi_done[i], 4);
      mbar_init(&b2_empty[i], 1);
    }
    mbar_init(d2_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(tmem_slot)), "r"(kTcTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // global row (tensor-map coordinate) of unit u; u non-decreasing per caller
  int pcur = tc_seg_first(p, u0);
  auto unit_row = [&](int u) -> int {
    const int s = tc_seg_at(p, u, pcur);
    return (int)(p.segs[s].map_row + (int64_t)(u - p.segs[s].unit_begin) * 64);
  };

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      mbar_expect_tx(h_full, (uint32_t)d * 32);
      for (int kc = 0; kc < d / 64; ++kc) tma2d<1>(hs + (size_t)kc * 2048, &p.tmH, kc * 64, 0, smem_u32(h_full));
      int it = 0;
      auto slot = [&]() -> uint8_t* {
        const int st = it % S;
        if (it >= S) tc_wait(&empty[st], ((it / S) - 1) & 1, dbg ? &w_empty : nullptr);
        mbar_expect_tx(&full[st], kTcStage);
        return smem + (size_t)st * kTcStage;
      };
      int rowsA[2] = {0, 0}, rowsB[2] = {0, 0};   // block j's unit rows, kept for dn(j)
      auto gu = [&](int j) {
        const int uA = u0 + 2 * j;
        const bool hasB = uA + 1 < u1;
        const int rA = unit_row(uA), rB = hasB ? unit_row(uA + 1) : 0;
        rowsA[j & 1] = rA;
        rowsB[j & 1] = rB;
        for (int kc = 0; kc < d / 64; kc += hasB ? 1 : 2, ++it) {
          uint8_t* sa = slot();
          const uint32_t fb = smem_u32(&full[it % S]);
          tma3d<1>(sa, &p.tmW, kc * 64, 0, rA, fb);
          tma3d<1>(sa + 16384, &p.tmW, kc * 64, 1, rA, fb);
          tma3d<1>(sa + 8192, &p.tmW, (hasB ? kc : kc + 1) * 64, 0, hasB ? rB : rA, fb);
          tma3d<1>(sa + 24576, &p.tmW, (hasB ? kc : kc + 1) * 64, 1, hasB ? rB : rA, fb);
        }
      };
      auto dn = [&](int j) {
        const bool hasB = u0 + 2 * j + 1 < u1;
        const int rA = rowsA[j & 1], rB = rowsB[j & 1];
        for (int mt = 0; mt < d / 128; mt += hasB ? 1 : 2, ++it) {
          uint8_t* sa = slot();
          const uint32_t fb = smem_u32(&full[it % S]);
          tma3d<1>(sa, &p.tmW, mt * 128, 2, rA, fb);
          tma3d<1>(sa + 8192, &p.tmW, mt * 128 + 64, 2, rA, fb);
          tma3d<1>(sa + 16384, &p.tmW, (hasB ? mt : mt + 1) * 128, 2, hasB ? rB : rA, fb);
          tma3d<1>(sa + 24576, &p.tmW, (hasB ? mt : mt + 1) * 128 + 64, 2, hasB ? rB : rA, fb);
        }
      };
      gu(0);
      for (int j = 1; j < nb; ++j) {
        gu(j);
        dn(j - 1);
      }
      dn(nb - 1);
      if (dbg) dbg[4] = w_empty;
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_gu = make_idesc(128, kTcN, 0, 0);   // A rows K-major, B h K-major
      constexpr uint32_t idesc_dn = make_idesc(128, kTcN, 0, 1, 1);   // fp16: A down columns MN-major, B = a
      int it = 0;
      mbar_wait(h_full, 0);
      const uint32_t hb = smem_u32(hs);
      auto gu = [&](int j) {
        const int buf = j & 1;
        const bool hasB = u0 + 2 * j + 1 < u1;
        if (j >= 2) tc_wait(&epi_done[buf], ((j >> 1) - 1) & 1, dbg ? &w_epi : nullptr);   // D_gu[buf] drained
        tc_fence_after();
        const uint32_t dg = tmem + (uint32_t)buf * 32, du = dg + 16;
        for (int kc = 0; kc < d / 64; kc += hasB ? 1 : 2, ++it) {
          const int st = it % S;
          tc_wait(&full[st], (it / S) & 1, dbg ? &w_full : nullptr);
          tc_fence_after();
          const unsigned long long ti = dbg ? clock64() : 0ull;
          const uint32_t sa = smem_u32(smem + (size_t)st * kTcStage);
          // full block: one k chunk, rows 0-63 unit A | 64-127 unit B.  Half block: chunks kc and
          // kc+1 of unit A at +0 / +8 KB; an M = 128 MMA then reads 64 more rows past its chunk
          // (the next tile) into TMEM lanes 64-127, which the epilogue ignores
          for (int sub = 0; sub < (hasB ? 1 : 2); ++sub) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint32_t acc = ((kc + sub) | kk) ? 1u : 0u;
              const uint64_t db = desc_k_sw128(hb + (uint32_t)(kc + sub) * 2048 + kk * 32);
              if (p.mode & 1) continue;   // diagnostics: stream the operands, no MMAs
              umma<1>(dg, desc_k_sw128(sa + sub * 8192 + kk * 32), db, idesc_gu, acc);
              umma<1>(du, desc_k_sw128(sa + 16384 + sub * 8192 + kk * 32), db, idesc_gu, acc);
            }
          }
          umma_commit<1>(&empty[st]);
          if (dbg) w_issue += clock64() - ti;
        }
        umma_commit<1>(&gu_full[buf]);
      };
      auto dn = [&](int j) {
        const int buf = j & 1;
        const bool hasB = u0 + 2 * j + 1 < u1;
        tc_wait(&epi_done[buf], (j >> 1) & 1, dbg ? &w_epi : nullptr);   // a[buf] of block j written
        tc_fence_after();
        const uint32_t ab = smem_u32(b2 + (size_t)buf * kTcB2);
        for (int mt = 0; mt < d / 128; mt += hasB ? 1 : 2, ++it) {
          const int st = it % S;
          tc_wait(&full[st], (it / S) & 1, dbg ? &w_full : nullptr);
          tc_fence_after();
          const unsigned long long ti = dbg ? clock64() : 0ull;
          const uint32_t sa = smem_u32(smem + (size_t)st * kTcStage);
          // full block: M tile mt, unit A at +0, unit B at +16 KB (K = 128 rows).  Half block:
          // M tiles mt and mt+1 of unit A at +0 / +16 KB (K = 64 rows each)
          for (int sub = 0; sub < 2; ++sub) {
            const uint32_t d2 = tmem + 64 + (uint32_t)(hasB ? mt : mt + sub) * kTcN;
            const uint32_t bu = hasB ? (uint32_t)sub * 2048 : 0u;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t da = desc_mn_sw128(sa + sub * 16384 + kk * 2048, 8192, 1024);
              const uint32_t acc = (j == 0 && (sub == 0 || !hasB) && kk == 0) ? 0u : 1u;
              if (p.mode & 1) continue;
              umma<1>(d2, da, desc_k_sw128(ab + bu + kk * 32), idesc_dn, acc);
            }
          }
          umma_commit<1>(&empty[st]);
          if (dbg) w_issue += clock64() - ti;
        }
        umma_commit<1>(&b2_empty[buf]);
      };
      gu(0);
      for (int j = 1; j < nb; ++j) {
        gu(j);
        dn(j - 1);
      }
      dn(nb - 1);
      umma_commit<1>(d2_full);
      if (dbg) {
        dbg[1] = gtimer();
        dbg[5] = w_full;
        dbg[6] = w_issue + (w_epi << 40);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 2..5)
    const int q = warp & 3;                 // TMEM lane quarter
    const int m = q * 32 + lane;            // row of the 128-row block
    const int unit = m >> 6, r64 = m & 63;
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    int ecur = tc_seg_first(p, u0);
    for (int j = 0; j < nb; ++j) {
      const int buf = j & 1;
      const int uA = u0 + 2 * j;
      const bool hasB = uA + 1 < u1;
      if (warp == 2) {   // Eq. 2 weight of (unit, token): 0 when the token does not use the segment
        const int uu = lane >> 4, t = lane & 15;
        float v = 0.f;
        if ((uu == 0 || hasB) && t < p.B) {
          const auto& sg = p.segs[tc_seg_at(p, uA + uu, ecur)];
          if ((sg.tok_mask >> t) & 1u) {
            if (sg.expert < 0) {
              v = 1.f;
            } else {
              for (int k = 0; k < p.K; ++k)
                if (p.ids[t * p.K + k] == sg.expert) v = p.w[t * p.K + k];
            }
          }
        }
        wt[buf * 32 + lane] = v;
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      tc_wait(&gu_full[buf], (j >> 1) & 1, dbg ? &w_gu : nullptr);
      if (j >= 2) mbar_wait(&b2_empty[buf], ((j >> 1) - 1) & 1);
      tc_fence_after();
      float g[16], u[16];
      tmem_ld16(lane_base + (uint32_t)buf * 32, g);
      tmem_ld16(lane_base + (uint32_t)buf * 32 + 16, u);
      const bool valid = unit == 0 || hasB;
      uint8_t* ab = b2 + (size_t)buf * kTcB2 + unit * 2048;
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const float wv = wt[buf * 32 + unit * 16 + t];
        const float a = (valid && wv != 0.f) ? g[t] / (1.f + __expf(-g[t])) * u[t] * wv : 0.f;
        // K-major 128-byte swizzle: token t = row (t & 7) of 8-row group t >> 3; 16-byte chunk
        // r64 / 8 stored at chunk (r64 / 8) ^ (t & 7)
        const uint32_t off = (uint32_t)((t >> 3) * 1024 + (t & 7) * 128 + ((((r64 >> 3) ^ (t & 7)) & 7) << 4) + (r64 & 7) * 2);
        *reinterpret_cast<uint16_t*>(ab + off) = (uint16_t)f16_sat(a);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&epi_done[buf]);
    }
    // flush this CTA's share of y: D2[mt] lane = column mt*128 + m, TMEM column t = token
    mbar_wait(d2_full, 0);
    tc_fence_after();
    if (dbg && threadIdx.x == 64) {
      dbg[2] = gtimer();
      dbg[7] = w_gu;
    }
    float* dst = p.ws + (int64_t)c * p.B * d;
    for (int mt = 0; mt < d / 128; ++mt) {
      float v[16];
      tmem_ld16(lane_base + 64 + (uint32_t)mt * kTcN, v);
      const int col = mt * 128 + m;
#pragma unroll
      for (int t = 0; t < 16; ++t)
        if (t < p.B) dst[(int64_t)t * d + col] = v[t];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTcTmemCols));
  }
  if (dbg && threadIdx.x == 0) dbg[3] = gtimer();
  stamp_end(p.tstamp);
}

template <int CAP>
struct K2TParamsCap {
  CUtensorMap tmW;   // 3-D {d, 3, rows} over the arena's row region (rows 6d bytes apart)
  CUtensorMap tmH;   // 2-D {d, B} over h, box {64, 16}: rows past B read as zeros
  const int32_t* ids;
  const float* w;
  float* ws;
  int d, K, B, nsegs, units, mode, stages;
  unsigned long long* tstamp;
  unsigned long long* dbg;
  K2TSeg segs[CAP];
};

// ring stages that fit next to the resident h (d * 32 bytes), the a buffers and the barriers
static int k2t_stages(int d) {
  const int s = (int)((kTcSmemMax - 1024 - 512 - 2 * kTcB2 - (uint32_t)d * 32) / kTcStage);
  return s < kTcMaxStages ? s : kTcMaxStages;
}
size_t k2t_smem_bytes(int d) { return (size_t)k2t_stages(d) * kTcStage + (size_t)d * 32 + 2 * kTcB2 + 1024 + 512; }

template <int CAP>
static void k2t_launch_cap(const K2TParams& p, int grid, cudaStream_t s) {
  K2TParamsCap<CAP> q;
  q.tmW = *p.tmW;
  q.tmH = p.tmH;
  q.ids = p.ids; q.w = p.w; q.ws = p.ws;
  q.d = p.d; q.K = p.K; q.B = p.B; q.nsegs = p.nsegs; q.units = p.units; q.mode = p.mode; q.stages = k2t_stages(p.d); q.tstamp = p.tstamp; q.dbg = p.dbg;
  for (int i = 0; i < p.nsegs; ++i) q.segs[i] = p.segs[i];
  k2t_split_expert<K2TParamsCap<CAP>><<<grid, kTcThreads, k2t_smem_bytes(p.d), s>>>(q);
}

void launch_k2t(const K2TParams& p, int grid, cudaStream_t s) {
  if (p.nsegs <= 32) k2t_launch_cap<32>(p, grid, s);
  else k2t_launch_cap<kMaxLaunchSegs>(p, grid, s);
}

cudaError_t k2t_init() {
  cudaError_t e = cudaSuccess, r;
  if ((r = cudaFuncSetAttribute(k2t_split_expert<K2TParamsCap<32>>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)kTcSmemMax)) != cudaSuccess) e = r;
  if ((r = cudaFuncSetAttribute(k2t_split_expert<K2TParamsCap<kMaxLaunchSegs>>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTcSmemMax)) != cudaSuccess)
    e = r;
  return e;
}

}  // namespace moepic
