// Probe (tools only): HBM streaming rate of the access patterns a tensor-core decode kernel can
// use on the row-interleaved expert layout (rows of [gate | up | down] = 6d bytes).  One
// persistent CTA per SM, a shared-memory ring filled by one producer thread and released by one
// consumer thread as soon as it lands (no math): the rate is the access pattern's alone.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/_tma_probe scripts/tma_pattern_probe.cu
//   ./scripts/_tma_probe
// Patterns (d = 2048, 12 KB rows):
//   bulk   1-D cp.async.bulk of whole rows (K2's pattern)
//   box64  3-D map {d, 3, rows}, box {64, 1, 64}: 128 B per row per request (K2T gate/up tiles)
//   box128 box {64, 1, 128};  box256 box {64, 1, 256}
//   c4     4-D map {64, rows, d/64, 3}, box {64, 64, 4, 1}: four 64-column chunks of 64 rows in one
//          request, smem [chunk][row][64] = four canonical K-major tiles
//   c4row  4-D map {64, d/64, rows, 3}, box {64, 4, 64, 1}: 512 contiguous bytes per row (smem
//          [row][chunk][64], not an MMA layout: the DRAM side of row-contiguous requests)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstring>

#define CKR(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mb_tx(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(su32(dst)), "l"(src), "r"(n), "r"(su32(b)) : "memory");
}
__device__ __forceinline__ void t3(void* dst, const CUtensorMap* m, int a, int b_, int c, uint64_t* bar) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
               ::"r"(su32(dst)), "l"(m), "r"(su32(bar)), "r"(a), "r"(b_), "r"(c) : "memory");
}
__device__ __forceinline__ void t4(void* dst, const CUtensorMap* m, int a, int b_, int c, int e, uint64_t* bar) {
  asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
               ::"r"(su32(dst)), "l"(m), "r"(su32(bar)), "r"(a), "r"(b_), "r"(c), "r"(e) : "memory");
}

struct Args {
  CUtensorMap m3_64, m3_128, m3_256, m4, m4r, mh;
  const uint8_t* base;
  int rows, d, pattern, stages, flags;   // flags: 1 = release by tcgen05.commit, 2 = + 2 KB h tile from L2
};

constexpr uint32_t kStage = 32768;

__global__ void __launch_bounds__(64, 1) probe(const __grid_constant__ Args a) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  const int S = a.stages;
  uint64_t* full = (uint64_t*)(sm + S * kStage);
  uint64_t* empty = full + S;
  // (flags & 2: the h tile lands at sm + S * kStage + 1024, shared by every stage: the probe only times it)
  const int G = gridDim.x, c = blockIdx.x;
  // 256-row blocks, contiguous per CTA
  const int nblk = a.rows / 256;
  const int b0 = c * nblk / G, b1 = (c + 1) * nblk / G;
  const int rb = 6 * a.d;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) { mb_init(&full[i], 1); mb_init(&empty[i], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // the work list: per 256-row block, gate + up of every 64-column chunk (the K2T gate/up phase)
  // as 32 KB stages; bulk streams the block's whole rows (12 KB each) in 32 KB-ish stages
  int total = 0;
  if (a.pattern == 0) total = (b1 - b0) * 256 * rb / (2 * rb);          // 2 rows per stage
  else total = (b1 - b0) * (a.d / 32);
  if (threadIdx.x == 0) {
    for (int it = 0; it < total; ++it) {
      const int st = it % S;
      if (it >= S) mb_wait(&empty[st], ((it / S) - 1) & 1);
      uint8_t* dst = sm + st * kStage;
      if (a.pattern == 0) {
        const int64_t row = (int64_t)b0 * 256 + 2 * it;
        mb_tx(&full[st], 2 * rb);
        bulk(dst, a.base + row * rb, 2 * rb, &full[st]);
      } else {
        const int per_blk = a.d / 32;          // 256 rows x 2 parts x 2d bytes / 32 KB
        const int blk = b0 + it / per_blk, r = it % per_blk;
        mb_tx(&full[st], kStage + ((a.flags & 2) ? 2048 : 0));
        if (a.flags & 2) {
          asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                       ::"r"(su32(sm + S * kStage + 1024)), "l"(&a.mh), "r"(su32(&full[st])), "r"((it % 32) * 64), "r"(0) : "memory");
        }
        if (a.pattern == 1 || a.pattern == 2) {   // stage: 128 rows x chunks (kp, kp+1) of one part
          const int nkp = a.d / 128;
          const int kp = r % nkp, half = (r / nkp) & 1, part = r / (2 * nkp);
          const int row = blk * 256 + half * 128;
          if (a.pattern == 1) {
            t3(dst, &a.m3_64, 2 * kp * 64, part, row, &full[st]);
            t3(dst + 8192, &a.m3_64, 2 * kp * 64, part, row + 64, &full[st]);
            t3(dst + 16384, &a.m3_64, (2 * kp + 1) * 64, part, row, &full[st]);
            t3(dst + 24576, &a.m3_64, (2 * kp + 1) * 64, part, row + 64, &full[st]);
          } else {
            t3(dst, &a.m3_128, 2 * kp * 64, part, row, &full[st]);
            t3(dst + 16384, &a.m3_128, (2 * kp + 1) * 64, part, row, &full[st]);
          }
        } else if (a.pattern == 3) {              // stage: 256 rows x one chunk
          const int nk = a.d / 64;
          const int kc = r % nk, part = r / nk;
          t3(dst, &a.m3_256, kc * 64, part, blk * 256, &full[st]);
        } else {                                  // stage: 64 rows x 4 chunks
          const int nq = a.d / 256;
          const int cq = r % nq, quarter = (r / nq) & 3, part = r / (4 * nq);
          if (a.pattern == 4) t4(dst, &a.m4, 0, blk * 256 + quarter * 64, cq * 4, part, &full[st]);
          else t4(dst, &a.m4r, 0, cq * 4, blk * 256 + quarter * 64, part, &full[st]);
        }
      }
    }
  } else if (threadIdx.x == 32) {
    for (int it = 0; it < total; ++it) {
      const int st = it % S;
      mb_wait(&full[st], (it / S) & 1);
      if (a.flags & 1)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&empty[st])) : "memory");
      else
        mb_arrive(&empty[st]);
    }
  }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int d = 2048, rows = 60 * 1024;
  const size_t rb = 6 * d, bytes = (size_t)rows * rb;
  uint8_t* base;
  CKR(cudaMalloc(&base, bytes));
  CKR(cudaMemset(base, 1, bytes));
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CKR(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  EncFn enc = (EncFn)fn;
  Args a{};
  a.base = base; a.rows = rows; a.d = d;
  for (int which = 0; which < 3; ++which) {
    cuuint64_t dims[3] = {(cuuint64_t)d, 3, (cuuint64_t)rows};
    cuuint64_t str[2] = {(cuuint64_t)d * 2, (cuuint64_t)rb};
    cuuint32_t box[3] = {64, 1, (cuuint32_t)(64 << which)};
    cuuint32_t es[3] = {1, 1, 1};
    CUtensorMap* m = which == 0 ? &a.m3_64 : which == 1 ? &a.m3_128 : &a.m3_256;
    if (enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, base, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      printf("encode3 %d failed\n", which);
      return 1;
    }
  }
  {
    cuuint64_t dims[4] = {64, (cuuint64_t)rows, (cuuint64_t)d / 64, 3};
    cuuint64_t str[3] = {(cuuint64_t)rb, 128, (cuuint64_t)d * 2};
    cuuint32_t box[4] = {64, 64, 4, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(&a.m4, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, base, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode4 failed (%d): pattern c4 skipped\n", (int)r);
    cuuint64_t dims2[4] = {64, (cuuint64_t)d / 64, (cuuint64_t)rows, 3};
    cuuint64_t str2[3] = {128, (cuuint64_t)rb, (cuuint64_t)d * 2};
    cuuint32_t box2[4] = {64, 4, 64, 1};
    r = enc(&a.m4r, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, base, dims2, str2, box2, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode4r failed (%d)\n", (int)r);
  }
  {
    static uint16_t* hbuf = nullptr;
    cudaMalloc(&hbuf, 16 * d * 2);
    cuuint64_t dims[2] = {(cuuint64_t)d, 16};
    cuuint64_t str[1] = {(cuuint64_t)d * 2};
    cuuint32_t box[2] = {64, 16};
    cuuint32_t es[2] = {1, 1};
    enc(&a.mh, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, hbuf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  const char* names[] = {"bulk", "box64", "box128", "box256", "c4", "c4row"};
  for (int flags : {0, 1, 2, 3}) for (int stages : {6}) {
    a.flags = flags;
    const size_t smem = stages * kStage + 1024 + 256 + 4096;
    CKR(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    for (int pat = 0; pat < 6; ++pat) {
      if (flags && pat != 1) continue;
      a.pattern = pat;
      a.stages = stages;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0); cudaEventCreate(&e1);
      probe<<<148, 64, smem>>>(a);
      CKR(cudaDeviceSynchronize());
      float best = 1e30f;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        probe<<<148, 64, smem>>>(a);
        cudaEventRecord(e1);
        CKR(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      // bytes streamed: bulk = all rows; tiles = gate + up of all rows (2/3 of the row bytes)
      const double moved = pat == 0 ? (double)(rows / 256 * 256) * rb : (double)(rows / 256 * 256) * 4.0 * d;
      printf("{\"flags\": %d, \"pattern\": \"%s\", \"stages\": %d, \"MB\": %.1f, \"us\": %.1f, \"GBps\": %.1f}\n", flags, names[pat], stages,
             moved / 1e6, best * 1e3, moved / (best * 1e-3) / 1e9);
    }
  }
  return 0;
}
