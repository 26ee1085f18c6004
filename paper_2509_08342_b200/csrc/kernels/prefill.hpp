// Prefill path: tokens permuted by expert, tcgen05 grouped GEMMs
// (gate/up with a SwiGLU epilogue, then down), unpermute-combine.  Internal interface.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace moepic {

constexpr int kPfBM = 128;          // tokens per M tile (UMMA M = 128, cta_group::1)
constexpr int kPfBN1 = 128;         // intermediate rows per gate/up tile (gate + up: one N = 256 MMA)
constexpr int kPfBN2 = 256;         // output columns per down tile (UMMA N = 256)
constexpr int kPfBK = 64;           // K per stage = one 128-byte swizzle row of bf16
constexpr int kPfMaxSegs = 136;     // weight segments (tensor maps) per GEMM launch (params ~24 KB)
constexpr int kPfMaxExperts = 136;  // experts (incl. shared) per launch

// One weight segment: rows [row0, row0 + nrows) of expert `e` (row0 = its first intermediate
// index), read through a 3-D tensor map over the row-interleaved layout {d, 3, rows}.
struct PfSeg {
  int32_t e;        // index into the launch's expert table
  int32_t row0;     // first intermediate index of the segment (0 for a top / full expert)
  int32_t nrows;    // multiple of 64 (gate/up tiles need a multiple of 128: tail masked)
  int32_t pad;
};

struct PfExpert {
  int32_t m_off;    // first padded row of the expert's token block in the permuted buffers
  int32_t count;    // tokens routed to it
  int32_t mtiles;   // ceil(count / 128)
  int32_t seg_begin, seg_end;   // its segments in the launch's segment table (down GEMM)
  int32_t pad[3];
};

struct PfGemmParams {
  CUtensorMap tmA;                    // A operand: X_perm (gate/up, bf16) or A_act (down, fp16), 2-D
  CUtensorMap tmB[kPfMaxSegs];        // weight segments, 3-D {d, 3, rows}
  PfSeg seg[kPfMaxSegs];
  PfExpert ex[kPfMaxExperts];
  int32_t nseg, nexp;
  int32_t ntiles;                     // total output tiles of the launch (CTA pairs if cta_pair)
  int32_t cta_pair;                   // 1: cta_group::2 pairs, 256-row tiles (UMMA M = 256)
  int32_t d, I;
  void* out;                          // gate/up: fp16 A_act [rows][I]; down: fp32 Y [rows][d]
  int32_t ld_out;                     // elements per output row
  int32_t accumulate;                 // down: add into `out` (second segment group)
  int32_t f16;                        // gate/up operands fp16 (Q4G64 experts, reading Q32)
};

// Q4G64 prefill (reading Q32): the step's segments are dequantised once into fp16 rows
// [gate | up | down] (6d bytes, the bf16 row geometry) so the GEMMs read them like bf16 rows.
struct PfDequantSeg {
  const uint8_t* src;       // packed Q4G64 rows
  uint16_t* dst;            // fp16 rows
  int32_t nrows;
  int32_t row_begin;        // prefix over the launch's segments
};
struct PfDequantParams {
  int32_t nseg, d, src_row_bytes, total_rows;
  PfDequantSeg seg[kPfMaxSegs];
};
void launch_pf_dequant(const PfDequantParams& p, cudaStream_t s);

// Tensor maps (driver entry point resolved at runtime; no -lcuda).
bool pf_tmap_2d(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows);
bool pf_tmap_weights(CUtensorMap* m, const void* seg_base, uint64_t rows, int d, uint32_t box_rows);

void launch_pf_gateup(const PfGemmParams& p, cudaStream_t s);
void launch_pf_down(const PfGemmParams& p, cudaStream_t s);

// permute: X_perm[pos(t,k)] = h[t]; pos from per-expert cursors (order within an expert is free:
// every row is an independent GEMM row).  slot[t*K+k] receives pos.
struct PfPermuteParams {
  const uint16_t* h;        // [T][d]
  const int32_t* ids;       // [T][K] routed expert ids (K1 output)
  int32_t* cursor;          // [N] zeroed before the launch
  int32_t* pos;             // [T][K] out (-1 for experts another EP rank owns)
  uint16_t* xperm;          // [rows][d]
  int T, K, d;
  int e_lo, e_hi;           // local experts [e_lo, e_hi)
  int n_shared;             // shared expert s: all T tokens at rows shared_off[s] + t
  int f16;                  // write X as fp16 (Q4G64 prefill, reading Q32)
  int32_t shared_off[8];
  int32_t m_off[kPfMaxExperts];   // first padded row of each routed expert's block
};
void launch_pf_permute(const PfPermuteParams& p, cudaStream_t s);

struct PfCombineParams {
  float* y;                 // [T][d]
  const uint16_t* h;        // residual
  const float* Y;           // [rows][d]
  const int32_t* pos;       // [T][K]
  const float* w;           // [T][K]
  int T, K, d, n_shared, residual;
  int32_t shared_off[8];    // first row of each shared expert's block (all T tokens)
};
void launch_pf_combine(const PfCombineParams& p, cudaStream_t s);

bool prefill_init(char* err, size_t errlen);
size_t pf_gemm_smem_bytes();

}  // namespace moepic
