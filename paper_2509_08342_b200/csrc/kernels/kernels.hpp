// Internal launch interface of the MoEpic sm_100a kernels (not part of the C ABI).
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#ifdef __CUDACC__
#define MOEPIC_HD __host__ __device__
#else
#define MOEPIC_HD
#endif

namespace moepic {

constexpr int kMaxN = 512;          // routed experts per layer supported by K1
constexpr int kK2Threads = 256;
constexpr int kK2Stages = 4;
constexpr int kMaxLaunchSegs = 256; // segments per K2 launch (kernel-parameter array)
constexpr int kMaxStepSegs = 1024;  // segments per combine launch

// ------------------------------------------------------------------ K1: router + predictor
struct RouterParams {
  const uint16_t* h;      // [B][d] bf16
  const uint16_t* W0;     // R^i [N][d] (routing) or nullptr
  const uint16_t* W1;     // R^j [N][d] (prediction) or nullptr
  double* logits;         // [2][B][N] scratch
  int32_t* ids;           // [B][K] out
  float* w;               // [B][K] out
  int32_t* ranking;       // [N] out
  unsigned int* ticket;   // zero-initialised, reset by the kernel
  // mapped pinned mailbox (device aliases)
  // mapped-pinned mailbox of self-validating 64-bit words: (seq << 32) | payload32.  The host
  // accepts a word once its tag equals seq, so no system-scope fence is needed (a fence.sys
  // waits behind the saturated host->device link).  Layout: ids [B*K], w bits [B*K], rank [N].
  unsigned long long* mb_ids;
  unsigned long long* mb_w;
  unsigned long long* mb_rank;
  uint32_t seq;
  int B, d, N, K, renorm;
  // batches above kRouterSplitB: phase 1 only in k1_router, selection in k1_select (one warp per
  // token, per-expert prediction count / max logit reduced with atomics into sel_cnt / sel_max)
  unsigned int* ticket2;            // zero-initialised, reset by k1_select
  int32_t* sel_cnt;                 // [N] zero-initialised, reset by k1_select
  unsigned long long* sel_max;      // [N] order-preserving max-logit keys, reset to 0
  unsigned long long* tstamp;       // profiling record (device_utils.cuh) or nullptr
  unsigned long long* dbg;          // MOEPIC_K1_TRACE phase stamps [8] (tools) or nullptr
};
constexpr int kRouterSplitB = 32;
constexpr int kProfRing = 4096;   // profiling records (events + in-kernel timestamps) per drain
// pdl: programmatic dependent launch after the previous kernel on s (its weight loads overlap
// that kernel's tail; h is read after griddepcontrol.wait)
void launch_router(const RouterParams& p, cudaStream_t s, bool pdl = false);
cudaError_t router_init();     // shared-memory carveout hints (called by kernels_init)
cudaError_t combine_init();

// ------------------------------------------------------------------ K2: split-expert stream
struct Seg {
  const uint8_t* base;    // first row of the segment (row-interleaved layout, 6d bytes/row)
  int32_t expert;         // routed expert id, or -1 - s for shared expert s (weight 1)
  int32_t nrows;
  uint32_t tok_mask;      // tokens (bits) this segment serves; popcount <= kMaxTB
  int32_t row_begin;      // prefix of rows in this launch
  int64_t ws_off;         // float offset of the segment's partial area in the workspace
  int32_t cta_first;      // first CTA whose row range overlaps this segment
  int32_t pad;
};

struct CombineSeg {
  int64_t ws_off;
  int32_t nchunks;
  uint32_t tok_mask;
};

struct K2Params {
  const uint16_t* h;      // [B][d]
  const int32_t* ids;     // [B][K]
  const float* w;         // [B][K]
  float* ws;              // partial sums
  int64_t total_rows;
  // gated rows: launch rows [rows_a, total_rows) are the tail of the step's last on-demand copy,
  // still in flight at launch; CTAs stream them after *gate reaches gate_val (written by the copy
  // stream after that copy).  rows [0, rows_a) over the first ga CTAs, the rest over the first gb.
  // Ungated: rows_a = total_rows, ga = grid, gb = 0, gate = nullptr.
  int64_t rows_a;
  int ga, gb;
  const unsigned int* gate;
  unsigned int gate_val;
  unsigned int* stall;    // gated: per-CTA ns spent waiting for the flag (mapped host memory) or nullptr
  int d, K, nsegs;
  int q4;                 // rows are Q4G64 (dequantised on the fly) instead of bf16
  Seg segs[kMaxLaunchSegs];
  // fused combine (the step's final K2 launch, cooperative): after a grid barrier every CTA adds
  // a slice of the step's partials in K3's fixed order
  int combine, B, residual, ncomb;
  int flat;                         // the combine lists per-token partial offsets in shared memory
  float* y;
  unsigned long long* bar;
  unsigned long long bar_target;
  unsigned long long* tstamp;       // profiling record or nullptr
  unsigned long long* dbg;          // per-CTA phase trace [G][8] (MOEPIC_K2_TRACE) or nullptr
  CombineSeg comb[kMaxLaunchSegs];
};
// Partition rule shared with the host: CTA c of G owns launch rows [c*R/G, (c+1)*R/G).
MOEPIC_HD inline int64_t k2_row_lo(int64_t c, int64_t R, int64_t G) { return c * R / G; }
int k2_rows_per_tile(int d, int q4);
int k2_max_tokens(int d, int q4);
size_t k2_smem_bytes(int d, int q4);
void launch_k2(const K2Params& p, int grid, int tb, cudaStream_t s);

// ------------------------------------------------------------------ K2T: tcgen05 decode (B_e > 4)
// Segments of 64-row units read through one tensor map over the arena's row region; the launch
// writes one partial [G][B][d] (combined by K3 like any (segment, CTA) partial with tok_mask
// (1 << B) - 1 and nchunks = G).  Needs bf16 rows, d % 256 == 0, d <= 2048, B <= 16.
struct K2TSeg {
  int64_t map_row;        // tensor-map row of the segment's first row
  int32_t unit_begin;     // first 64-row unit of the segment in this launch
  int32_t expert;         // routed expert id, or -1 - s for shared expert s (weight 1)
  uint32_t tok_mask;      // tokens this segment serves
  int32_t pad;
};
struct K2TParams {
  const CUtensorMap* tmW;
  CUtensorMap tmH;
  const int32_t* ids;
  const float* w;
  float* ws;              // this launch's partial area [G][B][d]
  int d, K, B, nsegs, units;
  int mode;               // MOEPIC_K2T_MODE diagnostics: 1 = no MMAs (operand streaming only)
  unsigned long long* tstamp;
  unsigned long long* dbg;          // MOEPIC_K2_TRACE per-CTA stamps [G][8] (tools) or nullptr
  K2TSeg segs[kMaxLaunchSegs];
};
constexpr int kK2TMaxB = 16;
constexpr int kK2TMaxD = 2048;
void launch_k2t(const K2TParams& p, int grid, cudaStream_t s);
size_t k2t_smem_bytes(int d);
cudaError_t k2t_init();

// ------------------------------------------------------------------ K3: combine
struct CombineParams {
  float* y;               // [B][d] fp32 out
  const uint16_t* h;      // residual source
  const float* ws;
  int B, d, residual, nsegs;
  unsigned long long* tstamp;       // profiling record or nullptr
  CombineSeg segs[kMaxStepSegs];
};
void launch_combine(const CombineParams& p, cudaStream_t s);

// Host-buffer entry (moepic_layer_forward_host): copy the step's input rows from mapped pinned
// host memory into device memory with SM loads, so the few KB do not queue behind the transfer
// engine's multi-MB chunks on the host->device copy engine.  bytes % 16 == 0.
void launch_stage_in(void* dst, const void* src_mapped, size_t bytes, cudaStream_t s);
// MOEPIC_FAULT_AT_STEP (tests): a one-thread kernel that executes a trap instruction
void launch_trap(cudaStream_t s);
// MOEPIC_TIMELINE (tools): one thread writes %globaltimer to *p when the stream reaches it
void launch_stamp(unsigned long long* p, cudaStream_t s);
void launch_clock_sync(unsigned long long* mapped, cudaStream_t s);

// Attention stand-in (attention.cu): GQA decode over a KV cache [B][S_max][Hkv][dh], dh = 128.
constexpr int kAttnChunk = 128;   // cache positions per split: one CTA (4 warps x 32) per split and kv head
struct AttnParams {
  const uint16_t* q;      // [B][Hq][dh] bf16
  const uint16_t* k;      // [B][S_max][Hkv][dh] bf16
  const uint16_t* v;
  float* out;             // [B][Hq][dh] fp32
  float* ws;              // [B][Hq][splits][dh + 2] partials
  int B, S, S_max, Hq, Hkv, splits;
};
int attn_splits(int S);
bool launch_attention(const AttnParams& p, cudaStream_t s);   // false: unsupported group size
cudaError_t attention_init();

bool kernels_init(char* err, size_t errlen);  // sets smem attributes; returns false on failure

}  // namespace moepic
