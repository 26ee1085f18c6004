// Launch interface of the multi-GPU data plane (kernels/ep.cu); see the header comment there.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace moepic {

constexpr int kEpMaxRanks = 8;
enum { kEpPhIds = 0, kEpPhDispatch = 1, kEpPhCombine = 2, kEpPhReduce = 3, kEpPhases = 4 };

// base[r] = rank r's exchange region mapped into this process (base[me] = own allocation)
struct EpPeers {
  uint8_t* base[kEpMaxRanks];
  int G, me;
};

// byte offsets inside every rank's exchange region (identical on all ranks)
struct EpOffsets {
  size_t sig;          // u64 [kEpPhases][kEpMaxRanks]: epoch published by source rank
  size_t ctr;          // u32 [kEpPhases]: CTA arrival counters of the signalling kernels
  size_t ids_all[2];   // int32 [T_max][K]: routed ids of the whole batch (rank-major)
  size_t w_all[2];     // fp32  [T_max][K]: gate weights
  size_t recv[2];      // bf16  [T_max][d]: dispatched token rows (sub-batch, global order)
  size_t comb[2];      // fp32  [ceil(T_max/G) * min(G,K)][d]: partial rows of my tokens
  size_t red[2];       // fp32  [G][B_dec_max][d]: replicated-token all-reduce slots
  size_t ysub;         // fp32  [T_max][d]: the sub-batch output (not exchanged)
  size_t sendbuf;      // bf16  [T_max][d]: NCCL transport packing buffer (not exchanged)
  size_t total;
};

struct EpIdsParams {
  EpPeers pr;
  EpOffsets of;
  const int32_t* ids;        // my tokens' routing [Bl][K] (arena)
  const float* w;
  int BlK, TK;
  int push;                  // 1: peer transport pushes + waits; 0: ids_all already gathered (NCCL)
  unsigned long long epoch;
  unsigned long long* mb_ids;   // host mailbox (mapped), tagged words
  unsigned long long* mb_w;
  uint32_t seq;
};
void launch_ep_ids(const EpIdsParams& p, cudaStream_t s);

struct EpDispatchParams {
  EpPeers pr;
  EpOffsets of;
  const uint16_t* h;         // my tokens [Bl][d] bf16
  int d, K, push;
  int n_disp;                // entries: my token d_tok[e] -> rank d_dst[e], row d_row[e]
  const int32_t* d_tok;
  const int32_t* d_dst;
  const int32_t* d_row;
  uint16_t* sendbuf;         // NCCL transport: rows packed in entry order
  int n_sub;                 // sub-batch computed here: global tokens sub[j]
  const int32_t* sub;
  int32_t* ids_out;          // [n_sub][K] routing of the sub-batch (arena ids / w)
  float* w_out;
  unsigned long long epoch;
};
void launch_ep_dispatch(const EpDispatchParams& p, int grid, cudaStream_t s);

void launch_ep_wait(const EpPeers& pr, const EpOffsets& of, int phase, unsigned long long epoch, cudaStream_t s);

struct EpCombineParams {
  EpPeers pr;
  EpOffsets of;
  const float* ysub;         // [n_sub][d]
  int d, n_sub;
  const int32_t* c_dst;      // owner rank of sub row j
  const int32_t* c_row;      // row in the owner's comb buffer
  unsigned long long epoch;
};
void launch_ep_combine(const EpCombineParams& p, int grid, cudaStream_t s);

struct EpReduceParams {
  EpPeers pr;
  EpOffsets of;
  const uint16_t* h;         // my tokens (residual source)
  float* y;                  // [Bl][d] out
  int d, Bl, residual, wait;
  const int32_t* r_off;      // [Bl + 1] CSR over r_row
  const int32_t* r_row;
  unsigned long long epoch;
};
void launch_ep_reduce(const EpReduceParams& p, int grid, cudaStream_t s);

struct EpAllreduceParams {
  EpPeers pr;
  EpOffsets of;
  float* y;                  // [n] in / out
  int n, slot_floats;
  unsigned long long epoch;
};
void launch_ep_allreduce(const EpAllreduceParams& p, int grid, cudaStream_t s);

}  // namespace moepic
