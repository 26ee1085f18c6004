// C ABI of the MoEpic library (include/moepic.h, include/moepic_hostsim.h).
//
// One context = one GPU: the host control plane (host/control.hpp), the device arena layout,
// the copy stream ("transfer engine"), the mapped-pinned routing mailbox and the kernel
// launches of one MoE layer step:
//   K1 router (+ next-layer predictor) -> host waits on the mailbox -> control-plane step
//   -> on-demand H2D copies of missing segments (copy stream) -> K2 over resident tops (no
//   wait) -> K2 over prefetched segments (wait plan event) -> K2 over on-demand segments
//   (wait copy event) -> K3 combine -> next-layer prefetch plan issued on the copy stream.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>
#include <new>
#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>   // types only: the library dlopens libnccl.so.2 (the process's own copy) at join

#include "../../include/moepic.h"
#include "../../include/moepic_hostsim.h"
#include "host/control.hpp"
#include "host/ep_plan.hpp"
#include "kernels/ep.hpp"
#include "kernels/kernels.hpp"
#include "kernels/prefill.hpp"

using namespace moepic;

namespace {

constexpr int kSMs = 148;
constexpr int kStallSlot = 160;   // per-CTA gate-wait records per gated K2 launch (>= kSMs)
constexpr size_t kAlign = 256;
inline size_t align_up(size_t x, size_t a = kAlign) { return (x + a - 1) / a * a; }

struct ArenaLayout {
  size_t routers, shared, pool, buf[2], ws, logits, ids, w, ranking, ticket, rsel, trec, hstage, ystage, total;
  uint64_t pool_rows, plan_rows, od_rows, ws_floats, map_rows;
  // prefill (max_batch > kDecodeMaxB): permuted tokens, intermediate activations, outputs
  size_t xperm, aact, yperm, pos, cursor, wdq;
  uint64_t pf_rows, wdq_rows;
};
constexpr int kDecodeMaxB = 32;   // decode path (K2) serves up to 32 tokens (token bit masks)

int n_local(const moepic_model_desc& d) { return d.N / d.ep_size; }

// K2T (kernels/expert_tc.cu) serves decode steps whose experts take more tokens than K2's token
// block: bf16 rows, d a multiple of 256 up to 2048 (TMEM holds the [d][16] accumulator), 64-row
// units (row granule), batches of 5..16 tokens.  MOEPIC_K2T=0 at create keeps every step on K2.
bool k2t_eligible(const moepic_model_desc& d) {
  return d.weight_format == MOEPIC_BF16 && d.d % 256 == 0 && d.d <= kK2TMaxD &&
         d.row_granule % 64 == 0 && d.max_batch > 4;
}

std::string validate_desc(const moepic_model_desc* d) {
  if (!d) return "desc is NULL";
  if (d->L < 1) return "L must be >= 1";
  if (d->N < 2 || d->N > kMaxN) return "N must be in [2, 512]";
  if (d->K < 1 || d->K >= d->N) return "K must be < N";
  if (d->K > 64) return "K must be <= 64";
  if (d->d < 8 || d->d % 8 != 0 || d->d > 4096) return "d must be a multiple of 8 in [8, 4096]";
  if (d->row_granule < 16 || d->row_granule % 16 != 0) return "row_granule must be a positive multiple of 16";
  if (d->I < d->row_granule || d->I % d->row_granule != 0) return "I must be a multiple of row_granule";
  if (d->n_shared < 0 || d->n_shared > 8) return "n_shared must be in [0, 8]";
  if (d->buffer_experts < d->K) return "buffer_experts must be >= K";
  if (d->max_batch < 1 || d->max_batch > 4096) return "max_batch must be in [1, 4096]";
  if (d->max_batch > kDecodeMaxB && (d->d % 256 != 0 || d->N + d->n_shared > kPfMaxExperts))
    return "prefill batches (max_batch > 32) need d % 256 == 0 and N + n_shared <= 136";
  if (d->L_host < 1 || d->L_host > d->L) return "L_host must be in [1, L]";
  if (!(d->v_e_max >= 0.0)) return "v_e_max must be >= 0";
  if (d->ep_size < 1 || d->ep_rank < 0 || d->ep_rank >= d->ep_size) return "ep_rank / ep_size invalid";
  if (d->N % d->ep_size != 0) return "N must be divisible by ep_size";
  if (d->tp_size < 1 || d->tp_rank < 0 || d->tp_rank >= d->tp_size) return "tp_rank / tp_size invalid";
  if (d->tp_size > 1 && d->ep_size != 1) return "tp_size > 1 needs ep_size == 1";
  if (d->I % ((int64_t)d->tp_size * d->row_granule) != 0) return "I must be a multiple of tp_size * row_granule";
  if (d->weight_format != MOEPIC_BF16 && d->weight_format != MOEPIC_Q4G64) return "weight_format invalid";
  if (d->weight_format == MOEPIC_Q4G64 && d->d % 64 != 0) return "Q4G64 experts need d % 64 == 0";
  if (d->max_batch > kDecodeMaxB && (d->row_granule % 64 != 0 || (d->I / d->tp_size) % 64 != 0))
    return "prefill batches (max_batch > 32) need row_granule and I / tp_size to be multiples of 64 (GEMM K tiles)";
  return "";
}

// Bytes of one interleaved expert row in the stored format: bf16 [gate|up|down]
// = 6d; Q4G64 = 3 x d/2 code bytes + 3 x d/64 (scale, min) bf16 pairs, padded to 16.
uint64_t row_bytes_of(const moepic_model_desc& d) {
  if (d.weight_format == MOEPIC_Q4G64) return (3ull * (d.d / 2) + 3ull * (d.d / 64) * 4 + 15) / 16 * 16;
  return 6ull * d.d;
}

// The context works on its tensor-parallel slice: I/tp_size rows of every expert (SURVEY
// §8(f) NEXT-4).  Everything below create / hostsim_create sees this local shape.
moepic_model_desc local_desc(const moepic_model_desc& d) {
  moepic_model_desc l = d;
  l.I = d.I / d.tp_size;
  return l;
}

// h is added to y by exactly one rank when the output is a sum over ranks (EP and TP)
inline bool adds_residual(const moepic_model_desc& d, uint32_t flags) {
  return (flags & MOEPIC_RESIDUAL) && d.ep_rank == 0 && d.tp_rank == 0;
}

ArenaLayout arena_layout(const moepic_model_desc& d) {
  ArenaLayout a{};
  const uint64_t rb = row_bytes_of(d);
  const int Nl = n_local(d);
  size_t off = 0;
  a.routers = off; off = align_up(off + (size_t)d.L * d.N * d.d * 2);
  // shared experts, slot pool and ping-pong buffers are one row region: every region starts a
  // whole number of rows after a.shared, so one 3-D tensor map {d, 3, rows} over it addresses
  // any segment by its row index (K2T)
  a.shared = off; off = align_up(off + (size_t)d.L * d.n_shared * d.I * rb);
  const size_t rowal = std::lcm((size_t)rb, kAlign);
  auto row_align = [&](size_t x) { return a.shared + align_up(x - a.shared, rowal); };
  a.pool_rows = (uint64_t)std::ceil(d.v_e_max * (double)d.I - 1e-9);
  off = row_align(off);
  a.pool = off; off = align_up(off + a.pool_rows * rb);
  a.plan_rows = (uint64_t)d.buffer_experts * d.I;
  a.od_rows = (uint64_t)std::min(Nl, d.max_batch * d.K) * d.I;
  for (int i = 0; i < 2; ++i) {
    off = row_align(off);
    a.buf[i] = off; off = align_up(off + (a.plan_rows + a.od_rows) * rb);
  }
  a.map_rows = (a.buf[1] - a.shared) / rb + a.plan_rows + a.od_rows;
  const uint64_t Bd = (uint64_t)std::min(d.max_batch, kDecodeMaxB);
  a.ws_floats = (uint64_t)d.d * (4ull * (Bd * d.K + d.n_shared * Bd) + 3ull * (kSMs + 1) * 8 + 64);
  if (k2t_eligible(d))   // K2T partials: one [G][B][d] area per launch, up to 3 launches per step
    a.ws_floats += 3ull * kSMs * std::min<uint64_t>(Bd, kK2TMaxB) * d.d;
  a.ws = off; off = align_up(off + a.ws_floats * 4);
  a.logits = off; off = align_up(off + (size_t)2 * d.max_batch * d.N * 8);
  a.ids = off; off = align_up(off + (size_t)d.max_batch * d.K * 4);
  a.w = off; off = align_up(off + (size_t)d.max_batch * d.K * 4);
  a.ranking = off; off = align_up(off + (size_t)d.N * 4);
  a.ticket = off; off = align_up(off + 64);
  a.rsel = off; off = align_up(off + (size_t)d.N * 16);   // k1_select: cnt int32 [N] | max u64 [N]
  a.trec = off; off = align_up(off + (size_t)2 * kProfRing * 8);   // profiling: start [ring] | end [ring]
  a.hstage = off; off = align_up(off + (size_t)d.max_batch * d.d * 2);   // layer_forward_host input rows
  a.ystage = off;                                                          // ... and prefill outputs
  if (d.max_batch > kDecodeMaxB) off = align_up(off + (size_t)d.max_batch * d.d * 4);
  a.pf_rows = a.wdq_rows = 0;
  a.xperm = a.aact = a.yperm = a.pos = a.cursor = a.wdq = off;
  if (d.max_batch > kDecodeMaxB) {
    const uint64_t T = d.max_batch;
    a.pf_rows = T * d.K + (uint64_t)d.N * (kPfBM - 1) + (uint64_t)d.n_shared * (T + kPfBM - 1) + kPfBM;
    a.xperm = off; off = align_up(off + a.pf_rows * d.d * 2, 1024);
    a.aact = off; off = align_up(off + a.pf_rows * d.I * 2, 1024);
    a.yperm = off; off = align_up(off + a.pf_rows * d.d * 4);
    a.pos = off; off = align_up(off + T * d.K * 4);
    a.cursor = off; off = align_up(off + (size_t)d.N * 4);
    if (d.weight_format == MOEPIC_Q4G64) {   // reading Q32: one group's segments dequantised to fp16 rows
      a.wdq_rows = (uint64_t)(Nl + d.n_shared) * d.I;
      a.wdq = off; off = align_up(off + a.wdq_rows * 6ull * d.d, 1024);
    }
  }
  a.total = off;
  return a;
}

moepic_status fail(std::string* err, moepic_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (err) *err = buf;
  return st;
}

CacheParams to_params(const moepic_cache_config* c, int L) {
  CacheParams p;
  p.v_e = c->v_e;
  if (c->v_i) p.v_i.assign(c->v_i, c->v_i + L);
  if (c->theta_i) p.theta_i.assign(c->theta_i, c->theta_i + L);
  p.use_solver = c->use_solver != 0;
  p.policy = c->policy;
  p.rho = c->rho;
  p.omega = c->omega;
  p.zeta = c->zeta;
  p.t_att = c->t_att; p.t_moe = c->t_moe; p.t_head = c->t_head; p.t_load = c->t_load_exp;
  if (c->y_cap_i) p.y_cap.assign(c->y_cap_i, c->y_cap_i + L);
  if (c->prefetch_rows_i) p.pf_rows.assign(c->prefetch_rows_i, c->prefetch_rows_i + L);
  p.prefetch = c->prefetch != 0;
  p.seed = c->seed;
  return p;
}

void write_config_out(const ControlPlane& cp, moepic_config_out* out) {
  if (!out) return;
  for (int i = 0; i < cp.L; ++i) {
    const LayerState& l = cp.layers[i];
    if (out->C_i) out->C_i[i] = l.C;
    if (out->I_top_i) out->I_top_i[i] = l.I_top;
    if (out->theta_eff_i) out->theta_eff_i[i] = (double)l.I_top / (double)cp.I;
    if (out->V_i) out->V_i[i] = l.V;
  }
}

// shared-expert rows this EP rank computes: [r*I/G, (r+1)*I/G) (split identity)
inline int64_t shared_lo(const ControlPlane& cp) { return (int64_t)cp.ep_rank * cp.I / cp.ep_size; }
inline int64_t shared_hi(const ControlPlane& cp) { return (int64_t)(cp.ep_rank + 1) * cp.I / cp.ep_size; }

uint64_t step_hbm_bytes(const ControlPlane& cp, const StepResult& r, int B, int n_router,
                        uint64_t prefetch_bytes) {
  const uint64_t rb = (uint64_t)cp.row_bytes;
  return (uint64_t)r.A.size() * cp.I * rb + (uint64_t)cp.n_shared * (shared_hi(cp) - shared_lo(cp)) * rb +
         (uint64_t)n_router * cp.N * cp.d * 2 + (uint64_t)B * cp.d * 2 + (uint64_t)B * cp.d * 4 + r.d2d_bytes +
         r.pcie_ondemand + prefetch_bytes;
}

void fill_step_trace(moepic_trace* tr, const StepResult& r, const Plan* next) {
  if (!tr) return;
  tr->n_act = (int32_t)r.A.size();
  for (size_t a = 0; a < r.A.size(); ++a) {
    if (tr->act_expert) tr->act_expert[a] = r.A[a];
    if (tr->act_class) tr->act_class[a] = r.cls[a];
  }
  tr->n_adm = (int32_t)r.adm.size();
  for (size_t a = 0; a < r.adm.size(); ++a) {
    if (tr->adm_expert) tr->adm_expert[a] = r.adm[a].expert;
    if (tr->adm_victim) tr->adm_victim[a] = r.adm[a].victim;
  }
  tr->n_plan = 0;
  tr->plan_layer = -1;
  tr->pcie_prefetch_bytes = 0;
  if (next && next->valid) {
    tr->plan_layer = next->target;
    tr->n_plan = (int32_t)next->items.size();
    if (tr->ranking)
      for (size_t k = 0; k < next->ranking.size(); ++k) tr->ranking[k] = next->ranking[k];
    for (size_t k = 0; k < next->items.size(); ++k) {
      if (tr->plan_expert) tr->plan_expert[k] = next->items[k].expert;
      if (tr->plan_full) tr->plan_full[k] = next->items[k].full ? 1 : 0;
    }
  }
  tr->pcie_ondemand_bytes = r.pcie_ondemand;
}

uint64_t plan_bytes(const Plan& p, int64_t rb) {
  uint64_t s = 0;
  for (auto& it : p.items) s += (uint64_t)it.rows * (uint64_t)rb;
  return s;
}

// NCCL entry points, resolved with dlsym from the libnccl.so.2 the process already has (torch's)
// or the system one: the library itself has no link-time NCCL dependency.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

const NcclApi& nccl_api() {
  static NcclApi a = [] {
    NcclApi x;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return x;
#define NCCL_SYM(f) x.f = reinterpret_cast<decltype(x.f)>(dlsym(h, "nccl" #f))
    NCCL_SYM(GetUniqueId); NCCL_SYM(CommInitRank); NCCL_SYM(CommDestroy); NCCL_SYM(AllGather);
    NCCL_SYM(AllReduce); NCCL_SYM(Send); NCCL_SYM(Recv); NCCL_SYM(GroupStart); NCCL_SYM(GroupEnd);
    NCCL_SYM(GetErrorString);
#undef NCCL_SYM
    x.ok = x.GetUniqueId && x.CommInitRank && x.CommDestroy && x.AllGather && x.AllReduce && x.Send && x.Recv &&
           x.GroupStart && x.GroupEnd && x.GetErrorString;
    return x;
  }();
  return a;
}

// handle blob one rank publishes (moepic_group_handle) and every rank joins with
struct GroupBlob {
  uint64_t magic;
  int32_t rank, world, transport, kind;
  uint64_t region_bytes;
  cudaIpcMemHandle_t ipc;
  ncclUniqueId nccl_id;
};
constexpr uint64_t kGroupMagic = 0x4d6f45706963477bull;   // "MoEpicG{"

// the group of ranks one context exchanges data with (EP or TP), SURVEY §8(e)
struct Group {
  int transport = MOEPIC_TRANSPORT_PEER;
  int G = 1, me = 0;
  int T_max = 0, Bl_max = 0, B_dec = 0;
  bool joined = false;
  uint8_t* region = nullptr;          // own exchange region (cudaMalloc: IPC-exportable)
  EpOffsets of{};
  EpPeers pr{};
  bool opened[kEpMaxRanks] = {};
  unsigned long long epoch[kEpPhases] = {};
  int32_t* idx_h = nullptr;           // mapped pinned index lists (host writes, kernels read)
  int32_t* idx_d = nullptr;
  size_t idx_ints = 0;
  ncclComm_t comm = nullptr;
  ncclUniqueId nccl_id{};
  std::vector<int32_t> ids_all;
  std::vector<float> w_all;
  EpLists lists;
};

EpOffsets ep_offsets(int G, int T_max, int Bl_max, int B_dec, int K, int d) {
  EpOffsets o{};
  size_t off = 0;
  auto take = [&](size_t bytes) { const size_t r = off; off = align_up(off + bytes); return r; };
  o.sig = take(sizeof(unsigned long long) * kEpPhases * kEpMaxRanks);
  o.ctr = take(sizeof(unsigned int) * kEpPhases);
  const size_t comb_rows = (size_t)Bl_max * std::min(G, K);
  for (int h = 0; h < 2; ++h) {
    o.ids_all[h] = take((size_t)T_max * K * 4);
    o.w_all[h] = take((size_t)T_max * K * 4);
    o.recv[h] = take((size_t)T_max * d * 2);
    o.comb[h] = take(comb_rows * d * 4);
    o.red[h] = take((size_t)G * B_dec * d * 4);
  }
  o.ysub = take((size_t)T_max * d * 4);
  o.sendbuf = take(comb_rows * d * 2);
  o.total = off;
  return o;
}

}  // namespace

// ====================================================================== context
struct moepic_ctx {
  // K2T: one tensor map over the arena's row region (shared experts | slot pool | buffers)
  alignas(64) CUtensorMap tm_rows;
  bool k2t = false;
  int k2t_mode = 0;   // MOEPIC_K2T_MODE (tools): 1 = K2T streams its operands without MMAs
  // kernel parameter blocks (large: built here, not on the stack; calls on a ctx are serialised)
  std::unique_ptr<K2Params> kp = std::make_unique<K2Params>();
  std::unique_ptr<K2TParams> ktp = std::make_unique<K2TParams>();
  std::unique_ptr<PfPermuteParams> pf_pp = std::make_unique<PfPermuteParams>();
  std::unique_ptr<PfGemmParams> pf_gp = std::make_unique<PfGemmParams>();
  std::unique_ptr<PfDequantParams> pf_dq = std::make_unique<PfDequantParams>();
  std::unique_ptr<CombineParams> cpar = std::make_unique<CombineParams>();
  std::unique_ptr<Group> grp;        // set by moepic_group_handle / moepic_group_join
  moepic_model_desc desc{};         // local shape: desc.I = I_full / tp_size rows per expert
  int32_t I_full = 0;               // rows per expert in the caller's (HF) tensors
  ArenaLayout lay{};
  std::unique_ptr<ControlPlane> cp;
  uint8_t* arena = nullptr;
  uint8_t* host_experts = nullptr;   // pinned [L_host][N_local][I][6d]
  uint8_t* mailbox = nullptr;        // mapped pinned
  uint8_t* mailbox_dev = nullptr;
  cudaStream_t copy = nullptr;
  cudaStream_t copy2 = nullptr;      // second on-demand copy stream (MOEPIC_COPY_STREAMS=2)
  cudaEvent_t ev_copy2 = nullptr;
  cudaEvent_t ev_od = nullptr, ev_od_head = nullptr, ev_plan[2] = {nullptr, nullptr}, ev_step[2] = {nullptr, nullptr};
  bool ev_step_rec[2] = {false, false};
  cudaEvent_t ev_tmp = nullptr;
  std::vector<uint64_t> slot_base;   // per layer: byte offset inside the pool
  bool configured = false;
  Plan pending;
  int last_buf = 1;
  uint32_t seq = 0;
  uint64_t bar_base = 0;             // grid-barrier arrivals so far (fused combine)
  bool poisoned = false;
  bool committed = false;            // layer_forward: the control plane committed this step
  // MOEPIC_FAULT_AT_STEP=n (tests): the n-th layer_forward launches a kernel that traps, so a
  // real CUDA failure travels the ERUNTIME -> ESTATE path
  int64_t fault_at_step = 0, fault_steps = 0;
  // MOEPIC_POISON=1 (tests): every ping-pong half and the K2 workspace are filled
  // with 0xFF bytes (bf16 / fp32 NaN) once the step that used them is done, the slot pool before
  // every re-layout, and a victim's slot before the new top lands in it -- a kernel that reads a
  // segment before its copy landed, or a stale buffer, produces NaN and fails parity
  bool poison = false;
  std::string err;
  moepic_counters ctr{};
  // event profiling (moepic_profile): pairs recorded on the launching stream
  struct ProfEv {
    cudaEvent_t a, b;
    int cls;
    uint64_t bytes;
  };
  // prefetch feed queue (cancel_prefetch): chunks of the pending plan, issued a few at a
  // time on the copy stream while the host waits for routing; unissued chunks of experts that
  // the router did not activate are dropped
  struct FeedChunk {
    uint8_t* dst;
    const uint8_t* src;
    size_t bytes;
    int32_t item;
  };
  size_t kFeedChunk = 8ull << 20;
  // decode: the step's last on-demand copy is split so its final tail_bytes land last; the K2
  // launch over everything else runs while the tail is still in flight (0 disables)
  size_t od_tail_bytes = 64ull << 20;
  // decode: a step whose last on-demand copy is too small to split makes that whole copy the tail
  // (MOEPIC_OD_SPLIT_BOUNDARY=0 turns this off)
  bool od_split_boundary = true;
  // decode, gated tail (MOEPIC_K2_GATE, default on): ONE K2 launch per step covers the resident,
  // prefetched and on-demand rows; the tail of the last on-demand copy is still in flight at
  // launch and the CTAs stream it after the copy stream's flag (cuStreamWriteValue32 after that
  // copy).  The tail is sized so that it lands while K2 streams the rest (od_tail_auto: a
  // fraction k2_gate_frac of the K2 time of the step's rows, at the measured link rate), so the
  // gate rarely stalls, and the link idles only for the tail's few rows + the combine.  Without
  // the gate (or when the step does not fit one K2 launch) the tail gets its own launch.
  bool k2_gate = true;
  bool pf_merge_ab = true;      // prefill: resident + prefetched segments in one GEMM group (MOEPIC_PF_MERGE_AB)
  bool k2_gate_force = false;   // MOEPIC_K2_GATE=2: gate every decode step, whatever its size
  bool od_tail_auto = true;
  double k2_gate_frac = 0.8;
  int64_t tail_split_x = 2;   // MOEPIC_TAIL_SPLIT_X
  unsigned int gate_seq = 0;
  // tail-size controller: each gated launch records every CTA's wait at the gate (ns) in mapped
  // host memory; the next gated step reads the previous launch's mean over the CTAs with gated
  // rows (that launch finished before this step's router, whose mailbox the host has seen) and
  // scales the tail: a mean wait over 8 us shrinks it 8 %, under 2 us grows it 3 % -- the tail
  // lands just after K2 reaches it, so K2 runs under the link and waits only a few us.
  // MOEPIC_GATE_ADAPT=0: fixed.
  bool gate_adapt = true;
  double gate_ctrl = 1.0;
  double gate_wait_lo_us = 2.0, gate_wait_hi_us = 8.0;   // mean-wait band (MOEPIC_GATE_WAIT_US=lo,hi)
  unsigned int* stall_h = nullptr;   // [2][kStallSlot] mapped pinned
  unsigned int* stall_d = nullptr;
  int stall_slot = 0, stall_prev = -1, stall_prev_g = 0;
  uint64_t gate_steps = 0;
  double gate_wait_us_sum = 0.0;
  using WriteValue32Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
  WriteValue32Fn write_value32 = nullptr;
  // MOEPIC_TIMELINE=<path> (tools): per decode layer step, %globaltimer stamps of the router, the
  // K2 launches before the final one, the final (combining) K2 and the completion of the step's
  // last on-demand copy (a one-thread kernel on the copy stream), plus host stamps of the call,
  // routing seen, first / last copy issued and return, converted to GPU time; JSON lines at destroy
  std::string tl_path;
  unsigned long long* tl_dev = nullptr;   // [kProfRing] starts | [kProfRing] ends (stamp_start/end)
  int64_t tl_off0 = 0, tl_h0 = 0;         // GPU ns - host steady_clock ns at host time tl_h0 (create)
  // clock offset by handshake over mapped host memory: the kernel announces itself, the host reads
  // its clock and releases it, the kernel stamps %globaltimer when it sees the release (one PCIe
  // read latency, ~1 us, after the host stamp); best of 10.  %globaltimer drifts against the host
  // clock by tens of ppm, so the dump re-calibrates and interpolates linearly.
  void tl_calibrate(int64_t& host_ns, int64_t& off) {
    auto* hv = reinterpret_cast<volatile unsigned long long*>(scratch_h);
    int64_t best = INT64_MAX;
    for (int it = 0; it < 10; ++it) {
      hv[0] = hv[1] = hv[2] = 0;
      launch_clock_sync(reinterpret_cast<unsigned long long*>(scratch_d), nullptr);
      while (hv[0] == 0) {
      }
      const auto a = std::chrono::steady_clock::now();
      hv[2] = 1;
      while (hv[1] == 0) {
      }
      const auto b = std::chrono::steady_clock::now();
      const int64_t ha = std::chrono::duration_cast<std::chrono::nanoseconds>(a.time_since_epoch()).count();
      const int64_t hb = std::chrono::duration_cast<std::chrono::nanoseconds>(b.time_since_epoch()).count();
      if (hb - ha < best) {
        best = hb - ha;
        host_ns = (ha + hb) / 2;
        off = (int64_t)hv[1] - host_ns;
      }
    }
    cudaDeviceSynchronize();
  }
  int tl_rec = -1;
  int64_t tl_skip = 0, tl_seen = 0;       // MOEPIC_TIMELINE_SKIP: layer steps before recording starts
  struct TlHost {
    int layer;
    int64_t t[5];
    uint64_t od_bytes;
  };
  std::vector<TlHost> tl_host;
  static constexpr int kTlMax = kProfRing / 8;
  unsigned long long* tl_slot(int k) const {
    return (tl_dev && tl_rec >= 0 && tl_rec < kTlMax) ? tl_dev + (size_t)tl_rec * 8 + k : nullptr;
  }
  // the decode router is launched as a programmatic dependent of the previous kernel on the
  // stream (MOEPIC_PDL=0 turns this off)
  bool pdl = true;
  size_t kFeedDepth = 3;
  static constexpr int kFeedRing = 16;
  bool cancel_prefetch = true;
  std::vector<FeedChunk> feed;
  size_t feed_next = 0;
  std::vector<char> feed_cancel;
  cudaEvent_t feed_ev[kFeedRing] = {};
  int feed_ev_next = 0;
  std::vector<int> feed_inflight;   // ring indices, oldest first

  // issue chunks until `depth` are in flight; returns false on a CUDA error
  bool feed_pump(size_t depth) {
    while (!feed_inflight.empty() && cudaEventQuery(feed_ev[feed_inflight.front()]) == cudaSuccess)
      feed_inflight.erase(feed_inflight.begin());
    const bool track = depth != (size_t)-1;
    while (feed_next < feed.size() && feed_inflight.size() < depth) {
      const FeedChunk& c = feed[feed_next++];
      if (feed_cancel[c.item]) continue;
      if (cudaMemcpyAsync(c.dst, c.src, c.bytes, cudaMemcpyHostToDevice, copy) != cudaSuccess) return false;
      ctr.h2d_copies++;
      ctr.pcie_prefetch_bytes += c.bytes;
      if (!track) continue;
      const int e = feed_ev_next;
      feed_ev_next = (feed_ev_next + 1) % kFeedRing;
      if (cudaEventRecord(feed_ev[e], copy) != cudaSuccess) return false;
      feed_inflight.push_back(e);
    }
    return true;
  }
  void feed_drop() {
    feed.clear();
    feed_next = 0;
    feed_cancel.clear();
  }

  // diagnostics switches, read once at create from the environment (tools only; no effect on
  // results): MOEPIC_K1_TRACE / MOEPIC_K2_TRACE phase stamps, MOEPIC_HOST_TIMING host phases,
  // MOEPIC_PF_CTA_PAIR = 0/1 forces the prefill CTA-pair choice (tests), MOEPIC_FEED_CHUNK_KB /
  // MOEPIC_FEED_DEPTH / MOEPIC_NO_SOLVER_YCAP prefetch-feed experiments (scripts/feed_sweep.py)
  bool k1_trace = false, k2_trace = false, host_timing = false;
  int pf_cta_pair = -1;
  double ht[4] = {0, 0, 0, 0};
  double hc[2] = {0, 0};
  double hp[4] = {0, 0, 0, 0};
  double hf[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  uint64_t hf_n = 0;
  double hh[3] = {0, 0, 0};   // host-buffer entry: stage-in, forward call, sync + y read (us)
  uint64_t hh_n = 0;
  uint64_t hc_n = 0;
  uint64_t ht_n = 0;
  unsigned long long* k1dbg = nullptr;   // MOEPIC_K1_TRACE ring (tools)
  uint64_t k1dbg_n = 0;
  bool profiling = false;
  std::vector<ProfEv> prof;
  size_t prof_used = 0;
  moepic_kernel_stats prof_acc[4]{};

  uint32_t prof_mask = 0xF;   // kernel classes timed (moepic_profile)
  int prof_begin(cudaStream_t s, int cls) {
    if (!profiling || !((prof_mask >> cls) & 1u)) return -1;
    if (prof_used == prof.size()) {
      ProfEv e{};
      if (cudaEventCreate(&e.a) != cudaSuccess || cudaEventCreate(&e.b) != cudaSuccess) return -1;
      prof.push_back(e);
    }
    ProfEv& e = prof[prof_used];
    e.cls = cls;
    e.bytes = 0;
    if (cudaEventRecord(e.a, s) != cudaSuccess) return -1;
    return (int)prof_used++;
  }
  void prof_end(int idx, cudaStream_t s, uint64_t bytes) {
    if (idx < 0) return;
    prof[idx].bytes = bytes;
    cudaEventRecord(prof[idx].b, s);
    if (prof_used >= (size_t)kProfRing) prof_drain();
  }
  // in-kernel timestamp record of profiling slot idx (device_utils.cuh), nullptr when off
  unsigned long long* tstamp(int idx) const {
    return idx < 0 ? nullptr : reinterpret_cast<unsigned long long*>(arena + lay.trec) + idx;
  }
  void tstamp_reset(size_t n) {
    if (n == 0) return;
    cudaMemset(arena + lay.trec, 0xFF, n * 8);
    cudaMemset(arena + lay.trec + (size_t)kProfRing * 8, 0, n * 8);
  }
  void prof_drain() {
    std::vector<unsigned long long> ts(prof_used), te(prof_used);
    if (prof_used) {
      cudaDeviceSynchronize();
      cudaMemcpy(ts.data(), arena + lay.trec, prof_used * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(te.data(), arena + lay.trec + (size_t)kProfRing * 8, prof_used * 8, cudaMemcpyDeviceToHost);
    }
    for (size_t i = 0; i < prof_used; ++i) {
      float ms = 0.f;
      cudaEventSynchronize(prof[i].b);
      cudaEventElapsedTime(&ms, prof[i].a, prof[i].b);
      moepic_kernel_stats& k = prof_acc[prof[i].cls];
      k.launches++;
      k.total_ms += ms;
      k.bytes += prof[i].bytes;
      if (te[i] > ts[i] && ts[i] != ~0ull) k.kernel_ms += (double)(te[i] - ts[i]) * 1e-6;
    }
    tstamp_reset(prof_used);
    if (prof_used) cudaDeviceSynchronize();
    prof_used = 0;
  }
  std::vector<int32_t> ids_h, rank_h;
  std::vector<float> w_h;
  uint8_t* scratch_h = nullptr;      // mapped pinned staging for *_host calls (h | y), sized at create
  uint8_t* scratch_d = nullptr;      // its device alias
  size_t scratch_bytes = 0;

  uint64_t rb() const { return row_bytes_of(desc); }
  int Nl() const { return n_local(desc); }
  int first_local() const { return desc.ep_rank * Nl(); }
  const uint8_t* host_expert(int layer, int e) const {
    const int pl = layer % desc.L_host;
    return host_experts + ((uint64_t)pl * Nl() + (e - first_local())) * desc.I * rb();
  }
  uint8_t* slot_ptr(int layer, int slot) const {
    return arena + lay.pool + slot_base[layer] + (uint64_t)slot * cp->layers[layer].I_top * rb();
  }
  uint8_t* plan_ptr(int buf, int64_t row) const { return arena + lay.buf[buf] + (uint64_t)row * rb(); }
  uint8_t* od_ptr(int buf, int64_t row) const {
    return arena + lay.buf[buf] + (lay.plan_rows + (uint64_t)row) * rb();
  }
  uint8_t* shared_ptr(int layer, int s) const {
    return arena + lay.shared + ((uint64_t)layer * desc.n_shared + s) * desc.I * rb();
  }
  const uint16_t* router(int layer) const {
    return reinterpret_cast<const uint16_t*>(arena + lay.routers) + (size_t)layer * desc.N * desc.d;
  }
};

#define CK(call)                                                                           \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess) {                                                               \
      ctx->poisoned = true;                                                                \
      return fail(&ctx->err, MOEPIC_ERUNTIME, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                     \
    }                                                                                      \
  } while (0)

#define CTX_GUARD()                                                     \
  do {                                                                  \
    if (!ctx) return MOEPIC_EINVAL;                                     \
    if (ctx->poisoned) return MOEPIC_ESTATE;                            \
  } while (0)

extern "C" {

moepic_status moepic_arena_bytes(const moepic_model_desc* desc, size_t* bytes) {
  if (!bytes || !validate_desc(desc).empty()) return MOEPIC_EINVAL;
  *bytes = arena_layout(local_desc(*desc)).total;
  return MOEPIC_OK;
}

moepic_status moepic_create(const moepic_model_desc* desc, void* dev_arena, size_t dev_bytes,
                            moepic_ctx** out) {
  if (!out) return MOEPIC_EINVAL;
  *out = nullptr;
  if (!validate_desc(desc).empty()) return MOEPIC_EINVAL;
  if (!dev_arena || (reinterpret_cast<uintptr_t>(dev_arena) % kAlign) != 0) return MOEPIC_EINVAL;
  const moepic_model_desc full = *desc;
  const moepic_model_desc local = local_desc(full);
  desc = &local;
  ArenaLayout lay = arena_layout(*desc);
  if (dev_bytes < lay.total) return MOEPIC_ENOMEM;
  auto* ctx = new (std::nothrow) moepic_ctx();
  if (!ctx) return MOEPIC_ENOMEM;
  ctx->desc = *desc;
  ctx->I_full = full.I;
  ctx->lay = lay;
  ctx->arena = static_cast<uint8_t*>(dev_arena);
  ctx->cp.reset(new ControlPlane(desc->L, desc->N, desc->K, desc->d, desc->I, desc->row_granule,
                                 desc->buffer_experts, desc->n_shared, desc->ep_rank, desc->ep_size));
  ctx->cp->row_bytes = (int64_t)row_bytes_of(*desc);
  char kerr[256];
  auto bail = [&](moepic_status st) {
    moepic_destroy(ctx);
    return st;
  };
  if (!kernels_init(kerr, sizeof kerr)) return bail(MOEPIC_ERUNTIME);
  ctx->scratch_bytes = align_up((size_t)desc->max_batch * desc->d * 2) + (size_t)desc->max_batch * desc->d * 4;
  if (cudaHostAlloc(&ctx->scratch_h, ctx->scratch_bytes, cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->scratch_d), ctx->scratch_h, 0) != cudaSuccess)
    return bail(MOEPIC_ENOMEM);
  if (desc->max_batch > kDecodeMaxB && !prefill_init(kerr, sizeof kerr)) return bail(MOEPIC_ERUNTIME);
  if (k2t_eligible(*desc) && !(getenv("MOEPIC_K2T") && atoi(getenv("MOEPIC_K2T")) == 0)) {
    if (!pf_tmap_weights(&ctx->tm_rows, ctx->arena + lay.shared, lay.map_rows, desc->d, 64))
      return bail(MOEPIC_ERUNTIME);
    ctx->k2t = true;
  }
  const uint64_t host_bytes = (uint64_t)desc->L_host * ctx->Nl() * desc->I * ctx->rb();
  if (cudaHostAlloc(&ctx->host_experts, host_bytes, cudaHostAllocDefault) != cudaSuccess) {
    cudaGetLastError();
    return bail(MOEPIC_ENOMEM);
  }
  const size_t mb_bytes = 64 + ((size_t)desc->max_batch * desc->K * 2 + (size_t)desc->N) * 8;
  if (cudaHostAlloc(&ctx->mailbox, mb_bytes, cudaHostAllocMapped) != cudaSuccess) return bail(MOEPIC_ENOMEM);
  memset(ctx->mailbox, 0, mb_bytes);
  if (cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->mailbox_dev), ctx->mailbox, 0) != cudaSuccess)
    return bail(MOEPIC_ERUNTIME);
  if (cudaStreamCreateWithFlags(&ctx->copy, cudaStreamNonBlocking) != cudaSuccess) return bail(MOEPIC_ERUNTIME);
  {
    const char* e = getenv("MOEPIC_COPY_STREAMS");   // default 1: two streams measured neutral
    if (e && atoi(e) >= 2) {
      if (cudaStreamCreateWithFlags(&ctx->copy2, cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&ctx->ev_copy2, cudaEventDisableTiming) != cudaSuccess)
        return bail(MOEPIC_ERUNTIME);
    }
  }
  cudaEvent_t* evs[] = {&ctx->ev_od, &ctx->ev_od_head, &ctx->ev_plan[0], &ctx->ev_plan[1], &ctx->ev_step[0], &ctx->ev_step[1],
                        &ctx->ev_tmp};
  for (auto* e : evs)
    if (cudaEventCreateWithFlags(e, cudaEventDisableTiming) != cudaSuccess) return bail(MOEPIC_ERUNTIME);
  for (auto& e : ctx->feed_ev)
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return bail(MOEPIC_ERUNTIME);
  if (cudaMemset(ctx->arena + lay.ticket, 0, 64) != cudaSuccess ||
      cudaMemset(ctx->arena + lay.rsel, 0, (size_t)desc->N * 16) != cudaSuccess)
    return bail(MOEPIC_ERUNTIME);
  if (const char* e = getenv("MOEPIC_FEED_CHUNK_KB")) ctx->kFeedChunk = (size_t)atol(e) << 10;
  if (const char* e = getenv("MOEPIC_OD_TAIL_MB")) ctx->od_tail_bytes = (size_t)atol(e) << 20, ctx->od_tail_auto = false;
  if (const char* e = getenv("MOEPIC_OD_TAIL_KB")) ctx->od_tail_bytes = (size_t)atol(e) << 10, ctx->od_tail_auto = false;   // tests: small shapes
  if (const char* e = getenv("MOEPIC_K2_GATE")) ctx->k2_gate = atoi(e) != 0, ctx->k2_gate_force = atoi(e) == 2;
  if (const char* e = getenv("MOEPIC_K2_GATE_FRAC")) ctx->k2_gate_frac = atof(e);
  if (const char* e = getenv("MOEPIC_PF_MERGE_AB")) ctx->pf_merge_ab = atoi(e) != 0;
  if (const char* e = getenv("MOEPIC_TAIL_SPLIT_X")) ctx->tail_split_x = std::max(2L, atol(e));
  if (const char* e = getenv("MOEPIC_GATE_ADAPT")) ctx->gate_adapt = atoi(e) != 0;
  if (const char* e = getenv("MOEPIC_GATE_WAIT_US")) {
    double lo = 0, hi = 0;
    if (sscanf(e, "%lf,%lf", &lo, &hi) == 2 && lo >= 0 && hi > lo) ctx->gate_wait_lo_us = lo, ctx->gate_wait_hi_us = hi;
  }
  if (ctx->k2_gate) {
    if (cudaHostAlloc(&ctx->stall_h, 2 * kStallSlot * sizeof(unsigned int), cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->stall_d), ctx->stall_h, 0) != cudaSuccess)
      return bail(MOEPIC_ENOMEM);
    memset(ctx->stall_h, 0, 2 * kStallSlot * sizeof(unsigned int));
  }
  if (ctx->k2_gate) {   // the copy stream's flag write (driver API, resolved through the runtime)
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess && fn)
      ctx->write_value32 = reinterpret_cast<moepic_ctx::WriteValue32Fn>(fn);
    else
      ctx->k2_gate = false;
  }
  if (const char* e = getenv("MOEPIC_OD_SPLIT_BOUNDARY")) ctx->od_split_boundary = atoi(e) != 0;
  if (const char* e = getenv("MOEPIC_PDL")) ctx->pdl = atoi(e) != 0;
  if (const char* e = getenv("MOEPIC_TIMELINE")) {
    ctx->tl_path = e;
    if (const char* k = getenv("MOEPIC_TIMELINE_SKIP")) ctx->tl_skip = atol(k);
    if (cudaMalloc(&ctx->tl_dev, (size_t)2 * kProfRing * 8) != cudaSuccess ||
        cudaMemset(ctx->tl_dev, 0xFF, (size_t)kProfRing * 8) != cudaSuccess ||
        cudaMemset(ctx->tl_dev + kProfRing, 0, (size_t)kProfRing * 8) != cudaSuccess)
      return bail(MOEPIC_ERUNTIME);
    ctx->tl_calibrate(ctx->tl_h0, ctx->tl_off0);
    cudaDeviceSynchronize();
  }
  if (const char* e = getenv("MOEPIC_FEED_DEPTH")) ctx->kFeedDepth = (size_t)std::min(atol(e), (long)moepic_ctx::kFeedRing);
  if (const char* e = getenv("MOEPIC_PF_CTA_PAIR")) ctx->pf_cta_pair = atoi(e) ? 1 : 0;
  if (const char* e = getenv("MOEPIC_K2T_MODE")) ctx->k2t_mode = atoi(e);
  ctx->k1_trace = getenv("MOEPIC_K1_TRACE") != nullptr;
  ctx->k2_trace = getenv("MOEPIC_K2_TRACE") != nullptr;
  ctx->host_timing = getenv("MOEPIC_HOST_TIMING") != nullptr;
  if (const char* e = getenv("MOEPIC_FAULT_AT_STEP")) ctx->fault_at_step = atol(e);
  ctx->poison = getenv("MOEPIC_POISON") != nullptr && atoi(getenv("MOEPIC_POISON")) != 0;
  ctx->cp->solver_y_cap = getenv("MOEPIC_NO_SOLVER_YCAP") == nullptr;
  ctx->slot_base.assign(desc->L, 0);
  ctx->ids_h.resize((size_t)desc->max_batch * desc->K);
  ctx->w_h.resize((size_t)desc->max_batch * desc->K);
  ctx->rank_h.resize(desc->N);
  *out = ctx;
  return MOEPIC_OK;
}

moepic_status moepic_load_router(moepic_ctx* ctx, int32_t layer, const uint16_t* w_bf16) {
  CTX_GUARD();
  if (layer < 0 || layer >= ctx->desc.L) return fail(&ctx->err, MOEPIC_EINVAL, "layer out of range");
  if (!w_bf16) return fail(&ctx->err, MOEPIC_EINVAL, "w_bf16 is NULL");
  CK(cudaMemcpy((void*)ctx->router(layer), w_bf16, (size_t)ctx->desc.N * ctx->desc.d * 2,
                cudaMemcpyHostToDevice));
  return MOEPIC_OK;
}

// HF layout -> row-interleaved rows [gate_r | up_r | down[:, r]] for r in [r0, r0 + I); the HF
// tensors hold I_full rows (gate/up [I_full][d], down [d][I_full]); r0 = tp_rank * I.
// The down column of a stored bf16 row is re-encoded as fp16 (reading Q31): exact for
// every bf16 value of magnitude in [2^-14, 65280] (the bf16 mantissa has 8 bits, fp16's 11), round
// to nearest even below 2^-14 (fp16 subnormals, absolute error <= 2^-25).  The down-projection
// MMAs then take an fp16 activation: one MMA per K step with an 11-bit activation mantissa.
static inline uint16_t bf16_to_f16(uint16_t b) {
  const uint32_t sign = (uint32_t)(b & 0x8000u);
  const uint32_t ax = (uint32_t)(b & 0x7FFFu) << 16;   // |x| as fp32 bits
  if (ax >= 0x47800000u) return (uint16_t)(sign | 0x7C00u | (ax > 0x7F800000u ? 0x200u : 0u));   // >= 2^16: inf / nan
  if (ax < 0x38800000u) {   // below 2^-14: fp16 subnormal (or zero), value = round(|x| * 2^24)
    float v;
    memcpy(&v, &ax, 4);
    return (uint16_t)(sign | (uint32_t)std::nearbyint(v * 16777216.0f));
  }
  return (uint16_t)(sign | ((((ax >> 23) - 112u) << 10) | ((ax >> 13) & 0x3FFu)));   // exact: 7-bit mantissa
}
// load_expert rejects down weights fp16 cannot hold (|x| >= 65536 or not finite)
static inline bool down_fits_f16(const uint16_t* down, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if ((down[i] & 0x7FFFu) >= 0x4780u) return false;
  return true;
}

static void pack_rows_bf16(uint8_t* dst, const uint16_t* gate, const uint16_t* up, const uint16_t* down, int d,
                           int I, int r0, int I_full) {
  gate += (size_t)r0 * d;
  up += (size_t)r0 * d;
  down += r0;
  const size_t rowe = 3ull * d;
  uint16_t* o = reinterpret_cast<uint16_t*>(dst);
#pragma omp parallel for schedule(static)
  for (int rb = 0; rb < I; rb += 64) {
    const int re = std::min(I, rb + 64);
    for (int r = rb; r < re; ++r) {
      memcpy(o + (size_t)r * rowe, gate + (size_t)r * d, (size_t)d * 2);
      memcpy(o + (size_t)r * rowe + d, up + (size_t)r * d, (size_t)d * 2);
    }
    for (int k0 = 0; k0 < d; k0 += 64) {
      const int ke = std::min(d, k0 + 64);
      for (int r = rb; r < re; ++r) {
        uint16_t* orow = o + (size_t)r * rowe + 2 * d;
        for (int k = k0; k < ke; ++k) orow[k] = bf16_to_f16(down[(size_t)k * I_full + r]);
      }
    }
  }
}

static inline float bf16f(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}
static inline uint16_t bf16_down(float v) {   // largest bf16 <= v (finite v)
  uint32_t u;
  memcpy(&u, &v, 4);
  uint16_t t = (uint16_t)(u >> 16);
  if (v < 0 && bf16f(t) > v) ++t;
  return t;
}
static inline uint16_t bf16_up(float v) {     // smallest bf16 >= v (v >= 0)
  uint32_t u;
  memcpy(&u, &v, 4);
  uint16_t t = (uint16_t)(u >> 16);
  if (bf16f(t) < v) ++t;
  return t;
}

// Q4G64 (reading Q28): per stored row vector and group of 64 entries, lo_b = bf16 round
// down of the minimum, s_b = bf16 round up of fp32((max - lo_b) / 15) (1.0 if 0), code =
// clamp(rint(fp32(fp32(x - lo_b) / s_b)), 0, 15) — fp32, this order, no contraction (the file is
// compiled with -ffp-contract=off), so codes equal the oracle's bit for bit.
static void quantize_group(const float* x, uint8_t* codes /*32 bytes*/, uint32_t* param) {
  float lo = x[0], hi = x[0];
  for (int k = 1; k < 64; ++k) {
    lo = std::min(lo, x[k]);
    hi = std::max(hi, x[k]);
  }
  const uint16_t lob = bf16_down(lo);
  const float lof = bf16f(lob);
  const float t = (hi - lof) / 15.0f;
  uint16_t sb = bf16_up(t);
  if (sb == 0) sb = 0x3F80;
  const float sf = bf16f(sb);
  for (int k = 0; k < 64; k += 2) {
    float q0 = std::nearbyint((x[k] - lof) / sf), q1 = std::nearbyint((x[k + 1] - lof) / sf);
    q0 = std::min(15.0f, std::max(0.0f, q0));
    q1 = std::min(15.0f, std::max(0.0f, q1));
    codes[k / 2] = (uint8_t)((int)q0 | ((int)q1 << 4));
  }
  *param = (uint32_t)sb | ((uint32_t)lob << 16);
}

static void pack_rows_q4(uint8_t* dst, const uint16_t* gate, const uint16_t* up, const uint16_t* down, int d, int I,
                         int r0, int I_full, uint64_t rb) {
  const int ng = d / 64;
#pragma omp parallel for schedule(static)
  for (int r = 0; r < I; ++r) {
    uint8_t* row = dst + (uint64_t)r * rb;
    memset(row, 0, rb);
    std::vector<float> x(d);
    for (int part = 0; part < 3; ++part) {
      for (int k = 0; k < d; ++k)
        x[k] = bf16f(part == 0 ? gate[(size_t)(r0 + r) * d + k]
                     : part == 1 ? up[(size_t)(r0 + r) * d + k] : down[(size_t)k * I_full + r0 + r]);
      for (int g = 0; g < ng; ++g) {
        uint32_t prm;
        quantize_group(&x[(size_t)g * 64], row + (size_t)part * (d / 2) + (size_t)g * 32, &prm);
        memcpy(row + 3ull * (d / 2) + ((size_t)part * ng + g) * 4, &prm, 4);
      }
    }
  }
}

static void pack_rows(const moepic_model_desc& d, uint8_t* dst, const uint16_t* gate, const uint16_t* up,
                      const uint16_t* down, int I_full) {
  if (d.weight_format == MOEPIC_Q4G64)
    pack_rows_q4(dst, gate, up, down, d.d, d.I, d.tp_rank * d.I, I_full, row_bytes_of(d));
  else
    pack_rows_bf16(dst, gate, up, down, d.d, d.I, d.tp_rank * d.I, I_full);
}

moepic_status moepic_load_expert(moepic_ctx* ctx, int32_t layer, int32_t expert, const uint16_t* gate,
                                 const uint16_t* up, const uint16_t* down) {
  CTX_GUARD();
  const auto& d = ctx->desc;
  if (!gate || !up || !down) return fail(&ctx->err, MOEPIC_EINVAL, "weight pointer is NULL");
  if (d.weight_format == MOEPIC_BF16 && !down_fits_f16(down, (size_t)d.d * ctx->I_full))
    return fail(&ctx->err, MOEPIC_EINVAL, "down weight outside the fp16 range of the stored row (|x| >= 65536)");
  if (expert >= 0) {
    if (expert >= d.N) return fail(&ctx->err, MOEPIC_EINVAL, "expert out of range");
    if (layer < 0 || layer >= d.L_host) return fail(&ctx->err, MOEPIC_EINVAL, "layer must be < L_host");
    if (!ctx->cp->is_local(expert)) return MOEPIC_OK;   // another EP rank owns it
    pack_rows(d, const_cast<uint8_t*>(ctx->host_expert(layer, expert)), gate, up, down, ctx->I_full);
    return MOEPIC_OK;
  }
  const int s = -1 - expert;
  if (s >= d.n_shared) return fail(&ctx->err, MOEPIC_EINVAL, "shared expert index out of range");
  if (layer < 0 || layer >= d.L) return fail(&ctx->err, MOEPIC_EINVAL, "layer out of range");
  std::vector<uint8_t> tmp((size_t)d.I * ctx->rb());
  pack_rows(d, tmp.data(), gate, up, down, ctx->I_full);
  CK(cudaMemcpy(ctx->shared_ptr(layer, s), tmp.data(), tmp.size(), cudaMemcpyHostToDevice));
  return MOEPIC_OK;
}

moepic_status moepic_pack_expert(const moepic_model_desc* desc, const uint16_t* gate, const uint16_t* up,
                                 const uint16_t* down, void* out, size_t* bytes) {
  if (!bytes || !validate_desc(desc).empty()) return MOEPIC_EINVAL;
  const moepic_model_desc l = local_desc(*desc);
  const size_t need = (size_t)l.I * row_bytes_of(l);
  if (!out) {
    *bytes = need;
    return MOEPIC_OK;
  }
  if (*bytes < need || !gate || !up || !down) return MOEPIC_EINVAL;
  if (l.weight_format == MOEPIC_BF16 && !down_fits_f16(down, (size_t)l.d * desc->I)) return MOEPIC_EINVAL;
  pack_rows(l, static_cast<uint8_t*>(out), gate, up, down, desc->I);
  *bytes = need;
  return MOEPIC_OK;
}

moepic_status moepic_configure(moepic_ctx* ctx, const moepic_cache_config* cfg, moepic_config_out* out) {
  CTX_GUARD();
  if (!cfg) return fail(&ctx->err, MOEPIC_EINVAL, "cfg is NULL");
  if (cfg->v_e > ctx->desc.v_e_max + 1e-9) return fail(&ctx->err, MOEPIC_EINVAL, "v_e exceeds v_e_max");
  CK(cudaDeviceSynchronize());        // "when the device is idle"
  std::string e = ctx->cp->configure(to_params(cfg, ctx->desc.L), ctx->lay.pool_rows);
  if (!e.empty()) return fail(&ctx->err, MOEPIC_EINVAL, "%s", e.c_str());
  // re-layout: per-layer slot regions, tops of cached experts H2D
  // (poison: on the copy stream, ordered before the top copies -- a legacy-stream cudaMemset is
  // not ordered against the non-blocking copy stream and could land after them)
  if (ctx->poison) CK(cudaMemsetAsync(ctx->arena + ctx->lay.pool, 0xFF, ctx->lay.pool_rows * ctx->rb(), ctx->copy));
  uint64_t off = 0;
  const uint64_t rb = ctx->rb();
  for (int i = 0; i < ctx->desc.L; ++i) {
    const LayerState& l = ctx->cp->layers[i];
    ctx->slot_base[i] = off;
    if (!l.cache_on()) continue;
    off += (uint64_t)l.C * l.I_top * rb;
  }
  for (int i = 0; i < ctx->desc.L; ++i) {
    const LayerState& l = ctx->cp->layers[i];
    if (!l.cache_on()) continue;
    for (int s = 0; s < (int)l.slot_expert.size(); ++s) {
      const int ex = l.slot_expert[s];
      if (ex < 0) continue;
      CK(cudaMemcpyAsync(ctx->slot_ptr(i, s), ctx->host_expert(i, ex), (size_t)l.I_top * rb,
                         cudaMemcpyHostToDevice, ctx->copy));
      ctx->ctr.h2d_copies++;
    }
  }
  CK(cudaStreamSynchronize(ctx->copy));
  ctx->pending = Plan();
  ctx->feed_drop();
  ctx->cancel_prefetch = cfg->cancel_prefetch != 0;
  ctx->configured = true;
  write_config_out(*ctx->cp, out);
  return MOEPIC_OK;
}

// Build K2 launches + combine segments for one group of segments.
struct StepSeg {
  const uint8_t* base;
  int32_t expert, nrows;
  uint32_t mask;    // decode: tokens served (bit b = token b)
  int32_t row0;     // first intermediate index of the segment inside its expert
};

struct FuseCombine {
  float* y;
  int residual;
  bool done;
};

// K2T launches over a segment group (kernels/expert_tc.cu): every weight row is read once for the
// whole batch; each launch leaves one [G][B][d] partial that K3 adds in its fixed order.
static moepic_status launch_group_tc(moepic_ctx* ctx, const std::vector<StepSeg>& segs, const uint16_t* h, int B,
                                     cudaStream_t s, int64_t& ws_next, std::vector<CombineSeg>& comb,
                                     int& launches) {
  const int d = ctx->desc.d;
  const uint8_t* rbase = ctx->arena + ctx->lay.shared;
  K2TParams& kp = *ctx->ktp;
  if (!pf_tmap_2d(&kp.tmH, h, (uint64_t)B, (uint64_t)d, kK2TMaxB))
    return ctx->poisoned = true, fail(&ctx->err, MOEPIC_ERUNTIME, "cuTensorMapEncodeTiled failed (h)");
  std::vector<const StepSeg*> work;
  for (const auto& sg : segs)
    if (sg.nrows > 0 && sg.mask != 0) work.push_back(&sg);
  for (size_t i0 = 0; i0 < work.size(); i0 += kMaxLaunchSegs) {
    const size_t i1 = std::min(work.size(), i0 + (size_t)kMaxLaunchSegs);
    int units = 0;
    uint64_t rows = 0;
    for (size_t i = i0; i < i1; ++i) {
      K2TSeg& g = kp.segs[i - i0];
      g.map_row = (int64_t)((uint64_t)(work[i]->base - rbase) / ctx->rb());
      g.unit_begin = units;
      g.expert = work[i]->expert;
      g.tok_mask = work[i]->mask;
      g.pad = 0;
      units += work[i]->nrows / 64;
      rows += (uint64_t)work[i]->nrows;
    }
    const int G = std::min(kSMs, units);
    if ((uint64_t)(ws_next + (int64_t)G * B * d) > ctx->lay.ws_floats)
      return ctx->poisoned = true, fail(&ctx->err, MOEPIC_ERUNTIME, "workspace overflow (%lld floats)", (long long)ws_next);
    kp.tmW = &ctx->tm_rows;
    kp.ids = reinterpret_cast<const int32_t*>(ctx->arena + ctx->lay.ids);
    kp.w = reinterpret_cast<const float*>(ctx->arena + ctx->lay.w);
    kp.ws = reinterpret_cast<float*>(ctx->arena + ctx->lay.ws) + ws_next;
    kp.d = d;
    kp.K = ctx->desc.K;
    kp.B = B;
    kp.nsegs = (int)(i1 - i0);
    kp.units = units;
    kp.mode = ctx->k2t_mode;
    comb.push_back(CombineSeg{ws_next, G, (uint32_t)((1ull << B) - 1)});
    ws_next += (int64_t)G * B * d;
    const int pe = ctx->prof_begin(s, MOEPIC_KERNEL_EXPERT);
    kp.tstamp = ctx->tl_slot(3) ? ctx->tl_slot(3) : ctx->tstamp(pe);
    static unsigned long long* dbg_buf = nullptr;   // MOEPIC_K2_TRACE: per-CTA phases to stderr (tools)
    kp.dbg = nullptr;
    if (ctx->k2_trace) {
      if (!dbg_buf) cudaMalloc(&dbg_buf, 148 * 8 * 8);
      cudaMemsetAsync(dbg_buf, 0, 148 * 8 * 8, s);
      kp.dbg = dbg_buf;
    }
    launch_k2t(kp, G, s);
    if (ctx->k2_trace) {
      unsigned long long hb[148 * 8];
      cudaStreamSynchronize(s);
      cudaMemcpy(hb, dbg_buf, sizeof hb, cudaMemcpyDeviceToHost);
      unsigned long long t0 = ~0ull, mx[4] = {0, 0, 0, 0}, mn[4] = {~0ull, ~0ull, ~0ull, ~0ull};
      double avg[4] = {0, 0, 0, 0};
      for (int c = 0; c < G; ++c) t0 = std::min(t0, hb[c * 8]);
      for (int c = 0; c < G; ++c) {
        for (int k = 0; k < 4; ++k) {
          const unsigned long long v = hb[c * 8 + k] - t0;
          mx[k] = std::max(mx[k], v);
          mn[k] = std::min(mn[k], v);
          avg[k] += (double)(k == 2 ? hb[c * 8 + 6] & ((1ull << 40) - 1) : hb[c * 8 + 4 + k]) / G;
        }
      }
      fprintf(stderr, "[k2ttrace] G=%d units=%d rows=%llu start %llu..%llu mma_done %llu..%llu flush %llu..%llu "
              "end %llu..%llu ns | avg wait cycles: producer-empty %.0f mma-full %.0f mma-issue %.0f epi-gu %.0f\n",
              G, units, (unsigned long long)rows, mn[0], mx[0], mn[1], mx[1], mn[2], mx[2], mn[3], mx[3], avg[0],
              avg[1], avg[2], avg[3]);
    }
    ctx->prof_end(pe, s, rows * ctx->rb() + (uint64_t)B * d * 2);   // each weight row once
    CK(cudaGetLastError());
    ++launches;
  }
  return MOEPIC_OK;
}

// Gated launch (K2Gate): segs[0, n_a) are ready at launch, segs[n_a, ...) are the tail of the
// step's last on-demand copy, streamed by the same launch once the copy stream's flag arrives.
constexpr size_t kGateOff = 32;   // the copy-stream gate word inside the arena's ticket block
constexpr uint64_t kGateMinBytes = 256ull << 20;   // gate steps whose K2 rows reach this size
constexpr double kGateLaunchS = 3e-6;   // K2 ramp (the launch latency is left out: a tail that
                                         // outlasts K2 stalls the gate, measured)

struct K2Gate {
  size_t n_a;
  const unsigned int* flag;
  unsigned int val;
  unsigned int* stall;   // per-CTA wait record (device alias of mapped host memory) or nullptr
};

// Can one gated K2 launch (with the fused combine) cover these segments?  Needs the CUDA-core K2
// (every expert within K2's token block, so no K2T) and one parameter block.
static bool k2_gate_feasible(const moepic_ctx* ctx, size_t nsegs, int B) {
  const int tbmax = k2_max_tokens(ctx->desc.d, ctx->desc.weight_format == MOEPIC_Q4G64);
  return ctx->k2_gate && B <= tbmax && nsegs <= (size_t)kMaxLaunchSegs;
}

static moepic_status launch_group(moepic_ctx* ctx, const std::vector<StepSeg>& segs, const uint16_t* h, int B,
                                  cudaStream_t s, int64_t& ws_next, std::vector<CombineSeg>& comb, int& launches,
                                  FuseCombine* fuse = nullptr, const K2Gate* gate = nullptr) {
  const int d = ctx->desc.d;
  const int tbmax = k2_max_tokens(d, ctx->desc.weight_format == MOEPIC_Q4G64);
  if (gate && (B > tbmax || !fuse))
    return fail(&ctx->err, MOEPIC_ERUNTIME, "internal: gated K2 launch outside K2's token block");
  if (!gate && ctx->k2t && B <= kK2TMaxB) {   // an expert with more tokens than K2's block: K2T reads it once
    bool hot = false, ok = true;
    const uint8_t* rbase = ctx->arena + ctx->lay.shared;
    for (const auto& sg : segs) {
      if (sg.nrows <= 0 || sg.mask == 0) continue;
      hot |= __builtin_popcount(sg.mask) > tbmax;
      ok &= sg.nrows % 64 == 0 && sg.base >= rbase && (uint64_t)(sg.base - rbase) % ctx->rb() == 0;
    }
    if (hot && ok) return launch_group_tc(ctx, segs, h, B, s, ws_next, comb, launches);
  }
  // split by token groups of <= tbmax tokens
  std::vector<StepSeg> work;
  size_t work_a = 0;   // gated: work items [0, work_a) are phase 0
  for (size_t si = 0; si < segs.size(); ++si) {
    const auto& sg = segs[si];
    if (gate && si == gate->n_a) work_a = work.size();
    if (sg.nrows <= 0 || sg.mask == 0) continue;
    uint32_t m = sg.mask;
    while (m) {
      uint32_t part = 0;
      for (int t = 0; t < tbmax && m; ++t) {
        uint32_t low = m & (~m + 1u);
        part |= low;
        m &= m - 1u;
      }
      StepSeg x = sg;
      x.mask = part;
      work.push_back(x);
    }
  }
  if (gate && gate->n_a >= segs.size()) work_a = work.size();
  if (gate && (work.size() > (size_t)kMaxLaunchSegs || comb.size() + work.size() > (size_t)kMaxLaunchSegs))
    return fail(&ctx->err, MOEPIC_ERUNTIME, "internal: gated K2 launch over more than one parameter block");
  size_t i0 = 0;
  K2Params& kp = *ctx->kp;
  while (i0 < work.size()) {
    const size_t i1 = std::min(work.size(), i0 + (size_t)kMaxLaunchSegs);
    int64_t R = 0, RA = 0;
    int maxtok = 1;
    for (size_t i = i0; i < i1; ++i) {
      R += work[i].nrows;
      if (!gate || i < work_a) RA += work[i].nrows;
      maxtok = std::max(maxtok, __builtin_popcount(work[i].mask));
    }
    const int64_t RB = R - RA;
    // phase 0 rows over the first GA CTAs, gated rows over the first GB (no CTA range is empty
    // inside a phase, so every CTA between a segment's first and last owner writes a partial)
    const int64_t G = std::min<int64_t>(kSMs, std::max(RA, RB));
    const int64_t GA = std::min(G, RA), GB = std::min(G, RB);
    kp.rows_a = RA;
    kp.ga = (int)GA;
    kp.gb = (int)GB;
    kp.gate = gate ? gate->flag : nullptr;
    kp.gate_val = gate ? gate->val : 0u;
    kp.stall = gate ? gate->stall : nullptr;
    kp.h = h;
    kp.ids = reinterpret_cast<const int32_t*>(ctx->arena + ctx->lay.ids);
    kp.w = reinterpret_cast<const float*>(ctx->arena + ctx->lay.w);
    kp.ws = reinterpret_cast<float*>(ctx->arena + ctx->lay.ws);
    kp.total_rows = R;
    kp.d = d;
    kp.q4 = ctx->desc.weight_format == MOEPIC_Q4G64;
    kp.K = ctx->desc.K;
    kp.nsegs = (int)(i1 - i0);
    int64_t rb = 0;
    for (size_t i = i0; i < i1; ++i) {
      Seg& g = kp.segs[i - i0];
      g.base = work[i].base;
      g.expert = work[i].expert;
      g.nrows = work[i].nrows;
      g.tok_mask = work[i].mask;
      g.row_begin = (int32_t)rb;
      // CTA owning the first / last row of the segment within its phase: largest c with
      // c*Rp/Gp <= row
      const bool ph1 = rb >= RA;
      const int64_t Rp = ph1 ? RB : RA, Gp = ph1 ? GB : GA, off = ph1 ? RA : 0;
      const int64_t first = rb - off, last = rb - off + work[i].nrows - 1;
      int64_t cf = (first * Gp) / Rp;
      while (cf + 1 < Gp && k2_row_lo(cf + 1, Rp, Gp) <= first) ++cf;
      while (k2_row_lo(cf, Rp, Gp) > first) --cf;
      int64_t cl = (last * Gp) / Rp;
      while (cl + 1 < Gp && k2_row_lo(cl + 1, Rp, Gp) <= last) ++cl;
      while (k2_row_lo(cl, Rp, Gp) > last) --cl;
      g.cta_first = (int32_t)cf;
      const int ntok = __builtin_popcount(work[i].mask);
      const int nchunks = (int)(cl - cf + 1);
      g.ws_off = ws_next;
      comb.push_back(CombineSeg{ws_next, nchunks, work[i].mask});
      ws_next += (int64_t)nchunks * ntok * d;
      rb += work[i].nrows;
    }
    if ((uint64_t)ws_next > ctx->lay.ws_floats)
      return fail(&ctx->err, MOEPIC_ERUNTIME, "workspace overflow (%lld floats)", (long long)ws_next);
    int tb = 1;
    while (tb < maxtok) tb <<= 1;
    // algorithmic bytes: each segment's rows once -- a segment split into token
    // groups streams its rows once per group, but only the first group counts -- plus activations
    uint64_t alg_bytes = 0;
    for (size_t i = i0; i < i1; ++i) {
      if (i == 0 || work[i].base != work[i - 1].base || work[i].nrows != work[i - 1].nrows)
        alg_bytes += (uint64_t)work[i].nrows * ctx->rb();
      alg_bytes += (uint64_t)__builtin_popcount(work[i].mask) * d * 2;
    }
    // the last launch of the step's last group also combines (grid barrier, no K3 launch)
    kp.combine = 0;
    if (fuse && i1 == work.size() && comb.size() <= (size_t)kMaxLaunchSegs) {
      kp.combine = 1;
      kp.B = B;
      kp.residual = fuse->residual;
      kp.y = fuse->y;
      kp.ncomb = (int)comb.size();
      for (size_t i = 0; i < comb.size(); ++i) kp.comb[i] = comb[i];
      // flattened offsets fit next to the reduction area and the segment table in the K2 ring
      uint64_t noff = 0;
      for (const auto& c : comb) noff += (uint64_t)c.nchunks * __builtin_popcount(c.tok_mask);
      const uint64_t need = 16ull * 32 * 16 + comb.size() * sizeof(CombineSeg) + 36 * 4 + noff * 4;
      kp.flat = need <= (uint64_t)k2_smem_bytes(d, kp.q4) ? 1 : 0;
      kp.bar = reinterpret_cast<unsigned long long*>(ctx->arena + ctx->lay.ticket + 8);
      ctx->bar_base += (uint64_t)G;
      kp.bar_target = ctx->bar_base;
      fuse->done = true;
    }
    const int pe = ctx->prof_begin(s, MOEPIC_KERNEL_EXPERT);
    kp.tstamp = ctx->tl_slot(kp.combine ? 1 : 3) ? ctx->tl_slot(kp.combine ? 1 : 3) : ctx->tstamp(pe);
    kp.dbg = nullptr;
    static unsigned long long* dbg_buf = nullptr;   // MOEPIC_K2_TRACE: phase spans to stderr (tools)
    const bool trace = ctx->k2_trace;
    if (trace) {
      if (!dbg_buf) cudaMalloc(&dbg_buf, 148 * 8 * 8);
      cudaMemsetAsync(dbg_buf, 0, 148 * 8 * 8, s);
      kp.dbg = dbg_buf;
    }
    launch_k2(kp, (int)G, tb, s);
    if (trace) {
      unsigned long long h[148 * 8];
      cudaStreamSynchronize(s);
      cudaMemcpy(h, dbg_buf, sizeof h, cudaMemcpyDeviceToHost);
      unsigned long long t0 = ~0ull, mx[8] = {0, 0, 0, 0, 0, 0, 0, 0}, mn[8];
      for (auto& v : mn) v = ~0ull;
      for (int c = 0; c < G; ++c) t0 = std::min(t0, h[c * 8]);
      for (int c = 0; c < G; ++c)
        for (int k = 0; k < 8; ++k)
          if (h[c * 8 + k]) {
            mx[k] = std::max(mx[k], h[c * 8 + k] - t0);
            mn[k] = std::min(mn[k], h[c * 8 + k] - t0);
          }
      fprintf(stderr, "[k2trace] G=%lld rows=%lld comb=%d start %llu..%llu first_tile %llu..%llu stream_done %llu..%llu "
              "barrier %llu..%llu end %llu..%llu ns | combine: walk-total %llu..%llu loads %llu..%llu reduce %llu..%llu\n",
              (long long)G, (long long)R, kp.combine, mn[0], mx[0], mn[1], mx[1], mn[2], mx[2], mn[3], mx[3], mn[4],
              mx[4], mn[5], mx[5], mn[6], mx[6], mn[7], mx[7]);
    }
    ctx->prof_end(pe, s, alg_bytes);
    CK(cudaGetLastError());
    ++launches;
    i0 = i1;
  }
  return MOEPIC_OK;
}

// Spin until the n tagged mailbox words starting at word index w0 all carry ctx->seq (each
// 64-bit word is written atomically by the router kernel: (seq << 32) | payload), pumping the
// prefetch feed meanwhile.  No system fence is involved on either side.
static moepic_status wait_mailbox(moepic_ctx* ctx, cudaStream_t s, size_t w0, size_t n) {
  volatile const uint64_t* words = reinterpret_cast<volatile const uint64_t*>(ctx->mailbox + 64) + w0;
  const uint64_t want = ctx->seq;
  auto t0 = std::chrono::steady_clock::now();
  uint64_t spins = 0;
  size_t ok = 0;   // words [0, ok) already verified
  for (;;) {
    while (ok < n && (words[ok] >> 32) == want) ++ok;
    if (ok == n) break;
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
    if ((spins & 0x3F) == 0 && !ctx->feed_pump(ctx->kFeedDepth)) {
      ctx->poisoned = true;
      return fail(&ctx->err, MOEPIC_ERUNTIME, "prefetch feed: %s", cudaGetErrorString(cudaGetLastError()));
    }
    if ((++spins & 0xFFF) == 0) {
      cudaError_t q = cudaStreamQuery(s);
      if (q != cudaSuccess && q != cudaErrorNotReady) {
        ctx->poisoned = true;
        return fail(&ctx->err, MOEPIC_ERUNTIME, "router kernel failed: %s", cudaGetErrorString(q));
      }
      if (q == cudaSuccess) {   // kernel done: every word must be there now
        std::atomic_thread_fence(std::memory_order_acquire);
        while (ok < n && (words[ok] >> 32) == want) ++ok;
        if (ok != n) {
          ctx->poisoned = true;
          return fail(&ctx->err, MOEPIC_ERUNTIME, "router mailbox not published");
        }
        break;
      }
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(60)) {
        ctx->poisoned = true;
        return fail(&ctx->err, MOEPIC_ERUNTIME, "router mailbox timeout");
      }
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  return MOEPIC_OK;
}

static moepic_status read_ranking(moepic_ctx* ctx, cudaStream_t s);

// MOEPIC_FAULT_AT_STEP: a trapping kernel on the caller's stream, then the stream is synchronised
// so the sticky launch failure surfaces here as it would from any real kernel fault
static moepic_status inject_fault(moepic_ctx* ctx, cudaStream_t s) {
  launch_trap(s);
  CK(cudaStreamSynchronize(s));
  return fail(&ctx->err, MOEPIC_ERUNTIME, "injected fault did not fail");
}

static moepic_status run_router(moepic_ctx* ctx, const uint16_t* h, int B, int layer_route, int layer_pred,
                                cudaStream_t s, bool read_ids, bool read_rank) {
  const auto& d = ctx->desc;
  RouterParams rp{};
  rp.h = h;
  rp.W0 = layer_route >= 0 ? ctx->router(layer_route) : nullptr;
  rp.W1 = layer_pred >= 0 ? ctx->router(layer_pred) : nullptr;
  rp.logits = reinterpret_cast<double*>(ctx->arena + ctx->lay.logits);
  rp.ids = reinterpret_cast<int32_t*>(ctx->arena + ctx->lay.ids);
  rp.w = reinterpret_cast<float*>(ctx->arena + ctx->lay.w);
  rp.ranking = reinterpret_cast<int32_t*>(ctx->arena + ctx->lay.ranking);
  rp.ticket = reinterpret_cast<unsigned int*>(ctx->arena + ctx->lay.ticket);
  rp.ticket2 = reinterpret_cast<unsigned int*>(ctx->arena + ctx->lay.ticket + 16);
  rp.sel_cnt = reinterpret_cast<int32_t*>(ctx->arena + ctx->lay.rsel);
  rp.sel_max = reinterpret_cast<unsigned long long*>(ctx->arena + ctx->lay.rsel + (size_t)d.N * 8);
  uint8_t* mb = ctx->mailbox_dev;
  const size_t BK = (size_t)d.max_batch * d.K;
  rp.mb_ids = reinterpret_cast<unsigned long long*>(mb + 64);
  rp.mb_w = rp.mb_ids + BK;
  rp.mb_rank = rp.mb_w + BK;
  rp.seq = ++ctx->seq;
  rp.B = B; rp.d = d.d; rp.N = d.N; rp.K = d.K; rp.renorm = d.renorm_topk;
  const int pe = ctx->prof_begin(s, MOEPIC_KERNEL_ROUTER);
  rp.tstamp = ctx->tl_slot(0) ? ctx->tl_slot(0) : ctx->tstamp(pe);
  rp.dbg = nullptr;
  if (ctx->k1_trace) {   // phase stamps per launch (tools): ring of 4096 x 8 u64
    if (!ctx->k1dbg) {
      cudaMalloc(&ctx->k1dbg, 4096 * 64);
      cudaMemset(ctx->k1dbg, 0, 4096 * 64);
    }
    rp.dbg = ctx->k1dbg + (ctx->k1dbg_n % 4096) * 8;
    cudaMemsetAsync(rp.dbg, 0xFF, 8, s);
    cudaMemsetAsync(rp.dbg + 1, 0, 56, s);
    ctx->k1dbg_n++;
  }
  launch_router(rp, s, ctx->pdl && read_ids && !ctx->k1_trace);
  ctx->prof_end(pe, s, (uint64_t)((rp.W0 ? 1 : 0) + (rp.W1 ? 1 : 0)) * d.N * d.d * 2 + (uint64_t)B * d.d * 2);
  CK(cudaGetLastError());
  ctx->ctr.kernel_launches += B > kRouterSplitB ? 2 : 1;
  if (read_ids) {
    const size_t n = (size_t)B * d.K;
    moepic_status st = wait_mailbox(ctx, s, 0, n);
    if (st == MOEPIC_OK) st = wait_mailbox(ctx, s, BK, n);
    if (st != MOEPIC_OK) return st;
    const uint64_t* words = reinterpret_cast<const uint64_t*>(ctx->mailbox + 64);
    for (size_t i = 0; i < n; ++i) {
      ctx->ids_h[i] = (int32_t)(uint32_t)words[i];
      const uint32_t wb = (uint32_t)words[BK + i];
      memcpy(&ctx->w_h[i], &wb, 4);
    }
  }
  if (read_rank) return read_ranking(ctx, s);
  return MOEPIC_OK;
}

// The next-layer ranking is published after the routing; the step plans its prefetch only at
// the end, so the host waits for it late (usually already there).
static moepic_status read_ranking(moepic_ctx* ctx, cudaStream_t s) {
  const auto& d = ctx->desc;
  const size_t off = 2 * (size_t)d.max_batch * d.K;
  moepic_status st = wait_mailbox(ctx, s, off, (size_t)d.N);
  if (st != MOEPIC_OK) return st;
  const uint64_t* words = reinterpret_cast<const uint64_t*>(ctx->mailbox + 64) + off;
  for (int i = 0; i < d.N; ++i) ctx->rank_h[i] = (int32_t)(uint32_t)words[i];
  return MOEPIC_OK;
}

// Issue the plan's H2D copies into ping-pong half `buf`.
// Queue the plan's H2D copies (into ping-pong half `buf`) on the feed; a few chunks are issued
// now, the rest while the host waits for the next routing (or all of them when cancel is off).
static moepic_status issue_plan(moepic_ctx* ctx, Plan& plan, int buf) {
  plan.buf = buf;
  ctx->feed_drop();
  if (ctx->ev_step_rec[buf]) CK(cudaStreamWaitEvent(ctx->copy, ctx->ev_step[buf], 0));
  const int j = plan.target;
  const LayerState& l = ctx->cp->layers[j];
  const uint64_t rb = ctx->rb();
  ctx->feed_cancel.assign(plan.items.size(), 0);
  for (size_t k = 0; k < plan.items.size(); ++k) {
    const PlanItem& it = plan.items[k];
    const uint8_t* src = ctx->host_expert(j, it.expert) + (it.full ? 0 : (uint64_t)l.I_top * rb);
    uint8_t* dst = ctx->plan_ptr(buf, it.buf_row);
    const size_t total = (size_t)it.rows * rb;
    for (size_t off = 0; off < total; off += ctx->kFeedChunk)
      ctx->feed.push_back({dst + off, src + off, std::min(ctx->kFeedChunk, total - off), (int32_t)k});
  }
  ctx->ctr.pcie_prefetch_planned_bytes += plan_bytes(plan, (int64_t)rb);
  if (!ctx->feed_pump(ctx->cancel_prefetch ? ctx->kFeedDepth : (size_t)-1)) {
    ctx->poisoned = true;
    return fail(&ctx->err, MOEPIC_ERUNTIME, "prefetch copy: %s", cudaGetErrorString(cudaGetLastError()));
  }
  return MOEPIC_OK;
}

// Routing of the plan's target layer is known: drop the unissued chunks of experts it did not
// activate, issue everything else, and mark the point the plan's segments wait for.
static moepic_status finish_plan(moepic_ctx* ctx, const Plan& plan, const StepResult& res) {
  const auto f0 = std::chrono::steady_clock::now();
  if (ctx->cancel_prefetch) {
    std::vector<char> act(ctx->desc.N, 0);
    for (int e : res.A) act[e] = 1;
    for (size_t k = 0; k < plan.items.size(); ++k)
      if (!act[plan.items[k].expert]) ctx->feed_cancel[k] = 1;
  }
  const auto f1 = std::chrono::steady_clock::now();
  const size_t issued0 = ctx->feed_next;
  const uint64_t copies0 = ctx->ctr.h2d_copies;
  const size_t infl0 = ctx->feed_inflight.size();
  int act_items = 0;
  for (size_t k = 0; k < plan.items.size(); ++k) act_items += ctx->feed_cancel.empty() || !ctx->feed_cancel[k];
  if (!ctx->feed_pump((size_t)-1)) {
    ctx->poisoned = true;
    return fail(&ctx->err, MOEPIC_ERUNTIME, "prefetch copy: %s", cudaGetErrorString(cudaGetLastError()));
  }
  const auto f2 = std::chrono::steady_clock::now();
  const size_t issued = ctx->feed_next - issued0;
  ctx->feed_drop();
  if (!plan.items.empty()) CK(cudaEventRecord(ctx->ev_plan[plan.buf], ctx->copy));   // gB waits on it
  if (ctx->host_timing) {
    auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
    ctx->hf[0] += us(f0, f1);
    ctx->hf[1] += us(f1, f2);
    ctx->hf[2] += us(f2, std::chrono::steady_clock::now());
    ctx->hf[3] += (double)issued;
    ctx->hf[4] += (double)plan.items.size();
    ctx->hf[5] += (double)(ctx->ctr.h2d_copies - copies0);
    ctx->hf[6] += (double)infl0;
    ctx->hf[7] += (double)act_items;
    ctx->hf[8] += (double)ctx->feed.size();
    ctx->hf_n++;
  }
  return MOEPIC_OK;
}

// Prefill batch (B > 32): tokens are permuted into per-expert blocks (padded to 128 rows), every
// segment group runs the tcgen05 gate/up GEMM (SwiGLU epilogue into A_act) and the down GEMM
// (accumulating into Y), then each token gathers its K rows.  Groups: resident tops + shared
// experts first (no wait), then prefetched segments (plan event), then on-demand ones (copy
// event), so the resident work overlaps the PCIe loads.
static moepic_status prefill_launch(moepic_ctx* ctx, const uint16_t* h, int T, float* y, cudaStream_t s,
                                    uint32_t flags, const std::vector<StepSeg>& gA,
                                    const std::vector<StepSeg>& gB, const std::vector<StepSeg>& gC, int buf,
                                    int& launches) {
  const auto& d = ctx->desc;
  const int N = d.N, K = d.K, NS = d.n_shared, NE = N + NS;
  const int lo_e = d.ep_rank * ctx->Nl(), hi_e = lo_e + ctx->Nl();
  const bool q4 = d.weight_format == MOEPIC_Q4G64;
  std::vector<int32_t> cnt(NE, 0), moff(NE, 0);
  for (int i = 0; i < T * K; ++i) {
    const int e = ctx->ids_h[i];
    if (e >= lo_e && e < hi_e) cnt[e]++;
  }
  for (int s2 = 0; s2 < NS; ++s2) cnt[N + s2] = T;
  int64_t rows = 0;
  std::vector<PfExpert> table(NE);
  for (int e = 0; e < NE; ++e) {
    moff[e] = (int32_t)rows;
    const int mt = (cnt[e] + kPfBM - 1) / kPfBM;
    table[e] = PfExpert{(int32_t)rows, cnt[e], mt, 0, 0, {0, 0, 0}};
    rows += (int64_t)mt * kPfBM;
  }
  if ((uint64_t)rows + kPfBM > ctx->lay.pf_rows) return fail(&ctx->err, MOEPIC_ERUNTIME, "prefill row overflow");
  uint16_t* xperm = reinterpret_cast<uint16_t*>(ctx->arena + ctx->lay.xperm);
  uint16_t* aact = reinterpret_cast<uint16_t*>(ctx->arena + ctx->lay.aact);   // fp16 a (reading Q31)
  float* Y = reinterpret_cast<float*>(ctx->arena + ctx->lay.yperm);
  int32_t* pos = reinterpret_cast<int32_t*>(ctx->arena + ctx->lay.pos);
  int32_t* cursor = reinterpret_cast<int32_t*>(ctx->arena + ctx->lay.cursor);

  // ---- permute (+ zero the accumulated outputs)
  CK(cudaMemsetAsync(cursor, 0, (size_t)N * 4, s));
  CK(cudaMemsetAsync(Y, 0, (size_t)rows * d.d * 4, s));
  PfPermuteParams& pp = *ctx->pf_pp;
  pp.h = h; pp.ids = reinterpret_cast<const int32_t*>(ctx->arena + ctx->lay.ids); pp.cursor = cursor;
  pp.pos = pos; pp.xperm = xperm; pp.T = T; pp.K = K; pp.d = d.d; pp.e_lo = lo_e; pp.e_hi = hi_e;
  pp.n_shared = NS;
  pp.f16 = q4 ? 1 : 0;
  for (int s2 = 0; s2 < NS; ++s2) pp.shared_off[s2] = moff[N + s2];
  for (int e = 0; e < N; ++e) pp.m_off[e] = moff[e];
  launch_pf_permute(pp, s);
  CK(cudaGetLastError());
  ++launches;

  PfGemmParams& gp = *ctx->pf_gp;
  CUtensorMap tm_x, tm_act;
  if (!pf_tmap_2d(&tm_x, xperm, (uint64_t)rows + kPfBM, d.d, kPfBM) ||
      !pf_tmap_2d(&tm_act, aact, (uint64_t)rows + kPfBM, d.I, kPfBM))
    return fail(&ctx->err, MOEPIC_ERUNTIME, "cuTensorMapEncodeTiled failed (activations)");
  auto tidx = [&](int expert) { return expert >= 0 ? expert : N + (-1 - expert); };
  // gate/up runs on CTA pairs (UMMA M = 256: half the B operand bytes per SM; ncu: tensor pipe
  // 88% vs 75% for single CTAs) unless rounding the experts' 128-row tiles up to pairs would
  // waste more than 1/10 of the MMA work (few tokens per expert, e.g. Qwen3-shaped prefill).
  int64_t mt1 = 0, mt2 = 0;
  for (int e = 0; e < NE; ++e) {
    mt1 += table[e].mtiles;
    mt2 += 2 * ((table[e].mtiles + 1) / 2);
  }
  const int CGu = ctx->pf_cta_pair >= 0 ? (ctx->pf_cta_pair ? 2 : 1) : (mt2 * 10 <= mt1 * 11 ? 2 : 1);
  // down follows the same choice since its activation is one fp16 operand (reading Q31): with the
  // bf16 hi / lo pair a single CTA's B tile fed two MMAs and pairs did not pay (90 % vs 84 %)
  const int CGd = ctx->pf_cta_pair >= 0 ? (ctx->pf_cta_pair ? 2 : 1) : CGu;
  auto ptiles = [&](int e, int CG) { return (int64_t)((table[e].mtiles + CG - 1) / CG); };

  auto run_group = [&](const std::vector<StepSeg>& g0) -> moepic_status {
    for (const auto& sg : g0)
      if (sg.nrows % kPfBK != 0 || (reinterpret_cast<uintptr_t>(sg.base) & 15))
        return fail(&ctx->err, MOEPIC_ERUNTIME, "prefill segment rows must be a multiple of 64");
    // Q4G64 (reading Q32): dequantise the group's segments once into fp16 rows; the GEMMs read those
    std::vector<StepSeg> gq;
    if (q4) {
      gq = g0;
      uint16_t* wdq = reinterpret_cast<uint16_t*>(ctx->arena + ctx->lay.wdq);
      PfDequantParams& dq = *ctx->pf_dq;
      int64_t next = 0;
      for (size_t i0 = 0; i0 < gq.size(); i0 += kPfMaxSegs) {
        const size_t i1 = std::min(gq.size(), i0 + (size_t)kPfMaxSegs);
        dq.nseg = (int)(i1 - i0);
        dq.d = d.d;
        dq.src_row_bytes = (int)ctx->rb();
        int rows_l = 0;
        for (size_t i = i0; i < i1; ++i) {
          if ((uint64_t)(next + gq[i].nrows) > ctx->lay.wdq_rows)
            return ctx->poisoned = true, fail(&ctx->err, MOEPIC_ERUNTIME, "dequant scratch overflow");
          uint16_t* dst = wdq + (size_t)next * 3 * d.d;
          dq.seg[i - i0] = PfDequantSeg{gq[i].base, dst, gq[i].nrows, rows_l};
          gq[i].base = reinterpret_cast<const uint8_t*>(dst);
          rows_l += gq[i].nrows;
          next += gq[i].nrows;
        }
        dq.total_rows = rows_l;
        const int pe = ctx->prof_begin(s, MOEPIC_KERNEL_EXPERT);
        launch_pf_dequant(dq, s);
        ctx->prof_end(pe, s, (uint64_t)rows_l * (ctx->rb() + 6ull * d.d));
        CK(cudaGetLastError());
        ++launches;
      }
    }
    const std::vector<StepSeg>& g = q4 ? gq : g0;
    // gate/up: chunks of <= kPfMaxSegs segments
    for (size_t i0 = 0; i0 < g.size(); i0 += kPfMaxSegs) {
      const size_t i1 = std::min(g.size(), i0 + (size_t)kPfMaxSegs);
      gp.tmA = tm_x;
      gp.nseg = (int)(i1 - i0);
      gp.nexp = NE;
      for (int e = 0; e < NE; ++e) gp.ex[e] = table[e];
      int64_t tiles = 0;
      double flops = 0;
      for (size_t i = i0; i < i1; ++i) {
        const StepSeg& sg = g[i];
        const int e = tidx(sg.expert);
        gp.seg[i - i0] = PfSeg{e, sg.row0, sg.nrows, 0};
        if (!pf_tmap_weights(&gp.tmB[i - i0], sg.base, (uint64_t)sg.nrows, d.d, kPfBN1))
          return fail(&ctx->err, MOEPIC_ERUNTIME, "cuTensorMapEncodeTiled failed (weights)");
        tiles += ptiles(e, CGu) * ((sg.nrows + kPfBN1 - 1) / kPfBN1);
        flops += 2.0 * 2.0 * cnt[e] * (double)d.d * sg.nrows;
      }
      gp.ntiles = (int32_t)tiles;
      gp.cta_pair = CGu == 2;
      gp.d = d.d; gp.I = d.I; gp.out = aact; gp.ld_out = d.I; gp.accumulate = 0; gp.f16 = q4 ? 1 : 0;
      const int pe = ctx->prof_begin(s, MOEPIC_KERNEL_GEMM);
      launch_pf_gateup(gp, s);
      ctx->prof_end(pe, s, (uint64_t)flops);
      CK(cudaGetLastError());
      ++launches;
    }
    // down: experts' segments are consecutive in g; chunk by whole experts
    size_t i0 = 0;
    while (i0 < g.size()) {
      size_t i1 = i0;
      while (i1 < g.size()) {
        size_t j = i1;
        while (j < g.size() && g[j].expert == g[i1].expert) ++j;
        if (j - i0 > (size_t)kPfMaxSegs && i1 > i0) break;
        i1 = j;
      }
      gp.tmA = tm_act;
      gp.nseg = (int)(i1 - i0);
      gp.nexp = NE;
      for (int e = 0; e < NE; ++e) {
        gp.ex[e] = table[e];
        gp.ex[e].mtiles = 0;
      }
      double flops = 0;
      for (size_t i = i0; i < i1; ++i) {
        const StepSeg& sg = g[i];
        const int e = tidx(sg.expert);
        const int li = (int)(i - i0);
        gp.seg[li] = PfSeg{e, sg.row0, sg.nrows, 0};
        if (!pf_tmap_weights(&gp.tmB[li], sg.base, (uint64_t)sg.nrows, d.d, kPfBK))
          return fail(&ctx->err, MOEPIC_ERUNTIME, "cuTensorMapEncodeTiled failed (weights)");
        if (gp.ex[e].mtiles == 0) {
          gp.ex[e].mtiles = table[e].mtiles;
          gp.ex[e].seg_begin = li;
        }
        gp.ex[e].seg_end = li + 1;
        flops += 2.0 * cnt[e] * (double)d.d * sg.nrows;
      }
      int64_t tiles = 0;
      for (int e = 0; e < NE; ++e) tiles += (gp.ex[e].mtiles ? ptiles(e, CGd) : 0) * (d.d / kPfBN2);
      gp.ntiles = (int32_t)tiles;
      gp.cta_pair = CGd == 2;
      gp.d = d.d; gp.I = d.I; gp.out = Y; gp.ld_out = d.d; gp.accumulate = 1; gp.f16 = 0;
      const int pe = ctx->prof_begin(s, MOEPIC_KERNEL_GEMM);
      launch_pf_down(gp, s);
      ctx->prof_end(pe, s, (uint64_t)flops);
      CK(cudaGetLastError());
      ++launches;
      i0 = i1;
    }
    return MOEPIC_OK;
  };
  // resident tops and prefetched rows as ONE group once the plan has landed (it was issued a layer
  // earlier, behind that layer's on-demand copies): two GEMM launches fewer per layer, and the
  // resident GEMMs still run while this layer's on-demand copies stream.  An expert's segments
  // stay consecutive, top first (the down GEMM groups by expert).
  moepic_status st;
  if (!gB.empty() && ctx->pf_merge_ab) {
    std::vector<StepSeg> gAB(gA);
    gAB.insert(gAB.end(), gB.begin(), gB.end());
    std::stable_sort(gAB.begin(), gAB.end(), [](const StepSeg& x, const StepSeg& y) {
      return x.expert != y.expert ? x.expert < y.expert : x.row0 < y.row0;
    });
    CK(cudaStreamWaitEvent(s, ctx->ev_plan[buf], 0));
    if ((st = run_group(gAB)) != MOEPIC_OK) return st;
  } else {
    if ((st = run_group(gA)) != MOEPIC_OK) return st;
    if (!gB.empty()) {
      CK(cudaStreamWaitEvent(s, ctx->ev_plan[buf], 0));
      if ((st = run_group(gB)) != MOEPIC_OK) return st;
    }
  }
  if (!gC.empty()) {
    CK(cudaStreamWaitEvent(s, ctx->ev_od, 0));
    if ((st = run_group(gC)) != MOEPIC_OK) return st;
  }
  PfCombineParams cp2{};
  cp2.y = y; cp2.h = h; cp2.Y = Y; cp2.pos = pos;
  cp2.w = reinterpret_cast<const float*>(ctx->arena + ctx->lay.w);
  cp2.T = T; cp2.K = K; cp2.d = d.d; cp2.n_shared = NS;
  cp2.residual = adds_residual(d, flags) ? 1 : 0;
  for (int s2 = 0; s2 < NS; ++s2) cp2.shared_off[s2] = moff[N + s2];
  const int pe = ctx->prof_begin(s, MOEPIC_KERNEL_COMBINE);
  launch_pf_combine(cp2, s);
  ctx->prof_end(pe, s, (uint64_t)T * K * d.d * 4 + (uint64_t)T * d.d * 4);
  CK(cudaGetLastError());
  ++launches;
  return MOEPIC_OK;
}

// cp_ids != nullptr (token-sharded EP): the routing is already known -- ctx->ids_h holds the
// computed sub-batch's ids (B tokens) and cp_ids / cp_B the whole batch the control plane sees.
static moepic_status layer_forward_impl(moepic_ctx* ctx, int32_t layer, const void* h_dev, int32_t B, float* y_dev,
                                        void* stream, uint32_t flags, moepic_trace* tr,
                                        const int32_t* cp_ids = nullptr, int cp_B = 0) {
  const auto& d = ctx->desc;
  if (!ctx->configured) return fail(&ctx->err, MOEPIC_EINVAL, "moepic_configure has not been called");
  if (layer < 0 || layer >= d.L) return fail(&ctx->err, MOEPIC_EINVAL, "layer out of range");
  if (B < 1 || B > d.max_batch) return fail(&ctx->err, MOEPIC_EINVAL, "B must be in [1, max_batch]");
  if (!h_dev || !y_dev) return fail(&ctx->err, MOEPIC_EINVAL, "h_dev / y_dev is NULL");
  if ((reinterpret_cast<uintptr_t>(h_dev) & 15) || (reinterpret_cast<uintptr_t>(y_dev) & 15))
    return fail(&ctx->err, MOEPIC_EINVAL, "h_dev and y_dev must be 16-byte aligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint16_t* h = static_cast<const uint16_t*>(h_dev);
  const bool predict = (flags & MOEPIC_FUSE_PREDICT) != 0;
  const int j = (layer + 1) % d.L;
  ControlPlane& cp = *ctx->cp;
  const LayerState& l = cp.layers[layer];
  const uint64_t rb = ctx->rb();
  int launches = 0;

  Plan used;
  const bool have_plan = ctx->pending.valid && ctx->pending.target == layer;
  if (have_plan) used = std::move(ctx->pending);
  else ctx->feed_drop();   // a plan for another layer is abandoned
  ctx->pending = Plan();
  const int buf = have_plan ? used.buf : (ctx->last_buf ^ 1);

  // ---- K1 (router + fused next-layer predictor) and the mailbox handoff
  const auto t_call = std::chrono::steady_clock::now();
  ctx->tl_rec = -1;
  if (ctx->tl_dev && B <= kDecodeMaxB && ctx->tl_seen++ >= ctx->tl_skip &&
      (int)ctx->tl_host.size() < moepic_ctx::kTlMax) {
    ctx->tl_rec = (int)ctx->tl_host.size();
    ctx->tl_host.push_back(moepic_ctx::TlHost{layer, {0, 0, 0, 0, 0}, 0});
  }
  moepic_status st = MOEPIC_OK;
  const bool route_here = cp_ids == nullptr;
  if (route_here) {
    st = run_router(ctx, h, B, layer, predict ? j : -1, s, true, false);
    ++launches;
    cp_ids = ctx->ids_h.data();
    cp_B = B;
  }
  const auto t_routed = std::chrono::steady_clock::now();
  auto t_first_copy = t_routed;   // MOEPIC_HOST_TIMING / MOEPIC_TIMELINE
  if (st != MOEPIC_OK) return st;

  // ---- control plane (classification, counters, admission)
  // ---- control plane: classification first; the beta bottoms it decides are issued on
  // the copy stream before the rest of the step (statistics, counters, admissions) is computed,
  // so the link starts streaming this layer's missing rows as early as possible
  StepResult res;
  const Plan* up = have_plan ? &used : nullptr;
  cp.classify(layer, cp_ids, cp_B, up, res);
  const auto t_cls = std::chrono::steady_clock::now();
  if (have_plan) {
    st = finish_plan(ctx, used, res);
    if (st != MOEPIC_OK) return st;
  }
  const auto t_fin = std::chrono::steady_clock::now();

  // token masks per activated expert
  const int K = d.K;
  auto mask_of = [&](int e) {
    uint32_t m = 0;
    if (B > kDecodeMaxB) return m;      // prefill segments carry no token masks
    for (int b = 0; b < B; ++b)
      for (int k = 0; k < K; ++k)
        if (ctx->ids_h[b * K + k] == e) m |= 1u << b;
    return m;
  };

  // ---- segment groups: resident now (A), prefetched (B, plan event), on-demand (C, copy event)
  std::vector<StepSeg> gA, gB, gC;
  int64_t od_row = 0;
  int n_od = 0;
  bool waited = false;
  // The step's last on-demand copy is split into head + tail (decode): which copy is last is
  // known from the classification alone (pass 1: beta / gamma bottoms, pass 2: gamma tops), so
  // that copy is issued as head, ev_od_head, tail right away -- nothing is held back, and the
  // K2 launch over everything but the tail runs while the tail is in flight.
  int n_copies = 0;
  for (size_t a = 0; a < res.A.size(); ++a) {
    const int c = res.cls[a];
    if (res.plan_idx[a] >= 0) {   // a window-cut prefix (Q30): the rest loads on demand
      if (c == kBeta || c == kGamma) ++n_copies;
      continue;
    }
    if (c == kBeta || (c == kGamma && l.I_top < d.I)) ++n_copies;
    if (c == kGamma && l.I_top > 0) ++n_copies;
  }
  // gated tail (one K2 launch per step, the last copy's tail streamed after the copy-stream flag)
  const bool q4 = d.weight_format == MOEPIC_Q4G64;
  // gated only where the step's K2 work is large (Mixtral-shaped layers, ~700 MB): there the
  // single launch matches the split's throughput and cuts the event-timed launch overhead; on
  // 75-140 MB layers (Qwen3 / DeepSeek shapes) it measured ~2 % slower than the split
  // (DESIGN.md §6b), so they keep the two launches unless MOEPIC_K2_GATE=2
  int64_t step_rows_all = (int64_t)res.A.size() * d.I + (int64_t)d.n_shared * (shared_hi(cp) - shared_lo(cp));
  const bool gate_mode = ctx->k2_gate && B <= k2_max_tokens(d.d, q4) &&
                         (ctx->k2_gate_force || (uint64_t)step_rows_all * rb >= kGateMinBytes);
  const bool split_ok = B <= kDecodeMaxB && ctx->od_tail_bytes > 0;
  int64_t tail_rows_split = split_ok ? (int64_t)((ctx->od_tail_bytes + rb - 1) / rb) : 0;
  if (gate_mode && ctx->stall_prev >= 0) {   // the previous gated launch has finished: its waits
    const unsigned int* rec = ctx->stall_h + (size_t)ctx->stall_prev * kStallSlot;
    double mean = 0.0;   // over the CTAs that stream gated rows
    for (int c = 0; c < ctx->stall_prev_g; ++c) mean += rec[c];
    mean = ctx->stall_prev_g ? mean / ctx->stall_prev_g * 1e-3 : 0.0;   // us
    ctx->gate_wait_us_sum += mean;
    ++ctx->gate_steps;
    if (ctx->gate_adapt) {
      if (mean > ctx->gate_wait_hi_us) ctx->gate_ctrl *= 0.92;
      else if (mean < ctx->gate_wait_lo_us) ctx->gate_ctrl *= 1.03;
      ctx->gate_ctrl = std::min(8.0, std::max(0.25, ctx->gate_ctrl));
    }
    ctx->stall_prev = -1;
  }
  if (split_ok && gate_mode && ctx->od_tail_auto) {
    // the tail lands while K2 streams the step's other rows: the link stays busy under K2 and the
    // gated rows are streamed as they land.  Tail = k2_gate_frac x (K2 time of the step's rows +
    // ~3 us ramp) at the link rate (K2 ~6 TB/s on bf16 rows, ~1.6 TB/s dequantising
    // Q4G64; link ~55 GB/s, both measured); below 1 so that the gate itself rarely waits
    const int64_t step_rows = step_rows_all;
    const double k2_s = (double)step_rows * rb / (q4 ? 1.6e12 : 6.0e12) + kGateLaunchS;
    tail_rows_split = std::max<int64_t>(1, (int64_t)(ctx->k2_gate_frac * ctx->gate_ctrl * k2_s * 55e9 / rb));
  }
  // a copy is split only when it is well above the tail (split_x x tail): every extra DMA costs
  // ~4 us of link time (scripts/dma_probe.cu), a somewhat long whole-copy tail only a short wait
  // at the gate
  const int64_t split_min_rows = (gate_mode && ctx->od_tail_auto ? ctx->tail_split_x : 2) * tail_rows_split;
  const uint8_t* split_dst = nullptr;   // segment whose tail was split off
  bool split_whole = false;             // ... or which is the tail as a whole (ev_od_head before it)
  // Two copy streams (MOEPIC_COPY_STREAMS=2; default 1): the step's on-demand copies alternate
  // between them, so one DMA engine's per-copy start-up overlaps the other's transfer (many
  // 2-10 MB bottoms per layer on Qwen3 / DeepSeek: MOEPIC_TIMELINE measured ~40 us per layer from
  // the first cudaMemcpyAsync to the link running at rate with one stream).  The step's last copy
  // always goes to ctx->copy, which first waits for the other stream, so ev_od / ev_od_head keep
  // their meaning and the prefetch feed (ctx->copy) still follows every on-demand byte.  Measured
  // neutral (Qwen3 32.48 vs 32.52, DeepSeek 46.34 vs 46.50 tokens/s): the start-up is not per copy.
  bool used2 = false;
  auto join2 = [&]() -> moepic_status {   // ctx->copy waits for everything issued on copy2 so far
    if (!used2) return MOEPIC_OK;
    CK(cudaEventRecord(ctx->ev_copy2, ctx->copy2));
    CK(cudaStreamWaitEvent(ctx->copy, ctx->ev_copy2, 0));
    used2 = false;
    return MOEPIC_OK;
  };
  auto copy = [&](uint8_t* dst, const uint8_t* src, int32_t rows, bool evicted = false) -> moepic_status {
    const size_t bytes = (size_t)rows * rb;
    const auto tw0 = std::chrono::steady_clock::now();
    if (!waited) {   // the buffers / slots written here were last read by earlier steps
      for (int b2 = 0; b2 < 2; ++b2)
        if (ctx->ev_step_rec[b2]) {
          CK(cudaStreamWaitEvent(ctx->copy, ctx->ev_step[b2], 0));
          if (ctx->copy2) CK(cudaStreamWaitEvent(ctx->copy2, ctx->ev_step[b2], 0));
        }
      waited = true;
    }
    const auto tw1 = std::chrono::steady_clock::now();
    const bool last = n_od == n_copies - 1;
    if (n_od == 0 && ctx->tl_slot(4)) launch_stamp(ctx->tl_slot(4), ctx->copy);   // MOEPIC_TIMELINE
    cudaStream_t cs = ctx->copy;
    if (ctx->copy2 && !last && (n_od & 1)) {
      cs = ctx->copy2;
      used2 = true;
    }
    if (evicted && ctx->poison) CK(cudaMemsetAsync(dst, 0xFF, bytes, cs));   // the victim's old top
    if (cs != ctx->copy) {
      CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, cs));
      ctx->ctr.h2d_copies++;
    } else if (split_ok && last && (int64_t)rows > split_min_rows) {
      moepic_status st2 = join2();
      if (st2 != MOEPIC_OK) return st2;
      const size_t head = bytes - (size_t)tail_rows_split * rb;
      CK(cudaMemcpyAsync(dst, src, head, cudaMemcpyHostToDevice, ctx->copy));
      CK(cudaEventRecord(ctx->ev_od_head, ctx->copy));
      CK(cudaMemcpyAsync(dst + head, src + head, bytes - head, cudaMemcpyHostToDevice, ctx->copy));
      ctx->ctr.h2d_copies += 2;
      split_dst = dst;
    } else if (split_ok && ctx->od_split_boundary && last && (n_copies >= 2 || gate_mode)) {
      // a small last copy is the tail as a whole: the K2 launch over everything else waits for
      // the copies before it, so only the last copy's rows remain after the link goes quiet
      moepic_status st2 = join2();
      if (st2 != MOEPIC_OK) return st2;
      CK(cudaEventRecord(ctx->ev_od_head, ctx->copy));
      CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->copy));
      ctx->ctr.h2d_copies++;
      split_dst = dst;
      split_whole = true;
    } else {
      CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->copy));
      ctx->ctr.h2d_copies++;
    }
    if (ctx->host_timing) {
      ctx->hc[0] += std::chrono::duration<double, std::micro>(tw1 - tw0).count();
      ctx->hc[1] += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - tw1).count();
      ctx->hc_n++;
    }
    if (n_od++ == 0 && (ctx->host_timing || ctx->tl_rec >= 0)) t_first_copy = std::chrono::steady_clock::now();
    return MOEPIC_OK;
  };
  const uint32_t all_tok = B >= 32 ? 0xFFFFFFFFu : ((1u << B) - 1u);
  {
    const int64_t lo = shared_lo(cp), hi = shared_hi(cp);
    for (int s2 = 0; s2 < d.n_shared; ++s2)
      if (hi > lo) gA.push_back(StepSeg{ctx->shared_ptr(layer, s2) + lo * rb, -1 - s2, (int32_t)(hi - lo), all_tok, (int32_t)lo});
  }
  std::vector<uint32_t> masks(res.A.size());
  std::vector<uint8_t*> od_rest(d.N, nullptr);   // gamma with a prefetched prefix: where row `prefix` lands
  for (size_t a = 0; a < res.A.size(); ++a) {   // pass 1: everything classification decides
    const int e = res.A[a];
    const uint32_t m = masks[a] = mask_of(e);
    const int c = res.cls[a];
    const int pj = res.plan_idx[a];
    const bool top_cached_before = (c != kGamma) && !(pj >= 0 && used.items[pj].full);
    if (top_cached_before && l.I_top > 0) gA.push_back(StepSeg{ctx->slot_ptr(layer, l.slot_of[e]), e, l.I_top, m, 0});
    if (pj >= 0) {
      const PlanItem& it = used.items[pj];
      gB.push_back(StepSeg{ctx->plan_ptr(buf, it.buf_row), e, it.rows, m, it.full ? 0 : l.I_top});
      if (c == kBeta || c == kGamma) {   // window-cut prefix (Q30): the rest of the rows on demand
        const int r0 = (it.full ? 0 : l.I_top) + it.rows, rows = d.I - r0;
        if (c == kGamma) od_rest[e] = ctx->od_ptr(buf, od_row);
        uint8_t* dst = ctx->od_ptr(buf, od_row);
        if ((uint64_t)(od_row + rows) > ctx->lay.od_rows) return ctx->poisoned = true, fail(&ctx->err, MOEPIC_ERUNTIME, "on-demand region overflow");
        if ((st = copy(dst, ctx->host_expert(layer, e) + (uint64_t)r0 * rb, rows)) != MOEPIC_OK) return st;
        gC.push_back(StepSeg{dst, e, rows, m, r0});
        od_row += rows;
      }
    } else if (c == kBeta || (c == kGamma && l.I_top < d.I)) {
      // missing bottom rows [I_top, I): known from classification alone (a gamma expert's top
      // rows follow in pass 2, once admission has chosen their destination)
      const int rows = d.I - l.I_top;
      uint8_t* dst = ctx->od_ptr(buf, od_row);
      if ((uint64_t)(od_row + rows) > ctx->lay.od_rows) return ctx->poisoned = true, fail(&ctx->err, MOEPIC_ERUNTIME, "on-demand region overflow");
      if ((st = copy(dst, ctx->host_expert(layer, e) + (uint64_t)l.I_top * rb, rows)) != MOEPIC_OK) return st;
      gC.push_back(StepSeg{dst, e, rows, m, l.I_top});
      od_row += rows;
    }
  }
  const auto t_p1 = std::chrono::steady_clock::now();
  cp.commit(layer, cp_ids, cp_B, up, res);
  ctx->committed = true;   // from here on, any failure leaves slots admitted with no landed rows
  const auto t_com = std::chrono::steady_clock::now();
  if (ctx->host_timing) {
    auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
    ctx->hp[0] += us(t_routed, t_cls);
    ctx->hp[1] += us(t_cls, t_fin);
    ctx->hp[2] += us(t_fin, t_p1);
    ctx->hp[3] += us(t_p1, t_com);
  }
  std::vector<int32_t> adm_slot(d.N, -2);   // expert -> slot for admitted, -1 if not admitted
  for (const auto& a : res.adm) adm_slot[a.expert] = a.victim == kAdmNone ? -1 : a.slot;
  for (size_t a = 0; a < res.A.size(); ++a) {   // pass 2: gamma tops -> the admitted slot (or the od region)
    if (res.cls[a] != kGamma || res.plan_idx[a] >= 0 || l.I_top == 0) continue;
    const int e = res.A[a];
    const int slot = adm_slot[e];
    uint8_t* top;
    if (slot >= 0) {
      top = ctx->slot_ptr(layer, slot);
    } else {
      if ((uint64_t)(od_row + l.I_top) > ctx->lay.od_rows) return ctx->poisoned = true, fail(&ctx->err, MOEPIC_ERUNTIME, "on-demand region overflow");
      top = ctx->od_ptr(buf, od_row);
      od_row += l.I_top;
    }
    if ((st = copy(top, ctx->host_expert(layer, e), l.I_top, slot >= 0)) != MOEPIC_OK) return st;
    gC.push_back(StepSeg{top, e, l.I_top, masks[a], 0});
  }
  // the split copy's segment is the last one pushed to gC: cut its tail into its own segment
  const uint8_t* tail_base = nullptr;
  if (split_dst) {
    StepSeg& last = gC.back();
    if (last.base != split_dst || n_od != n_copies)
      return fail(&ctx->err, MOEPIC_ERUNTIME, "internal: split copy is not the step's last on-demand segment");
    if (split_whole) {
      tail_base = split_dst;
    } else {
      StepSeg tail = last;
      last.nrows -= (int32_t)tail_rows_split;
      tail.base = split_dst + (size_t)last.nrows * rb;
      tail.nrows = (int32_t)tail_rows_split;
      tail.row0 = last.row0 + last.nrows;
      gC.push_back(tail);
      tail_base = tail.base;
    }
  }
  if ((st = join2()) != MOEPIC_OK) return st;
  if (n_od && ctx->tl_slot(2)) launch_stamp(ctx->tl_slot(2), ctx->copy);
  if (n_od) CK(cudaEventRecord(ctx->ev_od, ctx->copy));
  bool gated = false;          // the flag follows this step's last on-demand copy
  bool gate_consumed = false;  // ... and the single K2 launch streams the tail behind it
  if (tail_base && gate_mode && ctx->write_value32) {
    const CUdeviceptr flag = (CUdeviceptr)(ctx->arena + ctx->lay.ticket + kGateOff);
    if (ctx->write_value32((CUstream)ctx->copy, flag, (cuuint32_t)(ctx->gate_seq + 1), 0) != CUDA_SUCCESS)
      return ctx->poisoned = true, fail(&ctx->err, MOEPIC_ERUNTIME, "cuStreamWriteValue32 failed");
    ++ctx->gate_seq;
    gated = true;
  }
  {   // an expert's on-demand segments consecutive, tops first (the prefill down GEMM groups by expert)
    std::vector<int32_t> pos(d.N, 0);
    for (size_t a = 0; a < res.A.size(); ++a) pos[res.A[a]] = (int32_t)a;
    std::stable_sort(gC.begin(), gC.end(), [&](const StepSeg& x, const StepSeg& y) {
      const int px = x.expert >= 0 ? pos[x.expert] : -1, py = y.expert >= 0 ? pos[y.expert] : -1;
      return px != py ? px < py : x.row0 < y.row0;
    });
    if (tail_base)   // the split tail lands last: it goes last (its own K2 launch)
      std::stable_partition(gC.begin(), gC.end(), [&](const StepSeg& x) { return x.base != tail_base; });
  }
  const auto t_copies = std::chrono::steady_clock::now();

  if (B > kDecodeMaxB) {
    // ---- prefill: permute, tcgen05 GEMMs per segment group, combine
    st = prefill_launch(ctx, h, B, y_dev, s, flags, gA, gB, gC, buf, launches);
    if (st != MOEPIC_OK) return st;
  } else {
  // ---- K2 launches: resident now / prefetched / on-demand, then the combine
  int64_t ws_next = 0;
  std::vector<CombineSeg> comb;
  FuseCombine fuse{y_dev, adds_residual(d, flags) ? 1 : 0, false};
  if (tail_base) {
    // split last copy: ONE launch over the resident, prefetched and on-demand rows except the
    // tail once the head has landed (it runs while the tail is in flight), then the tail with
    // the fused combine -- the link idles only for the tail's K2, not for the whole on-demand set
    std::vector<StepSeg> first(gA);
    first.insert(first.end(), gB.begin(), gB.end());
    first.insert(first.end(), gC.begin(), gC.end() - 1);
    std::vector<StepSeg> tail(gC.end() - 1, gC.end());
    if (!gB.empty()) CK(cudaStreamWaitEvent(s, ctx->ev_plan[buf], 0));
    CK(cudaStreamWaitEvent(s, ctx->ev_od_head, 0));
    if (gated && tail[0].mask != 0 && k2_gate_feasible(ctx, first.size() + 1, B)) {
      // ONE launch: everything but the tail now, the tail behind the copy-stream flag
      unsigned int* srec = nullptr;
      if (ctx->stall_h) {   // this launch's wait record: zeroed, read back at the next gated step
        memset(ctx->stall_h + (size_t)ctx->stall_slot * kStallSlot, 0, kStallSlot * sizeof(unsigned int));
        srec = ctx->stall_d + (size_t)ctx->stall_slot * kStallSlot;
        ctx->stall_prev = ctx->stall_slot;
        ctx->stall_prev_g = (int)std::min<int64_t>(kSMs, tail[0].nrows);   // CTAs with gated rows (GB)
        ctx->stall_slot ^= 1;
      }
      const K2Gate gate{first.size(), reinterpret_cast<const unsigned int*>(ctx->arena + ctx->lay.ticket + kGateOff),
                        ctx->gate_seq, srec};
      std::vector<StepSeg> all(first);
      all.push_back(tail[0]);
      st = launch_group(ctx, all, h, B, s, ws_next, comb, launches, &fuse, &gate);
      if (st != MOEPIC_OK) return ctx->poisoned = true, st;
      gate_consumed = true;
    } else {
      st = launch_group(ctx, first, h, B, s, ws_next, comb, launches, nullptr);
      if (st != MOEPIC_OK) return st;
      CK(cudaStreamWaitEvent(s, ctx->ev_od, 0));
      st = launch_group(ctx, tail, h, B, s, ws_next, comb, launches, &fuse);
      if (st != MOEPIC_OK) return st;
    }
  } else {
  const bool lastA = gB.empty() && gC.empty(), lastB = gC.empty();
  st = launch_group(ctx, gA, h, B, s, ws_next, comb, launches, lastA ? &fuse : nullptr);
  if (st != MOEPIC_OK) return st;
  if (!gB.empty()) {
    CK(cudaStreamWaitEvent(s, ctx->ev_plan[buf], 0));
    st = launch_group(ctx, gB, h, B, s, ws_next, comb, launches, lastB ? &fuse : nullptr);
    if (st != MOEPIC_OK) return st;
  }
  if (!gC.empty()) {
    CK(cudaStreamWaitEvent(s, ctx->ev_od, 0));
    st = launch_group(ctx, gC, h, B, s, ws_next, comb, launches, &fuse);
    if (st != MOEPIC_OK) return st;
  }
  }
  if (!fuse.done) {   // no K2 launch fused the combine (no segments, or too many): run K3
  if (comb.size() > (size_t)kMaxStepSegs) return fail(&ctx->err, MOEPIC_ERUNTIME, "too many segments in one step");
  CombineParams& cpar = *ctx->cpar;
  cpar.y = y_dev;
  cpar.h = h;
  cpar.ws = reinterpret_cast<const float*>(ctx->arena + ctx->lay.ws);
  cpar.B = B;
  cpar.d = d.d;
  cpar.residual = adds_residual(d, flags) ? 1 : 0;   // h added once across ranks
  cpar.nsegs = (int)comb.size();
  for (size_t i = 0; i < comb.size(); ++i) cpar.segs[i] = comb[i];
  const int pe = ctx->prof_begin(s, MOEPIC_KERNEL_COMBINE);
  cpar.tstamp = ctx->tstamp(pe);
  launch_combine(cpar, s);
  {
    uint64_t cb = (uint64_t)B * d.d * 4;
    for (const auto& c : comb) cb += (uint64_t)c.nchunks * __builtin_popcount(c.tok_mask) * d.d * 4;
    ctx->prof_end(pe, s, cb);
  }
  CK(cudaGetLastError());
  ++launches;
  }
  }
  // admitted experts that arrived as full prefetches (or a prefix of one, Q30): D2D their top
  // rows -- from the plan buffer, and past the prefix from the on-demand region (after a gated
  // launch the compute stream has not waited for the copy event itself: it does here)
  bool od_synced = !gate_consumed;
  for (const auto& a : res.adm) {
    if (!a.d2d_from_plan || a.victim == kAdmNone || l.I_top == 0) continue;
    const int pj = [&] { for (size_t k = 0; k < used.items.size(); ++k) if (used.items[k].expert == a.expert) return (int)k; return -1; }();
    if (pj < 0) continue;
    const int pre = std::min(used.items[pj].rows, l.I_top);
    CK(cudaMemcpyAsync(ctx->slot_ptr(layer, a.slot), ctx->plan_ptr(buf, used.items[pj].buf_row),
                       (size_t)pre * rb, cudaMemcpyDeviceToDevice, s));
    if (pre < l.I_top) {
      if (!od_rest[a.expert]) return fail(&ctx->err, MOEPIC_ERUNTIME, "internal: prefix rest not on demand");
      if (!od_synced) CK(cudaStreamWaitEvent(s, ctx->ev_od, 0));
      od_synced = true;
      CK(cudaMemcpyAsync(ctx->slot_ptr(layer, a.slot) + (size_t)pre * rb, od_rest[a.expert],
                         (size_t)(l.I_top - pre) * rb, cudaMemcpyDeviceToDevice, s));
    }
  }
  if (ctx->poison) {   // this step's half and partials are dead once its kernels are done
    CK(cudaMemsetAsync(ctx->arena + ctx->lay.buf[buf], 0xFF, (ctx->lay.plan_rows + ctx->lay.od_rows) * rb, s));
    CK(cudaMemsetAsync(ctx->arena + ctx->lay.ws, 0xFF, ctx->lay.ws_floats * 4, s));
  }
  CK(cudaEventRecord(ctx->ev_step[buf], s));
  ctx->ev_step_rec[buf] = true;
  ctx->last_buf = buf;

  // ---- next-layer prefetch, issued after this layer's on-demand copies
  Plan next;
  if (predict) {
    st = read_ranking(ctx, s);
    if (st != MOEPIC_OK) return st;
    cp.make_plan(j, ctx->rank_h.data(), next);
    st = issue_plan(ctx, next, buf ^ 1);
    if (st != MOEPIC_OK) return st;
    ctx->pending = next;
  }

  if (ctx->tl_rec >= 0) {
    auto ns = [&](std::chrono::steady_clock::time_point t) {   // raw host ns: converted at the dump
      return (int64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(t.time_since_epoch()).count();
    };
    auto& hr = ctx->tl_host[ctx->tl_rec];
    hr.t[0] = ns(t_call);
    hr.t[1] = ns(t_routed);
    hr.t[2] = n_od ? ns(t_first_copy) : 0;
    hr.t[3] = ns(t_copies);
    hr.t[4] = ns(std::chrono::steady_clock::now());
    hr.od_bytes = res.pcie_ondemand;
  }
  if (ctx->host_timing) {   // MOEPIC_HOST_TIMING (tools): host-side phases of the call, us
    const auto t_end = std::chrono::steady_clock::now();
    auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
    ctx->ht[0] += us(t_call, t_routed);
    ctx->ht[1] += us(t_routed, n_od ? t_first_copy : t_copies);
    ctx->ht[2] += us(t_routed, t_copies);
    ctx->ht[3] += us(t_copies, t_end);
    ctx->ht_n++;
  }
  // ---- trace + counters
  const uint64_t pb = predict ? plan_bytes(next, (int64_t)rb) : 0;
  const uint64_t hbm = step_hbm_bytes(cp, res, B, predict ? 2 : 1, pb);
  if (tr) {
    for (int i = 0; i < B * K; ++i) {
      if (tr->ids) tr->ids[i] = ctx->ids_h[i];
      if (tr->w) tr->w[i] = ctx->w_h[i];
    }
    fill_step_trace(tr, res, predict ? &next : nullptr);
    tr->pcie_prefetch_bytes = pb;
    tr->hbm_bytes = hbm;
    tr->kernel_launches = launches;
  }
  ctx->ctr.layer_steps++;
  ctx->ctr.kernel_launches += launches - (route_here ? 1 : 0);   // run_router counts its own
  ctx->ctr.pcie_ondemand_bytes += res.pcie_ondemand;
  ctx->ctr.hbm_bytes += hbm;
  ctx->ctr.act_alpha += res.alpha;
  ctx->ctr.act_beta += res.beta;
  ctx->ctr.act_gamma += res.gamma;
  ctx->ctr.pred_hits += res.pred_hits;
  ctx->ctr.pred_total += res.A.size();
  return MOEPIC_OK;
}

// ====================================================================== multi-GPU group
#define NCK(call)                                                                          \
  do {                                                                                     \
    ncclResult_t r_ = (call);                                                              \
    if (r_ != ncclSuccess) {                                                               \
      ctx->poisoned = true;                                                                \
      return fail(&ctx->err, MOEPIC_ERUNTIME, "%s: %s", #call, nccl_api().GetErrorString(r_)); \
    }                                                                                      \
  } while (0)

static int group_size(const moepic_model_desc& d) { return d.ep_size > 1 ? d.ep_size : d.tp_size; }
static int group_rank(const moepic_model_desc& d) { return d.ep_size > 1 ? d.ep_rank : d.tp_rank; }

static inline int ep_grid(int64_t warps_of_work) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((warps_of_work + 7) / 8, 2 * kSMs));
}

// replicated-token group (decode EP / TP): y <- sum over ranks of the partial outputs
static moepic_status group_allreduce(moepic_ctx* ctx, float* y, int B, cudaStream_t s) {
  Group& g = *ctx->grp;
  const int n = B * ctx->desc.d;
  if (g.transport == MOEPIC_TRANSPORT_NCCL) {
    NCK(nccl_api().AllReduce(y, y, (size_t)n, ncclFloat32, ncclSum, g.comm, s));
    return MOEPIC_OK;
  }
  EpAllreduceParams p{};
  p.pr = g.pr; p.of = g.of; p.y = y; p.n = n; p.slot_floats = g.B_dec * ctx->desc.d;
  p.epoch = ++g.epoch[kEpPhReduce];
  launch_ep_allreduce(p, (int)std::min<int64_t>(32, std::max<int64_t>(1, (n / 4 + 255) / 256)), s);
  CK(cudaGetLastError());
  ctx->ctr.kernel_launches++;
  return MOEPIC_OK;
}

// token-sharded EP layer: route own tokens -> all-gather routing ->
// dispatch rows to the experts' ranks -> compute the sub-batch -> combine back -> reduce
static moepic_status sharded_forward(moepic_ctx* ctx, int32_t layer, const void* h_dev, int32_t Bl, float* y_dev,
                                     void* stream, uint32_t flags, moepic_trace* tr) {
  const auto& d = ctx->desc;
  Group& g = *ctx->grp;
  const int G = g.G, K = d.K, T = G * Bl;
  if (!ctx->configured) return fail(&ctx->err, MOEPIC_EINVAL, "moepic_configure has not been called");
  if (layer < 0 || layer >= d.L) return fail(&ctx->err, MOEPIC_EINVAL, "layer out of range");
  if (d.ep_size < 2) return fail(&ctx->err, MOEPIC_EINVAL, "MOEPIC_TOKENS_SHARDED needs an expert-parallel group");
  if (d.n_shared) return fail(&ctx->err, MOEPIC_EINVAL, "MOEPIC_TOKENS_SHARDED needs n_shared == 0");
  if (flags & MOEPIC_FUSE_PREDICT) return fail(&ctx->err, MOEPIC_EINVAL, "MOEPIC_TOKENS_SHARDED excludes FUSE_PREDICT");
  if (Bl < 1 || T > d.max_batch || Bl > g.Bl_max) return fail(&ctx->err, MOEPIC_EINVAL, "B must be in [1, max_batch / G]");
  if (!h_dev || !y_dev || (reinterpret_cast<uintptr_t>(h_dev) & 15) || (reinterpret_cast<uintptr_t>(y_dev) & 15))
    return fail(&ctx->err, MOEPIC_EINVAL, "h_dev / y_dev must be 16-byte aligned device pointers");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint16_t* h = static_cast<const uint16_t*>(h_dev);
  const bool nccl = g.transport == MOEPIC_TRANSPORT_NCCL;
  const NcclApi& nc = nccl_api();
  int32_t* ids_loc = reinterpret_cast<int32_t*>(ctx->arena + ctx->lay.ids);
  float* w_loc = reinterpret_cast<float*>(ctx->arena + ctx->lay.w);

  // ---- route my tokens, gather the batch's routing on every rank, publish it to the host
  moepic_status st = run_router(ctx, h, Bl, layer, -1, s, false, false);
  if (st != MOEPIC_OK) return st;
  const unsigned long long e_ids = ++g.epoch[kEpPhIds];
  const int half = (int)(e_ids & 1);
  if (nccl) {
    NCK(nc.GroupStart());
    NCK(nc.AllGather(ids_loc, g.region + g.of.ids_all[half], (size_t)Bl * K, ncclInt32, g.comm, s));
    NCK(nc.AllGather(w_loc, g.region + g.of.w_all[half], (size_t)Bl * K, ncclFloat32, g.comm, s));
    NCK(nc.GroupEnd());
  }
  EpIdsParams ip{};
  ip.pr = g.pr; ip.of = g.of; ip.ids = ids_loc; ip.w = w_loc; ip.BlK = Bl * K; ip.TK = T * K;
  ip.push = nccl ? 0 : 1; ip.epoch = e_ids;
  const size_t BK = (size_t)d.max_batch * K;
  ip.mb_ids = reinterpret_cast<unsigned long long*>(ctx->mailbox_dev + 64);
  ip.mb_w = ip.mb_ids + BK;
  ip.seq = ++ctx->seq;
  launch_ep_ids(ip, s);
  CK(cudaGetLastError());
  ctx->ctr.kernel_launches++;
  if ((st = wait_mailbox(ctx, s, 0, (size_t)T * K)) != MOEPIC_OK) return st;
  if ((st = wait_mailbox(ctx, s, BK, (size_t)T * K)) != MOEPIC_OK) return st;
  {
    const uint64_t* words = reinterpret_cast<const uint64_t*>(ctx->mailbox + 64);
    for (int i = 0; i < T * K; ++i) {
      g.ids_all[i] = (int32_t)(uint32_t)words[i];
      const uint32_t wb = (uint32_t)words[BK + i];
      memcpy(&g.w_all[i], &wb, 4);
    }
  }
  // ---- exchange lists (host, mapped memory; the previous layer's readers are done: this
  // layer's routing kernel ran after them on the same stream)
  EpLists& L = g.lists;
  if (!ep_plan(g.ids_all.data(), d.N, K, G, g.me, Bl, L))
    return fail(&ctx->err, MOEPIC_ERUNTIME, "routing produced an expert id out of range");
  const int n_disp = (int)L.d_tok.size(), n_sub = (int)L.sub.size();
  const size_t cap_d = (size_t)g.Bl_max * std::min(G, K), cap_s = (size_t)g.T_max;
  int32_t* I = g.idx_h;
  int32_t *dt = I, *dd = dt + cap_d, *dr = dd + cap_d, *sb = dr + cap_d, *cd = sb + cap_s, *cr = cd + cap_s,
          *ro = cr + cap_s, *rr = ro + g.Bl_max + 1;
  std::copy(L.d_tok.begin(), L.d_tok.end(), dt);
  std::copy(L.d_dst.begin(), L.d_dst.end(), dd);
  std::copy(L.d_row.begin(), L.d_row.end(), dr);
  std::copy(L.sub.begin(), L.sub.end(), sb);
  std::copy(L.c_dst.begin(), L.c_dst.end(), cd);
  std::copy(L.c_row.begin(), L.c_row.end(), cr);
  std::copy(L.r_off.begin(), L.r_off.end(), ro);
  std::copy(L.r_row.begin(), L.r_row.end(), rr);
  std::atomic_thread_fence(std::memory_order_release);
  auto dev = [&](int32_t* hp) { return g.idx_d + (hp - g.idx_h); };

  // ---- dispatch: my rows to the ranks owning their experts; the sub-batch routing to the arena
  const unsigned long long e_disp = ++g.epoch[kEpPhDispatch];
  const int hd = (int)(e_disp & 1);
  EpDispatchParams dp{};
  dp.pr = g.pr; dp.of = g.of; dp.h = h; dp.d = d.d; dp.K = K; dp.push = nccl ? 0 : 1;
  dp.n_disp = n_disp; dp.d_tok = dev(dt); dp.d_dst = dev(dd); dp.d_row = dev(dr);
  dp.sendbuf = reinterpret_cast<uint16_t*>(g.region + g.of.sendbuf);
  dp.n_sub = n_sub; dp.sub = dev(sb); dp.ids_out = ids_loc; dp.w_out = w_loc; dp.epoch = e_disp;
  launch_ep_dispatch(dp, ep_grid(std::max(n_disp, (n_sub * K + 31) / 32)), s);
  CK(cudaGetLastError());
  ctx->ctr.kernel_launches++;
  const uint16_t* hsub = reinterpret_cast<const uint16_t*>(g.region + g.of.recv[hd]);
  if (nccl) {
    NCK(nc.GroupStart());
    size_t soff = 0, roff = 0;
    for (int q = 0; q < G; ++q) {
      if (L.n_send[q]) NCK(nc.Send(dp.sendbuf + soff * d.d, (size_t)L.n_send[q] * d.d, ncclBfloat16, q, g.comm, s));
      if (L.n_recv[q])
        NCK(nc.Recv(g.region + g.of.recv[hd] + roff * d.d * 2, (size_t)L.n_recv[q] * d.d, ncclBfloat16, q, g.comm, s));
      soff += L.n_send[q];
      roff += L.n_recv[q];
    }
    NCK(nc.GroupEnd());
  } else {
    launch_ep_wait(g.pr, g.of, kEpPhDispatch, e_disp, s);
    CK(cudaGetLastError());
    ctx->ctr.kernel_launches++;
  }

  // ---- the sub-batch through the split-expert path (control plane sees all T tokens)
  float* ysub = reinterpret_cast<float*>(g.region + g.of.ysub);
  for (int i = 0; i < n_sub * K; ++i) ctx->ids_h[i] = g.ids_all[(size_t)L.sub[i / K] * K + i % K];
  if (n_sub > 0) {
    st = layer_forward_impl(ctx, layer, hsub, n_sub, ysub, stream, 0, tr, g.ids_all.data(), T);
    if (st != MOEPIC_OK) return st;
  } else {   // no token routes here: the control plane still sees the step (counters, stats)
    StepResult res;
    Plan used;
    const bool have_plan = ctx->pending.valid && ctx->pending.target == layer;
    if (have_plan) used = std::move(ctx->pending);
    ctx->pending = Plan();
    ctx->cp->step(layer, g.ids_all.data(), T, have_plan ? &used : nullptr, res);
    ctx->committed = true;
    fill_step_trace(tr, res, nullptr);
    ctx->ctr.layer_steps++;
  }

  // ---- combine: partial rows back to the token owners, owners reduce in rank order
  const unsigned long long e_comb = ++g.epoch[kEpPhCombine];
  const int hc = (int)(e_comb & 1);
  if (nccl) {
    NCK(nc.GroupStart());
    size_t soff = 0, roff = 0;
    for (int q = 0; q < G; ++q) {
      if (L.n_recv[q]) NCK(nc.Send(ysub + soff * d.d, (size_t)L.n_recv[q] * d.d, ncclFloat32, q, g.comm, s));
      if (L.n_send[q])
        NCK(nc.Recv(g.region + g.of.comb[hc] + roff * d.d * 4, (size_t)L.n_send[q] * d.d, ncclFloat32, q, g.comm, s));
      soff += L.n_recv[q];
      roff += L.n_send[q];
    }
    NCK(nc.GroupEnd());
  } else {
    EpCombineParams cpp{};
    cpp.pr = g.pr; cpp.of = g.of; cpp.ysub = ysub; cpp.d = d.d; cpp.n_sub = n_sub;
    cpp.c_dst = dev(cd); cpp.c_row = dev(cr); cpp.epoch = e_comb;
    launch_ep_combine(cpp, ep_grid(n_sub), s);
    CK(cudaGetLastError());
    ctx->ctr.kernel_launches++;
  }
  EpReduceParams rp{};
  rp.pr = g.pr; rp.of = g.of; rp.h = h; rp.y = y_dev; rp.d = d.d; rp.Bl = Bl;
  rp.residual = (flags & MOEPIC_RESIDUAL) ? 1 : 0; rp.wait = nccl ? 0 : 1;
  rp.r_off = dev(ro); rp.r_row = dev(rr); rp.epoch = e_comb;
  launch_ep_reduce(rp, (int)std::min<int64_t>(2 * kSMs, std::max<int64_t>(1, ((int64_t)Bl * d.d / 4 + 255) / 256)), s);
  CK(cudaGetLastError());
  ctx->ctr.kernel_launches++;
  if (tr) {   // the caller's own tokens
    for (int i = 0; i < Bl * K; ++i) {
      if (tr->ids) tr->ids[i] = g.ids_all[(size_t)g.me * Bl * K + i];
      if (tr->w) tr->w[i] = g.w_all[(size_t)g.me * Bl * K + i];
    }
  }
  return MOEPIC_OK;
}

moepic_status moepic_group_handle(moepic_ctx* ctx, int32_t transport, void* out, size_t* bytes) {
  CTX_GUARD();
  const auto& d = ctx->desc;
  if (!bytes) return fail(&ctx->err, MOEPIC_EINVAL, "bytes is NULL");
  if (!out) { *bytes = sizeof(GroupBlob); return MOEPIC_OK; }
  if (*bytes < sizeof(GroupBlob)) return fail(&ctx->err, MOEPIC_EINVAL, "handle buffer too small");
  const int G = group_size(d);
  if (G < 2 || G > kEpMaxRanks) return fail(&ctx->err, MOEPIC_EINVAL, "a group needs ep_size or tp_size in [2, 8]");
  if (transport != MOEPIC_TRANSPORT_PEER && transport != MOEPIC_TRANSPORT_NCCL)
    return fail(&ctx->err, MOEPIC_EINVAL, "unknown transport");
  if (transport == MOEPIC_TRANSPORT_NCCL && !nccl_api().ok)
    return fail(&ctx->err, MOEPIC_EINVAL, "libnccl.so.2 could not be loaded");
  if (ctx->grp && ctx->grp->joined) return fail(&ctx->err, MOEPIC_EINVAL, "already joined");
  if (!ctx->grp) {
    auto g = std::make_unique<Group>();
    g->G = G;
    g->me = group_rank(d);
    g->T_max = d.max_batch;
    g->Bl_max = (d.max_batch + G - 1) / G;
    g->B_dec = std::min(d.max_batch, kDecodeMaxB);
    g->of = ep_offsets(G, g->T_max, g->Bl_max, g->B_dec, d.K, d.d);
    if (cudaMalloc(&g->region, g->of.total) != cudaSuccess) {
      cudaGetLastError();
      return fail(&ctx->err, MOEPIC_ENOMEM, "exchange region (%zu bytes)", g->of.total);
    }
    CK(cudaMemset(g->region, 0, g->of.sig + 0 + (g->of.ctr - g->of.sig) + sizeof(unsigned int) * kEpPhases));
    g->idx_ints = 3 * (size_t)g->Bl_max * std::min(G, d.K) + 3 * (size_t)g->T_max + g->Bl_max + 1 +
                  (size_t)g->Bl_max * std::min(G, d.K) + 64;
    if (cudaHostAlloc(&g->idx_h, g->idx_ints * 4, cudaHostAllocMapped) != cudaSuccess) {
      cudaFree(g->region);
      return fail(&ctx->err, MOEPIC_ENOMEM, "index lists (mapped pinned)");
    }
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&g->idx_d), g->idx_h, 0));
    g->ids_all.assign((size_t)g->T_max * d.K, 0);
    g->w_all.assign((size_t)g->T_max * d.K, 0.f);
    g->pr.G = G;
    g->pr.me = g->me;
    g->pr.base[g->me] = g->region;
    if (transport == MOEPIC_TRANSPORT_NCCL && g->me == 0) NCK(nccl_api().GetUniqueId(&g->nccl_id));
    ctx->grp = std::move(g);
  }
  ctx->grp->transport = transport;
  GroupBlob b{};
  b.magic = kGroupMagic;
  b.rank = ctx->grp->me;
  b.world = G;
  b.transport = transport;
  b.kind = d.ep_size > 1 ? 0 : 1;
  b.region_bytes = ctx->grp->of.total;
  CK(cudaIpcGetMemHandle(&b.ipc, ctx->grp->region));
  b.nccl_id = ctx->grp->nccl_id;
  memcpy(out, &b, sizeof b);
  *bytes = sizeof b;
  return MOEPIC_OK;
}

moepic_status moepic_group_join(moepic_ctx* ctx, const void* handles, size_t bytes_each) {
  CTX_GUARD();
  if (!ctx->grp) return fail(&ctx->err, MOEPIC_EINVAL, "moepic_group_handle has not been called");
  Group& g = *ctx->grp;
  if (g.joined) return fail(&ctx->err, MOEPIC_EINVAL, "already joined");
  if (!handles || bytes_each != sizeof(GroupBlob)) return fail(&ctx->err, MOEPIC_EINVAL, "handle size mismatch");
  std::vector<GroupBlob> bl(g.G);
  for (int r = 0; r < g.G; ++r) {
    memcpy(&bl[r], static_cast<const uint8_t*>(handles) + (size_t)r * bytes_each, sizeof(GroupBlob));
    const GroupBlob& b = bl[r];
    if (b.magic != kGroupMagic || b.rank != r || b.world != g.G || b.transport != g.transport ||
        b.region_bytes != g.of.total || b.kind != (ctx->desc.ep_size > 1 ? 0 : 1))
      return fail(&ctx->err, MOEPIC_EINVAL, "handle %d does not match this group (rank, world, transport, shape)", r);
  }
  if (g.transport == MOEPIC_TRANSPORT_PEER) {
    for (int r = 0; r < g.G; ++r) {
      if (r == g.me) continue;
      void* p = nullptr;
      CK(cudaIpcOpenMemHandle(&p, bl[r].ipc, cudaIpcMemLazyEnablePeerAccess));
      g.pr.base[r] = static_cast<uint8_t*>(p);
      g.opened[r] = true;
    }
  } else {
    NCK(nccl_api().CommInitRank(&g.comm, g.G, bl[0].nccl_id, g.me));
    for (int r = 0; r < g.G; ++r) g.pr.base[r] = g.region;   // kernels only touch base[me]
  }
  CK(cudaDeviceSynchronize());
  g.joined = true;
  return MOEPIC_OK;
}

moepic_status moepic_ep_plan(int32_t N, int32_t K, int32_t G, int32_t me, int32_t Bl, const int32_t* ids_all,
                             int32_t* d_tok, int32_t* d_dst, int32_t* d_row, int32_t* n_disp,
                             int32_t* sub, int32_t* c_dst, int32_t* c_row, int32_t* n_sub,
                             int32_t* r_off, int32_t* r_row) {
  if (N < 2 || K < 1 || K >= N || G < 1 || G > kEpMaxRanks || N % G || me < 0 || me >= G || Bl < 1 || !ids_all)
    return MOEPIC_EINVAL;
  EpLists o;
  if (!ep_plan(ids_all, N, K, G, me, Bl, o)) return MOEPIC_EINVAL;
  auto put = [](int32_t* dst, const std::vector<int32_t>& v) { if (dst) std::copy(v.begin(), v.end(), dst); };
  put(d_tok, o.d_tok); put(d_dst, o.d_dst); put(d_row, o.d_row);
  put(sub, o.sub); put(c_dst, o.c_dst); put(c_row, o.c_row);
  put(r_off, o.r_off); put(r_row, o.r_row);
  if (n_disp) *n_disp = (int32_t)o.d_tok.size();
  if (n_sub) *n_sub = (int32_t)o.sub.size();
  return MOEPIC_OK;
}

// The step's admissions, counters and statistics are committed (and copies into admitted slots
// may be queued) before the kernels are launched: a failure after that point cannot be undone,
// so it poisons the context (moepic.h: ERUNTIME -> every later call returns ESTATE).
moepic_status moepic_layer_forward(moepic_ctx* ctx, int32_t layer, const void* h_dev, int32_t B, float* y_dev,
                                   void* stream, uint32_t flags, moepic_trace* tr) {
  CTX_GUARD();
  ctx->committed = false;
  const bool grouped = ctx->grp && ctx->grp->joined;
  if ((flags & MOEPIC_TOKENS_SHARDED) && !grouped)
    return fail(&ctx->err, MOEPIC_EINVAL, "MOEPIC_TOKENS_SHARDED needs a joined group");
  if (grouped && !(flags & MOEPIC_TOKENS_SHARDED) && B > kDecodeMaxB)
    return fail(&ctx->err, MOEPIC_EINVAL, "replicated tokens over a group need B <= 32 (use MOEPIC_TOKENS_SHARDED)");
  moepic_status st;
  if (ctx->fault_at_step > 0 && ++ctx->fault_steps == ctx->fault_at_step) {
    st = inject_fault(ctx, static_cast<cudaStream_t>(stream));
  } else if (flags & MOEPIC_TOKENS_SHARDED) {
    st = sharded_forward(ctx, layer, h_dev, B, y_dev, stream, flags, tr);
  } else {
    st = layer_forward_impl(ctx, layer, h_dev, B, y_dev, stream, flags, tr);
    if (st == MOEPIC_OK && grouped) st = group_allreduce(ctx, y_dev, B, static_cast<cudaStream_t>(stream));
  }
  if (st != MOEPIC_OK && (ctx->committed || st == MOEPIC_ERUNTIME)) {
    ctx->poisoned = true;
    if (st != MOEPIC_ERUNTIME) st = MOEPIC_ERUNTIME;
  }
  ctx->committed = false;
  return st;
}

// host memcpy of prefill-sized buffers (tens of MB) split over the OpenMP threads
static void par_memcpy(void* dst, const void* src, size_t bytes) {
  constexpr size_t kPiece = 1u << 20;
  if (bytes <= 2 * kPiece) {
    memcpy(dst, src, bytes);
    return;
  }
  const long n = (long)((bytes + kPiece - 1) / kPiece);
#pragma omp parallel for schedule(static)
  for (long i = 0; i < n; ++i) {
    const size_t off = (size_t)i * kPiece;
    memcpy(static_cast<uint8_t*>(dst) + off, static_cast<const uint8_t*>(src) + off, std::min(kPiece, bytes - off));
  }
}

moepic_status moepic_layer_forward_host(moepic_ctx* ctx, int32_t layer, const uint16_t* h_host, int32_t B,
                                        float* y_host, void* stream, uint32_t flags, moepic_trace* tr) {
  CTX_GUARD();
  const auto& d = ctx->desc;
  if (!h_host || !y_host) return fail(&ctx->err, MOEPIC_EINVAL, "h_host / y_host is NULL");
  if (B < 1 || B > d.max_batch) return fail(&ctx->err, MOEPIC_EINVAL, "B must be in [1, max_batch]");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t hb = (size_t)B * d.d * 2, yb = (size_t)B * d.d * 4;
  const size_t yoff = align_up((size_t)d.max_batch * d.d * 2);
  // h: host -> mapped pinned staging -> arena (SM loads, not the busy H2D copy engine);
  // y: the combine stores straight into the mapped staging (zero-copy), read after the sync.
  // Both buffers are allocated at create, so no allocation happens on this path.
  const auto th0 = std::chrono::steady_clock::now();
  par_memcpy(ctx->scratch_h, h_host, hb);
  uint8_t* ds = ctx->arena + ctx->lay.hstage;
  launch_stage_in(ds, ctx->scratch_d, (hb + 15) / 16 * 16, s);
  CK(cudaGetLastError());
  // prefill outputs (MBs) are written to device memory and read back by the D2H copy engine
  // (the device->host direction is idle; scattered SM stores into host memory crawl)
  const bool big = B > kDecodeMaxB;
  float* yd = big ? reinterpret_cast<float*>(ctx->arena + ctx->lay.ystage)
                  : reinterpret_cast<float*>(ctx->scratch_d + yoff);
  const auto th1 = std::chrono::steady_clock::now();
  moepic_status st = moepic_layer_forward(ctx, layer, ds, B, yd, stream, flags, tr);
  if (st != MOEPIC_OK) return st;
  const auto th2 = std::chrono::steady_clock::now();
  if (big) CK(cudaMemcpyAsync(ctx->scratch_h + yoff, yd, yb, cudaMemcpyDeviceToHost, s));
  // wait for the layer while pumping the next layer's prefetch feed (cancel-at-router, Q7): a
  // plain stream synchronise would stall the feed, and the link with it, for the whole wait and
  // the caller's round trip (Qwen3 B = 16: e2e 0.917 vs 0.964 of the PCIe roofline)
  CK(cudaEventRecord(ctx->ev_tmp, s));
  for (uint64_t spins = 0;; ++spins) {
    const cudaError_t q = cudaEventQuery(ctx->ev_tmp);
    if (q == cudaSuccess) break;
    if (q != cudaErrorNotReady) return ctx->poisoned = true, fail(&ctx->err, MOEPIC_ERUNTIME, "layer failed: %s", cudaGetErrorString(q));
    if ((spins & 0x7) == 0 && !ctx->feed_pump(ctx->cancel_prefetch ? ctx->kFeedDepth : (size_t)-1)) {
      ctx->poisoned = true;
      return fail(&ctx->err, MOEPIC_ERUNTIME, "prefetch feed: %s", cudaGetErrorString(cudaGetLastError()));
    }
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
  }
  par_memcpy(y_host, ctx->scratch_h + yoff, yb);
  if (ctx->host_timing) {   // MOEPIC_HOST_TIMING (tools)
    auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
    const auto th3 = std::chrono::steady_clock::now();
    ctx->hh[0] += us(th0, th1);
    ctx->hh[1] += us(th1, th2);
    ctx->hh[2] += us(th2, th3);
    ctx->hh_n++;
  }
  return MOEPIC_OK;
}

moepic_status moepic_predict_prefetch(moepic_ctx* ctx, int32_t next_layer, const void* h_dev, int32_t B,
                                      void* stream, moepic_trace* tr) {
  CTX_GUARD();
  const auto& d = ctx->desc;
  if (!ctx->configured) return fail(&ctx->err, MOEPIC_EINVAL, "moepic_configure has not been called");
  if (next_layer < 0 || next_layer >= d.L) return fail(&ctx->err, MOEPIC_EINVAL, "next_layer out of range");
  if (B < 1 || B > d.max_batch) return fail(&ctx->err, MOEPIC_EINVAL, "B must be in [1, max_batch]");
  if (!h_dev || (reinterpret_cast<uintptr_t>(h_dev) & 15))
    return fail(&ctx->err, MOEPIC_EINVAL, "h_dev must be a 16-byte aligned device pointer");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  moepic_status st = run_router(ctx, static_cast<const uint16_t*>(h_dev), B, -1, next_layer, s, false, true);
  if (st != MOEPIC_OK) return st;
  Plan next;
  ctx->cp->make_plan(next_layer, ctx->rank_h.data(), next);
  ctx->pending = Plan();
  st = issue_plan(ctx, next, ctx->last_buf ^ 1);
  if (st != MOEPIC_OK) return st;
  ctx->pending = next;
  if (tr) {
    StepResult empty;
    fill_step_trace(tr, empty, &next);
    tr->n_act = 0;
    tr->n_adm = 0;
    tr->pcie_ondemand_bytes = 0;
    tr->pcie_prefetch_bytes = plan_bytes(next, (int64_t)ctx->rb());
    tr->hbm_bytes = tr->pcie_prefetch_bytes + (uint64_t)d.N * d.d * 2;
    tr->kernel_launches = 1;
  }
  return MOEPIC_OK;
}

// statistics snapshot: header {L, N, K} then per layer: q, q_pred, freq[N], rank_hit[N+1],
// pred_hit[N+1], pred_rank[(N+1)^2], mu[N], nu[N], last[N], step_no   (all int64)
static size_t stats_bytes(const moepic_model_desc& d) {
  const size_t N = d.N;
  return 8 * (3 + (size_t)d.L * (2 + N + (N + 1) + (N + 1) + (N + 1) * (N + 1) + 3 * N + 1));
}

static moepic_status stats_save(const ControlPlane& cp, const moepic_model_desc& d, std::string* err, void* buf,
                                size_t* bytes) {
  if (!bytes) return fail(err, MOEPIC_EINVAL, "bytes is NULL");
  const size_t need = stats_bytes(d);
  if (!buf) { *bytes = need; return MOEPIC_OK; }
  if (*bytes < need) return fail(err, MOEPIC_EINVAL, "buffer too small (%zu < %zu)", *bytes, need);
  int64_t* o = static_cast<int64_t*>(buf);
  *o++ = d.L; *o++ = d.N; *o++ = d.K;
  for (const auto& l : cp.layers) {
    *o++ = l.st.q; *o++ = l.st.q_pred;
    for (auto v : l.st.freq) *o++ = v;
    for (auto v : l.st.rank_hit) *o++ = v;
    for (auto v : l.st.pred_hit) *o++ = v;
    for (auto v : l.st.pred_rank) *o++ = v;
    for (auto v : l.mu) *o++ = v;
    for (auto v : l.nu) *o++ = v;
    for (auto v : l.last) *o++ = v;
    *o++ = l.step_no;
  }
  *bytes = need;
  return MOEPIC_OK;
}

static moepic_status stats_load(ControlPlane& cp, const moepic_model_desc& d, std::string* err, const void* buf,
                                size_t bytes) {
  if (!buf || bytes != stats_bytes(d)) return fail(err, MOEPIC_EINVAL, "snapshot size mismatch");
  const int64_t* in = static_cast<const int64_t*>(buf);
  if (in[0] != d.L || in[1] != d.N || in[2] != d.K)
    return fail(err, MOEPIC_EINVAL, "snapshot shape (L, N, K) mismatch");
  in += 3;
  for (auto& l : cp.layers) {
    l.st.q = *in++; l.st.q_pred = *in++;
    for (auto& v : l.st.freq) v = *in++;
    for (auto& v : l.st.rank_hit) v = *in++;
    for (auto& v : l.st.pred_hit) v = *in++;
    for (auto& v : l.st.pred_rank) v = *in++;
    for (auto& v : l.mu) v = *in++;
    for (auto& v : l.nu) v = *in++;
    for (auto& v : l.last) v = *in++;
    l.step_no = *in++;
    l.st.dirty = true;
  }
  return MOEPIC_OK;
}

moepic_status moepic_get_stats(moepic_ctx* ctx, void* buf, size_t* bytes) {
  CTX_GUARD();
  return stats_save(*ctx->cp, ctx->desc, &ctx->err, buf, bytes);
}

moepic_status moepic_set_stats(moepic_ctx* ctx, const void* buf, size_t bytes) {
  CTX_GUARD();
  return stats_load(*ctx->cp, ctx->desc, &ctx->err, buf, bytes);
}

moepic_status moepic_get_counters(moepic_ctx* ctx, moepic_counters* out) {
  CTX_GUARD();
  if (!out) return MOEPIC_EINVAL;
  *out = ctx->ctr;
  return MOEPIC_OK;
}

moepic_status moepic_profile(moepic_ctx* ctx, int32_t enable) {
  CTX_GUARD();
  ctx->prof_drain();
  for (auto& k : ctx->prof_acc) k = moepic_kernel_stats{};
  ctx->profiling = enable != 0;
  ctx->prof_mask = (enable & MOEPIC_PROFILE_CLASSES) ? (uint32_t)(enable & 0xF) : 0xFu;
  if (ctx->profiling) {
    ctx->tstamp_reset(kProfRing);
    if (cudaDeviceSynchronize() != cudaSuccess) return fail(&ctx->err, MOEPIC_ERUNTIME, "profile reset failed");
  }
  return MOEPIC_OK;
}

moepic_status moepic_profile_read(moepic_ctx* ctx, int32_t kernel_class, moepic_kernel_stats* out) {
  CTX_GUARD();
  if (!out || kernel_class < 0 || kernel_class > 3) return fail(&ctx->err, MOEPIC_EINVAL, "bad profile_read args");
  ctx->prof_drain();
  *out = ctx->prof_acc[kernel_class];
  return MOEPIC_OK;
}

moepic_status moepic_attention_ws_bytes(int32_t B, int32_t S, int32_t Hq, int32_t Hkv, int32_t dh, size_t* bytes) {
  if (!bytes || B < 1 || S < 1 || S > 1024 * kAttnChunk || Hq < 1 || Hkv < 1 || dh != 128) return MOEPIC_EINVAL;
  *bytes = (size_t)B * Hq * attn_splits(S) * (dh + 2) * sizeof(float);
  return MOEPIC_OK;
}

moepic_status moepic_attention_decode(const void* q, const void* k_cache, const void* v_cache, int32_t B,
                                      int32_t S, int32_t S_max, int32_t Hq, int32_t Hkv, int32_t dh,
                                      float* out, void* ws, size_t ws_bytes, void* stream) {
  size_t need = 0;
  if (moepic_attention_ws_bytes(B, S, Hq, Hkv, dh, &need) != MOEPIC_OK) return MOEPIC_EINVAL;
  if (!q || !k_cache || !v_cache || !out || !ws || S > S_max || Hq % Hkv != 0 || ws_bytes < need) return MOEPIC_EINVAL;
  for (const void* ptr : {q, k_cache, v_cache, (const void*)out, (const void*)ws})
    if (reinterpret_cast<uintptr_t>(ptr) & 7) return MOEPIC_EINVAL;
  const int G = Hq / Hkv;
  if (G != 1 && G != 2 && G != 4 && G != 8 && G != 16) return MOEPIC_EINVAL;
  static const bool attrs_ok = attention_init() == cudaSuccess;   // context-free entry: set once
  (void)attrs_ok;
  AttnParams p{};
  p.q = static_cast<const uint16_t*>(q);
  p.k = static_cast<const uint16_t*>(k_cache);
  p.v = static_cast<const uint16_t*>(v_cache);
  p.out = out;
  p.ws = static_cast<float*>(ws);
  p.B = B; p.S = S; p.S_max = S_max; p.Hq = Hq; p.Hkv = Hkv; p.splits = attn_splits(S);
  if (!launch_attention(p, static_cast<cudaStream_t>(stream))) return MOEPIC_EINVAL;
  return cudaGetLastError() == cudaSuccess ? MOEPIC_OK : MOEPIC_ERUNTIME;
}

const char* moepic_last_error(const moepic_ctx* ctx) { return ctx ? ctx->err.c_str() : "ctx is NULL"; }

void moepic_destroy(moepic_ctx* ctx) {
  if (!ctx) return;
  cudaDeviceSynchronize();
  if (ctx->tl_dev && !ctx->tl_host.empty()) {   // MOEPIC_TIMELINE
    int64_t h1 = 0, off1 = 0;
    ctx->tl_calibrate(h1, off1);
    auto conv = [&](int64_t h) -> long long {
      if (h == 0) return 0;
      const double f = h1 > ctx->tl_h0 ? (double)(h - ctx->tl_h0) / (double)(h1 - ctx->tl_h0) : 0.0;
      return (long long)(h + ctx->tl_off0 + (int64_t)((double)(off1 - ctx->tl_off0) * f));
    };
    std::vector<unsigned long long> g((size_t)2 * kProfRing);
    cudaMemcpy(g.data(), ctx->tl_dev, g.size() * 8, cudaMemcpyDeviceToHost);
    if (FILE* f = fopen(ctx->tl_path.c_str(), "w")) {
      auto st = [&](size_t i) { return g[i] == ~0ull ? -1LL : (long long)g[i]; };
      auto en = [&](size_t i) { return g[kProfRing + i] == 0 ? -1LL : (long long)g[kProfRing + i]; };
      for (size_t r = 0; r < ctx->tl_host.size(); ++r) {
        const auto& h = ctx->tl_host[r];
        fprintf(f, "{\"rec\": %zu, \"layer\": %d, \"host\": [%lld, %lld, %lld, %lld, %lld], \"od_bytes\": %llu, "
                "\"router\": [%lld, %lld], \"k2_first\": [%lld, %lld], \"k2_final\": [%lld, %lld], \"copy_done\": %lld, "
                "\"copy_start\": %lld}\n",
                r, h.layer, conv(h.t[0]), conv(h.t[1]), conv(h.t[2]), conv(h.t[3]), conv(h.t[4]),
                (unsigned long long)h.od_bytes, st(r * 8), en(r * 8), st(r * 8 + 3), en(r * 8 + 3), st(r * 8 + 1),
                en(r * 8 + 1), st(r * 8 + 2), st(r * 8 + 4));
      }
      fclose(f);
    }
  }
  if (ctx->tl_dev) cudaFree(ctx->tl_dev);
  if (ctx->ht_n)
    fprintf(stderr, "[hosttiming] %llu calls: launch router + wait routing %.1f | routing -> first copy issued %.1f | "
            "routing -> all copies issued %.1f | K2 launches + next plan %.1f us\n", (unsigned long long)ctx->ht_n,
            ctx->ht[0] / ctx->ht_n, ctx->ht[1] / ctx->ht_n, ctx->ht[2] / ctx->ht_n, ctx->ht[3] / ctx->ht_n);
  if (ctx->hh_n)
    fprintf(stderr, "[hosttiming] host-buffer entry x%llu: stage-in %.1f, forward call %.1f, sync + y read %.1f us\n",
            (unsigned long long)ctx->hh_n, ctx->hh[0] / ctx->hh_n, ctx->hh[1] / ctx->hh_n, ctx->hh[2] / ctx->hh_n);
  if (ctx->ht_n)
    fprintf(stderr, "[hosttiming] classify %.1f, finish_plan %.1f, pass 1 %.1f, commit %.1f us\n", ctx->hp[0] / ctx->ht_n,
            ctx->hp[1] / ctx->ht_n, ctx->hp[2] / ctx->ht_n, ctx->hp[3] / ctx->ht_n);
  if (ctx->hf_n)
    fprintf(stderr, "[hosttiming] finish_plan x%llu: cancel %.1f, pump %.1f (feed %.2f chunks, %.2f walked, %.2f copied, "
            "%.2f in flight before; %.2f items, %.2f kept), drop+record %.1f us\n",
            (unsigned long long)ctx->hf_n, ctx->hf[0] / ctx->hf_n, ctx->hf[1] / ctx->hf_n, ctx->hf[8] / ctx->hf_n,
            ctx->hf[3] / ctx->hf_n, ctx->hf[5] / ctx->hf_n, ctx->hf[6] / ctx->hf_n, ctx->hf[4] / ctx->hf_n,
            ctx->hf[7] / ctx->hf_n, ctx->hf[2] / ctx->hf_n);
  if (ctx->hc_n)
    fprintf(stderr, "[hosttiming] %llu copies: stream waits %.1f us, cudaMemcpyAsync %.1f us per copy\n",
            (unsigned long long)ctx->hc_n, ctx->hc[0] / ctx->hc_n, ctx->hc[1] / ctx->hc_n);
  if (ctx->gate_steps && ctx->host_timing)
    fprintf(stderr, "[hosttiming] gated K2: %llu steps, mean max gate wait %.1f us, tail controller %.3f\n",
            (unsigned long long)ctx->gate_steps, ctx->gate_wait_us_sum / ctx->gate_steps, ctx->gate_ctrl);
  if (ctx->k1dbg) {   // MOEPIC_K1_TRACE summary: mean phase offsets from the first CTA start (us)
    std::vector<unsigned long long> h(4096 * 8);
    cudaMemcpy(h.data(), ctx->k1dbg, h.size() * 8, cudaMemcpyDeviceToHost);
    const size_t n = std::min<uint64_t>(ctx->k1dbg_n, 4096);
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    size_t cnt = 0;
    for (size_t i = 0; i < n; ++i) {
      const unsigned long long* r = &h[i * 8];
      if (r[0] == ~0ull || r[4] < r[0] || r[3] < r[0]) continue;
      for (int k = 1; k < 8; ++k) acc[k] += r[k] >= r[0] && r[k] != ~0ull ? (double)(r[k] - r[0]) * 1e-3 : 0.0;
      ++cnt;
    }
    if (cnt)
      fprintf(stderr, "[k1trace] %zu launches: phase1_end %.2f select_start %.2f selected %.2f routed %.2f "
              "pred_topk %.2f ranked %.2f end %.2f us\n", cnt, acc[1] / cnt, acc[2] / cnt, acc[5] / cnt,
              acc[3] / cnt, acc[6] / cnt, acc[7] / cnt, acc[4] / cnt);
    cudaFree(ctx->k1dbg);
  }
  if (ctx->grp) {
    Group& g = *ctx->grp;
    for (int r = 0; r < kEpMaxRanks; ++r)
      if (g.opened[r]) cudaIpcCloseMemHandle(g.pr.base[r]);
    if (g.comm) nccl_api().CommDestroy(g.comm);
    if (g.region) cudaFree(g.region);
    if (g.idx_h) cudaFreeHost(g.idx_h);
  }
  if (ctx->copy) cudaStreamDestroy(ctx->copy);
  if (ctx->copy2) cudaStreamDestroy(ctx->copy2);
  if (ctx->ev_copy2) cudaEventDestroy(ctx->ev_copy2);
  for (auto e : ctx->feed_ev)
    if (e) cudaEventDestroy(e);
  for (auto& pe : ctx->prof) {
    cudaEventDestroy(pe.a);
    cudaEventDestroy(pe.b);
  }
  cudaEvent_t evs[] = {ctx->ev_od, ctx->ev_od_head, ctx->ev_plan[0], ctx->ev_plan[1], ctx->ev_step[0], ctx->ev_step[1], ctx->ev_tmp};
  for (auto e : evs)
    if (e) cudaEventDestroy(e);
  if (ctx->host_experts) cudaFreeHost(ctx->host_experts);
  if (ctx->mailbox) cudaFreeHost(ctx->mailbox);
  if (ctx->scratch_h) cudaFreeHost(ctx->scratch_h);
  if (ctx->stall_h) cudaFreeHost(ctx->stall_h);
  delete ctx;
}

// ====================================================================== host-only simulator
struct moepic_hostsim {
  moepic_model_desc desc{};
  std::unique_ptr<ControlPlane> cp;
  ArenaLayout lay{};
  Plan pending;
  std::string err;
};

moepic_status moepic_hostsim_create(const moepic_model_desc* desc, moepic_hostsim** out) {
  if (!out) return MOEPIC_EINVAL;
  *out = nullptr;
  if (!validate_desc(desc).empty()) return MOEPIC_EINVAL;
  auto* hs = new (std::nothrow) moepic_hostsim();
  if (!hs) return MOEPIC_ENOMEM;
  const moepic_model_desc local = local_desc(*desc);
  desc = &local;
  hs->desc = *desc;
  hs->lay = arena_layout(*desc);
  hs->cp.reset(new ControlPlane(desc->L, desc->N, desc->K, desc->d, desc->I, desc->row_granule,
                                desc->buffer_experts, desc->n_shared, desc->ep_rank, desc->ep_size));
  hs->cp->row_bytes = (int64_t)row_bytes_of(*desc);
  *out = hs;
  return MOEPIC_OK;
}

moepic_status moepic_hostsim_configure(moepic_hostsim* hs, const moepic_cache_config* cfg,
                                       moepic_config_out* out) {
  if (!hs) return MOEPIC_EINVAL;
  if (!cfg) return fail(&hs->err, MOEPIC_EINVAL, "cfg is NULL");
  if (cfg->v_e > hs->desc.v_e_max + 1e-9) return fail(&hs->err, MOEPIC_EINVAL, "v_e exceeds v_e_max");
  std::string e = hs->cp->configure(to_params(cfg, hs->desc.L), hs->lay.pool_rows);
  if (!e.empty()) return fail(&hs->err, MOEPIC_EINVAL, "%s", e.c_str());
  hs->pending = Plan();
  write_config_out(*hs->cp, out);
  return MOEPIC_OK;
}

moepic_status moepic_hostsim_step(moepic_hostsim* hs, int32_t layer, const int32_t* ids, int32_t B,
                                  int32_t next_layer, const int32_t* ranking_next, moepic_trace* tr) {
  if (!hs) return MOEPIC_EINVAL;
  const auto& d = hs->desc;
  if (!hs->cp->configured) return fail(&hs->err, MOEPIC_EINVAL, "not configured");
  if (layer < 0 || layer >= d.L) return fail(&hs->err, MOEPIC_EINVAL, "layer out of range");
  if (B < 1 || B > 4096 || !ids) return fail(&hs->err, MOEPIC_EINVAL, "bad ids / B");
  for (int i = 0; i < B * d.K; ++i)
    if (ids[i] < 0 || ids[i] >= d.N) return fail(&hs->err, MOEPIC_EINVAL, "expert id out of range");
  if (ranking_next && (next_layer < 0 || next_layer >= d.L)) return fail(&hs->err, MOEPIC_EINVAL, "next_layer out of range");
  Plan used;
  const bool have = hs->pending.valid && hs->pending.target == layer;
  if (have) used = std::move(hs->pending);
  hs->pending = Plan();
  StepResult res;
  hs->cp->step(layer, ids, B, have ? &used : nullptr, res);
  Plan next;
  if (ranking_next) {
    hs->cp->make_plan(next_layer, ranking_next, next);
    hs->pending = next;
  }
  const uint64_t pb = ranking_next ? plan_bytes(next, hs->cp->row_bytes) : 0;
  if (tr) {
    fill_step_trace(tr, res, ranking_next ? &next : nullptr);
    tr->pcie_prefetch_bytes = pb;
    tr->hbm_bytes = step_hbm_bytes(*hs->cp, res, B, ranking_next ? 2 : 1, pb);
    tr->kernel_launches = 0;
  }
  return MOEPIC_OK;
}

moepic_status moepic_hostsim_predict(moepic_hostsim* hs, int32_t next_layer, const int32_t* ranking,
                                     moepic_trace* tr) {
  if (!hs) return MOEPIC_EINVAL;
  if (!hs->cp->configured) return fail(&hs->err, MOEPIC_EINVAL, "not configured");
  if (next_layer < 0 || next_layer >= hs->desc.L || !ranking) return fail(&hs->err, MOEPIC_EINVAL, "bad args");
  Plan next;
  hs->cp->make_plan(next_layer, ranking, next);
  hs->pending = next;
  if (tr) {
    StepResult empty;
    fill_step_trace(tr, empty, &next);
    tr->pcie_prefetch_bytes = plan_bytes(next, hs->cp->row_bytes);
    tr->hbm_bytes = tr->pcie_prefetch_bytes + (uint64_t)hs->desc.N * hs->desc.d * 2;
    tr->kernel_launches = 0;
  }
  return MOEPIC_OK;
}

moepic_status moepic_hostsim_cached(moepic_hostsim* hs, int32_t layer, int32_t* out, int32_t* n) {
  if (!hs || !out || !n || layer < 0 || layer >= hs->desc.L) return MOEPIC_EINVAL;
  int c = 0;
  const LayerState& l = hs->cp->layers[layer];
  for (int e = 0; e < hs->desc.N; ++e)
    if (l.cached(e)) out[c++] = e;
  *n = c;
  return MOEPIC_OK;
}

moepic_status moepic_hostsim_get_stats(moepic_hostsim* hs, void* buf, size_t* bytes) {
  if (!hs) return MOEPIC_EINVAL;
  return stats_save(*hs->cp, hs->desc, &hs->err, buf, bytes);
}

moepic_status moepic_hostsim_set_stats(moepic_hostsim* hs, const void* buf, size_t bytes) {
  if (!hs) return MOEPIC_EINVAL;
  return stats_load(*hs->cp, hs->desc, &hs->err, buf, bytes);
}

const char* moepic_hostsim_last_error(const moepic_hostsim* hs) { return hs ? hs->err.c_str() : "hs is NULL"; }
void moepic_hostsim_destroy(moepic_hostsim* hs) { delete hs; }

}  // extern "C"
