/* moepic.h — C ABI of the B200-native MoEpic split-expert MoE layer library.
 *
 * MoEpic (arXiv 2509.08342, "Accelerating Mixture-of-Expert Inference with Adaptive Expert
 * Split Mechanism").  Citations "P:<n>" are lines of the paper text; readings of
 * silent or ambiguous passages are numbered Q1..Q26 in DESIGN.md.
 *
 * What one library context does:
 *   - every expert of every layer lives in pinned host RAM in a row-interleaved layout
 *     (row r = [gate_r | up_r | down[:, r]], 6*d bytes);
 *   - each expert is split along its intermediate dimension I at I_top rows (reading Q1/Q2);
 *     the TOP rows of the C_i hottest experts of layer i stay cached in HBM;
 *   - layer_forward routes the batch (top-K gate softmax), computes the resident
 *     segments at once, streams missing bottoms / experts over PCIe on a copy stream and
 *     computes them when they land, sums the partial down-projections;
 *   - the same call runs the NEXT layer's router on the current activation (Eq. 3)
 *     and prefetches that layer's bottoms (or full experts) in descending predicted score
 *      into a ping-pong HBM buffer of U_b expert units;
 *   - a host cache manager (LCP Eq. 4 / LRU / LFU / RND) admits missed experts;
 *   - configure runs Alg. 1 on the recorded statistics and re-lays out the cache.
 *
 * Conventions for every function:
 *   - returns moepic_status; nothing throws across the ABI; on a non-OK status
 *     moepic_last_error(ctx) names the offending argument or the failing CUDA call.
 *   - MOEPIC_EINVAL leaves the context unchanged.  MOEPIC_ERUNTIME (a CUDA failure) poisons
 *     the context: every later call returns MOEPIC_ESTATE.
 *   - "device pointer" = CUDA global memory of the context's device; "host pointer" = plain
 *     process memory (pageable is fine; it is copied).
 *   - bf16 values are passed as uint16_t bit patterns.
 *   - calls on one context must be serialised by the caller (one ctx per process and GPU).
 */
#ifndef MOEPIC_H
#define MOEPIC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MOEPIC_OK = 0,
  MOEPIC_EINVAL = 1,   /* bad argument or configuration; context unchanged            */
  MOEPIC_ERUNTIME = 2, /* a CUDA call failed; context poisoned                           */
  MOEPIC_ENOMEM = 3,   /* the arena (or pinned host memory) is too small                 */
  MOEPIC_ESTATE = 4    /* context poisoned by an earlier MOEPIC_ERUNTIME                 */
} moepic_status;

/* cache replacement policy (Table 1) */
typedef enum { MOEPIC_LCP = 0, MOEPIC_LRU = 1, MOEPIC_LFU = 2, MOEPIC_RND = 3 } moepic_policy;

/* activation classes: all rows resident / top only / nothing resident */
enum { MOEPIC_ALPHA = 0, MOEPIC_BETA = 1, MOEPIC_GAMMA = 2 };
/* admission victim codes in moepic_trace.adm_victim */
enum { MOEPIC_ADM_FREE_SLOT = -1, MOEPIC_ADM_NONE = -2 };

/* layer_forward flags */
enum {
  MOEPIC_FUSE_PREDICT = 1, /* run R^{(i+1) mod L} on h^i and prefetch that layer (Eq. 3)    */
  MOEPIC_RESIDUAL = 2,     /* y = h + MoE(h) instead of MoE(h) (Eq. 2's inner h + sum) */
  MOEPIC_TOKENS_SHARDED = 4 /* expert parallel with tokens sharded over the group (SURVEY §8(e),
                              prefill config 5): see moepic_group_join                          */
};

typedef struct moepic_ctx moepic_ctx;

/* Model shape (Table 2).  Invariants (EINVAL otherwise):
 *   1 <= K < N; L >= 1; d % 8 == 0 and d >= 8; I % row_granule == 0;
 *   row_granule % 16 == 0; buffer_experts >= K (U_b); 1 <= max_batch <= 4096;
 *   1 <= L_host <= L; 0 <= ep_rank < ep_size; N % ep_size == 0; tp fields as documented below;
 *   max_batch > 32 (prefill) additionally needs d % 256 == 0, N + n_shared <= 136 and
 *   row_granule, I / tp_size multiples of 64.                                                  */
typedef struct {
  int32_t L, N, K, d, I;  /* layers, routed experts per layer, top-K, hidden, intermediate     */
  int32_t n_shared;       /* shared experts per layer: always resident, weight 1, unsplit (Q6) */
  int32_t row_granule;    /* g: I_top is a multiple of g (reading Q2); default 64              */
  int32_t buffer_experts; /* U_b in full-expert units per ping-pong half (default K)      */
  int32_t max_batch;      /* largest B passed to layer_forward / predict_prefetch              */
  int32_t renorm_topk;    /* 1: Eq. 2 renormalised gate (default); 0: raw softmax s_j (Q4)      */
  int32_t L_host;         /* distinct layers stored in pinned host RAM; logical layer i reads
                             physical layer i % L_host (bench aliasing)             */
  double v_e_max;         /* largest expert-cache budget V_e (full-expert units) configure may
                             request; sizes the HBM slot pool                                  */
  int32_t ep_rank, ep_size; /* expert parallel: expert e is local iff e*ep_size/N == ep_rank   */
  int32_t tp_rank, tp_size; /* tensor parallel along I (the split identity
                             P:254 applied across GPUs): this context holds intermediate rows
                             [tp_rank*I/tp_size, (tp_rank+1)*I/tp_size) of EVERY routed and
                             shared expert; load_expert takes the full HF tensors and keeps that
                             slice.  Every size the context reports or accepts (row_granule
                             multiples, I_top_i, v_e / v_i in full-expert units, byte counters)
                             refers to the local slice of I/tp_size rows.  Routing is replicated
                             (bit-identical fp64 logits on every rank), so all ranks take the
                             same cache decisions.  y_dev is this rank's partial output; the
                             caller sums it over ranks (all-reduce).  MOEPIC_RESIDUAL adds h on
                             tp_rank 0 only.  EINVAL unless 0 <= tp_rank < tp_size,
                             I % (tp_size*row_granule) == 0, and ep_size == 1 when tp_size > 1. */
  int32_t weight_format;  /* MOEPIC_BF16 (0): experts stored and streamed as bf16.
                             MOEPIC_Q4G64 (1): low-bit experts (the paper's
                             Mixtral ran HQQ low-bit experts): load_expert quantises
                             every stored row vector (gate row, up row, down column) in groups
                             of 64 to 4-bit codes with a bf16 scale and minimum (DESIGN.md
                             reading Q28); K2 dequantises on the fly (fp32 accumulation).  A
                             row then takes 27d/16 bytes (padded to 16) instead of 6d, so every
                             PCIe and HBM byte count shrinks ~3.5x.  Needs d % 64 == 0.  Prefill
                             batches (> 32 tokens) dequantise each segment group once into fp16
                             rows for the tcgen05 GEMMs (reading Q32).                         */
} moepic_model_desc;
enum { MOEPIC_BF16 = 0, MOEPIC_Q4G64 = 1 };

/* Cache configuration.  EINVAL when: v_e < 0 or
 * v_e > v_e_max; any theta_i outside (0, 1]; any v_i < 0; sum v_i > v_e (+1e-9); policy out
 * of range; rho outside (0,1); omega < 1; zeta outside (0,1); use_solver with an empty
 * statistics accumulator on some layer; t_load_exp <= 0 or t_moe <= 0 with use_solver. */
typedef struct {
  double v_e;              /* V_e: expert-cache budget in full-expert units             */
  const double* v_i;       /* [L] per-layer budgets, or NULL -> uniform V_e / L         */
  const double* theta_i;   /* [L] split ratios in (0,1], or NULL -> 0.5; ignored when
                              use_solver = 1                                                    */
  int32_t use_solver;      /* 1: run Alg. 1 VramAllocation on the recorded stats        */
  int32_t policy;          /* moepic_policy                                                     */
  double rho;              /* LCP rho (default 0.25)                                     */
  int32_t omega;           /* LCP omega (default 128)                                    */
  double zeta;             /* allocation granularity (default 0.01)                      */
  double t_att, t_moe, t_head, t_load_exp; /* profiled latencies, any one time unit   */
  const int32_t* y_cap_i;  /* [L] max prefetch count per layer, or NULL (buffer-bound)          */
  int32_t prefetch;        /* 0: no speculative prefetch (cache-only baseline); 1: on          */
  uint64_t seed;           /* splitmix64 seed: initial random cached set, RND victims   */
  int32_t cancel_prefetch; /* 1: prefetch is fed in chunks while the host waits for routing and
                              the unissued chunks of experts the router did not activate are
                              dropped ("terminates the prefetch operation").  Plans,
                              classes and traces are unchanged; only the bytes actually moved
                              (moepic_counters) differ.  0: every planned byte is transferred.  */
  const int64_t* prefetch_rows_i; /* [L] prefetch window W_i in expert rows, or NULL.  Reading Q30
                              (DESIGN.md): the plan for layer i is cut at min(U_b*I, W_i) rows
                              and the bottom at the cut keeps its first g*floor(rest/g) rows --
                              the deterministic form of "the router terminates the prefetch"
                              (P:291); an activated expert with such a prefix is beta and loads
                              only the rest of its bottom.  With a window, Alg. 1's Y_i is not a
                              planner cap (y_cap_i still is).  EINVAL if any W_i < 0.          */
} moepic_cache_config;

/* configure output: caller-owned arrays of length L (any may be NULL) */
typedef struct {
  int32_t* C_i;        /* cache size (experts whose top is cached)                            */
  int32_t* I_top_i;    /* rows per cached top segment = g*floor(theta_i*I/g + 1e-9) (Q2)      */
  double* theta_eff_i; /* I_top_i / I                                                          */
  double* V_i;         /* budget per layer after Alg. 1                                        */
} moepic_config_out;

/* Per-call trace; every array is caller-owned and may be NULL (then it is not written).
 * Capacities: ids/w >= B*K; act_* , adm_*, plan_* >= N.                                       */
typedef struct {
  int32_t* ids;           /* [B*K] routed experts per token in key order (l desc, id asc)    */
  float* w;               /* [B*K] gate weights (Eq. 2)                                       */
  int32_t* act_expert;    /* distinct activated experts, order (B_e desc, id asc)  (Q9)      */
  int8_t* act_class;      /* MOEPIC_ALPHA / BETA / GAMMA, state before the call      */
  int32_t n_act;
  int32_t* adm_expert;    /* cache admissions in order (Q11)                           */
  int32_t* adm_victim;    /* evicted expert, or MOEPIC_ADM_FREE_SLOT / MOEPIC_ADM_NONE       */
  int32_t n_adm;
  int32_t* plan_expert;   /* prefetch plan made by this call for the next layer  */
  int8_t* plan_full;      /* 1 = full expert, 0 = bottom segment only                 */
  int32_t n_plan;
  int32_t plan_layer;     /* layer the plan targets, -1 if none                               */
  uint64_t pcie_ondemand_bytes; /* H2D bytes of missing segments of this layer        */
  uint64_t pcie_prefetch_bytes; /* H2D bytes of the plan issued by this call                  */
  uint64_t hbm_bytes;     /* algorithmic HBM bytes of this call          */
  int32_t kernel_launches;/* kernels this call enqueued                                       */
  int32_t* ranking;       /* [N] predicted ranking R' the plan was built from (Eq. 3, Q9)    */
} moepic_trace;

/* Bytes of device memory moepic_create needs for this model (slot pool for v_e_max, two
 * ping-pong buffers, routers, shared experts, workspace).  Host-only; no CUDA call.            */
moepic_status moepic_arena_bytes(const moepic_model_desc* desc, size_t* bytes);

/* Create a context on the current CUDA device.  dev_arena: caller-owned device allocation of
 * >= moepic_arena_bytes bytes, 256-byte aligned, that outlives the context.  The context
 * allocates pinned host memory for L_host*N experts (+ a mapped mailbox), a copy stream and
 * events.  On success *out is a new context; on failure *out is NULL.                         */
moepic_status moepic_create(const moepic_model_desc* desc, void* dev_arena, size_t dev_bytes,
                            moepic_ctx** out);

/* Host-only (no context, no GPU): the pinned-arena image of one expert as load_expert stores
 * it — this rank's I/tp_size interleaved rows in desc->weight_format (bf16: 6d bytes per row;
 * Q4G64: codes + group parameters).  out must hold *bytes = rows x row bytes;
 * out == NULL queries that size.  Lets tests compare the quantiser with the oracle bit for bit. */
moepic_status moepic_pack_expert(const moepic_model_desc* desc, const uint16_t* gate, const uint16_t* up,
                                 const uint16_t* down, void* out, size_t* bytes);

/* Router R^layer: w_bf16 host pointer to [N][d] bf16 (row j = expert j), copied.  layer < L. */
moepic_status moepic_load_router(moepic_ctx* ctx, int32_t layer, const uint16_t* w_bf16);

/* Expert weights in HuggingFace layout, host pointers, copied into the pinned arena in the
 * row-interleaved layout: gate [I][d], up [I][d], down [d][I] (bf16).  layer < L_host for
 * routed experts (expert in [0,N)); shared expert s is expert = -1 - s with layer < L.        */
moepic_status moepic_load_expert(moepic_ctx* ctx, int32_t layer, int32_t expert,
                                 const uint16_t* gate, const uint16_t* up, const uint16_t* down);

/* Blocking ("when the device is idle"): synchronises the device, computes
 * {V_i, theta_i, C_i} (uniform/given, or Alg. 1 when use_solver), ranks experts by cache
 * priority and copies the top segments of the top-C_i experts into HBM; drops
 * any pending prefetch.  out may be NULL.                                                      */
moepic_status moepic_configure(moepic_ctx* ctx, const moepic_cache_config* cfg,
                               moepic_config_out* out);

/* One MoE layer over a batch.
 *   h_dev: device pointer, bf16 [B][d] row-major (h^i);  1 <= B <= max_batch.
 *   y_dev: device pointer, fp32 [B][d] (written; Eq. 2 inner sum, + h if MOEPIC_RESIDUAL).
 *   stream: cudaStream_t (as void*; NULL = legacy default stream) all compute is ordered on.
 *   trace: may be NULL.
 * Blocks the host only until the routing of this batch is known (it plans copies); returns
 * with the GPU work enqueued on `stream`.  y_dev is valid after the stream reaches it.
 * Schedule (decode): on-demand copies on the context's copy stream; the split-
 * expert kernel covers the resident, prefetched and landed rows, and the tail of the last copy
 * either in the same launch behind a copy-stream flag (steps with >= 256 MB of rows;
 * MOEPIC_K2_GATE=0 never, =2 always) or in a second launch.  Results do not depend on it.     */
moepic_status moepic_layer_forward(moepic_ctx* ctx, int32_t layer, const void* h_dev, int32_t B,
                                   float* y_dev, void* stream, uint32_t flags,
                                   moepic_trace* trace);

/* Same as moepic_layer_forward with HOST buffers: h_host bf16 [B][d] is copied to the device,
 * y_host fp32 [B][d] is written before return (the call synchronises `stream`).               */
moepic_status moepic_layer_forward_host(moepic_ctx* ctx, int32_t layer, const uint16_t* h_host,
                                        int32_t B, float* y_host, void* stream, uint32_t flags,
                                        moepic_trace* trace);

/* Speculative prefetch for layer next_layer from activation h_dev (bf16 [B][d], device):
 * runs R^{next_layer}(h) (Eq. 3), ranks experts (Q9) and issues the prefetch plan.
 * Used for layer 0 with the previous token's last activation (Q23).  Replaces any
 * pending plan.  trace (plan fields only) may be NULL.                                         */
moepic_status moepic_predict_prefetch(moepic_ctx* ctx, int32_t next_layer, const void* h_dev,
                                      int32_t B, void* stream, moepic_trace* trace);

/* Statistics snapshot (checkpoint / offline configurator experiments).  buf == NULL queries the
 * size into *bytes; otherwise writes at most *bytes bytes.  set_stats restores a snapshot taken
 * from a context with the same (L, N, K).                                                      */
moepic_status moepic_get_stats(moepic_ctx* ctx, void* buf, size_t* bytes);
moepic_status moepic_set_stats(moepic_ctx* ctx, const void* buf, size_t bytes);

/* Cumulative counters since create. */
typedef struct {
  uint64_t layer_steps, kernel_launches, h2d_copies;
  uint64_t pcie_ondemand_bytes, pcie_prefetch_bytes, hbm_bytes;
  uint64_t act_alpha, act_beta, act_gamma;    /* class counts over all steps                  */
  uint64_t pred_hits, pred_total;             /* activated experts that were planned / total  */
  uint64_t pcie_prefetch_planned_bytes;       /* planned prefetch bytes (pcie_prefetch_bytes
                                                 counts what was actually transferred)        */
} moepic_counters;
moepic_status moepic_get_counters(moepic_ctx* ctx, moepic_counters* out);

/* Kernel timing with CUDA events recorded on the launching stream around every launch of the
 * given kernel class while profiling is enabled.  bytes = algorithmic HBM bytes of those
 * launches (K2: weight rows x 6d + activations).  kernel_ms sums, per
 * launch, the span from the first CTA's start to the last CTA's end read from %globaltimer
 * inside the kernels (0 for the prefill GEMMs), so total_ms - kernel_ms is launch latency.    */
typedef struct {
  uint64_t launches;
  double total_ms;
  uint64_t bytes;
  double kernel_ms;
} moepic_kernel_stats;
enum { MOEPIC_KERNEL_ROUTER = 0, MOEPIC_KERNEL_EXPERT = 1, MOEPIC_KERNEL_COMBINE = 2,
       MOEPIC_KERNEL_GEMM = 3 /* prefill tcgen05 GEMMs; `bytes` holds algorithmic FLOPs */ };
/* enable != 0 starts (and resets) event timing; 0 stops it.  enable = 1 times every class;
 * enable = MOEPIC_PROFILE_CLASSES | (1 << class) | ... times only those classes (each timing event
 * pair sits on the compute stream's critical path: ~4 us per record, more under a saturated H2D
 * link).                                                                        */
enum { MOEPIC_PROFILE_CLASSES = 0x100 };
moepic_status moepic_profile(moepic_ctx* ctx, int32_t enable);
/* Synchronises the recorded events and returns the totals for one kernel class.               */
moepic_status moepic_profile_read(moepic_ctx* ctx, int32_t kernel_class, moepic_kernel_stats* out);

/* Attention stand-in: the paper's Att^i (Eq. 1), whose duration
 * T_att is the prefetch window of Alg. 1.  Not part of the MoE layer; context-free.
 * Grouped-query decode attention of B tokens over a KV cache:
 *   out[b][h] = sum_s softmax_s(q[b][h] . k[b][s][h/G] / sqrt(dh)) v[b][s][h/G],  G = Hq / Hkv,
 * positions s < S of caches holding S_max positions.  Device pointers: q bf16 [B][Hq][dh],
 * k_cache / v_cache bf16 [B][S_max][Hkv][dh], out fp32 [B][Hq][dh], ws caller-owned scratch of
 * moepic_attention_ws_bytes bytes.  Enqueued on `stream` (cudaStream_t as void*).  EINVAL unless
 * dh == 128, Hq % Hkv == 0 with G in {1, 2, 4, 8, 16}, 1 <= S <= S_max <= 131072, B >= 1, pointers non-NULL
 * and 8-byte aligned, ws large enough; ERUNTIME if the launch fails.                          */
moepic_status moepic_attention_ws_bytes(int32_t B, int32_t S, int32_t Hq, int32_t Hkv, int32_t dh, size_t* bytes);
moepic_status moepic_attention_decode(const void* q, const void* k_cache, const void* v_cache, int32_t B,
                                      int32_t S, int32_t S_max, int32_t Hq, int32_t Hkv, int32_t dh,
                                      float* out, void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------------------------
 * Multi-GPU group (expert parallel; NEXT-4: tensor parallel along I).  The ranks
 * of one EP (ep_size > 1) or TP (tp_size > 1) layer form a group of G = ep_size or tp_size
 * <= 8 contexts, one per process and GPU.  The data plane is the library's: either
 *   MOEPIC_TRANSPORT_PEER: every rank's exchange region is mapped into every peer with CUDA IPC
 *     (P2P over NVLink / NVSwitch between GPUs; also works for ranks sharing one GPU), and the
 *     library's kernels store rows straight into the consumer's region and publish per-phase
 *     epoch flags (release / acquire at system scope);
 *   MOEPIC_TRANSPORT_NCCL: a communicator the library creates (ncclCommInitRank) from the
 *     unique id in rank 0's handle: ncclAllGather / grouped ncclSend-ncclRecv / ncclAllReduce
 *     on the compute stream (libnccl.so.2 is dlopened at join; NCCL refuses two ranks on one GPU).
 * Joining: every rank calls moepic_group_handle, the caller all-gathers the handles with its
 * own process group (torch.distributed: plumbing only), then every rank calls moepic_group_join
 * with the G handles in rank order (collective: all ranks must call it).  The handle is a
 * fixed-size opaque blob (*bytes = its size; query with out == NULL).  Blocking; EINVAL on
 * mismatched handles (world, transport, shapes), ERUNTIME on a CUDA / NCCL failure.
 * After a join, moepic_layer_forward on the group:
 *   - without MOEPIC_TOKENS_SHARDED (decode: every rank passes the SAME h, B <= 32): y_dev is the
 *     full layer output on every rank -- the partial outputs are summed over the group in rank
 *     order inside the call (identical bits on every rank);
 *   - with MOEPIC_TOKENS_SHARDED (EP only, n_shared == 0, no FUSE_PREDICT; rank r passes its own
 *     B tokens, the same B on every rank, G*B <= max_batch): rank r's tokens are global tokens
 *     [r*B, (r+1)*B).  The ranks route their own tokens, all-gather the routing (every control
 *     plane sees the whole batch: traces / stats as if one context ran G*B tokens with ep_rank),
 *     dispatch each token row once to every rank owning one of its experts, compute the
 *     sub-batch there (K2 or the tcgen05 prefill GEMMs), return each rank's weighted partial sum
 *     to the token's owner, and the owner adds them in rank order (+ h if MOEPIC_RESIDUAL).
 *     y_dev holds rank r's B output rows.  The trace's ids / w are rank r's tokens.            */
enum { MOEPIC_TRANSPORT_PEER = 0, MOEPIC_TRANSPORT_NCCL = 1 };
moepic_status moepic_group_handle(moepic_ctx* ctx, int32_t transport, void* out, size_t* bytes);
moepic_status moepic_group_join(moepic_ctx* ctx, const void* handles, size_t bytes_each);

/* Host-only (no context, no GPU): the exchange lists of the token-sharded EP layer for rank
 * `me` of G (the library computes the same lists inside layer_forward).  ids_all [G*Bl][K]
 * routed ids of the whole batch (rank-major), experts owned by rank e*G/N.  Caller-owned
 * outputs with the capacities below (any may be NULL); counts written to n_disp / n_sub:
 *   d_tok / d_dst / d_row [Bl*min(G,K)]: dispatch entries (my token, destination rank, row in
 *     the destination's sub-batch), grouped by destination, tokens ascending;
 *   sub / c_dst / c_row [G*Bl]: the sub-batch this rank computes (global tokens ascending), and
 *     for each of its rows the owner rank and the row in the owner's combine buffer;
 *   r_off [Bl+1], r_row [Bl*min(G,K)]: per own token, its combine-buffer rows (owner rank asc).
 * EINVAL on an id outside [0, N) or bad sizes.                                                  */
moepic_status moepic_ep_plan(int32_t N, int32_t K, int32_t G, int32_t me, int32_t Bl, const int32_t* ids_all,
                             int32_t* d_tok, int32_t* d_dst, int32_t* d_row, int32_t* n_disp,
                             int32_t* sub, int32_t* c_dst, int32_t* c_row, int32_t* n_sub,
                             int32_t* r_off, int32_t* r_row);

const char* moepic_last_error(const moepic_ctx* ctx);   /* never NULL; "" when none           */
void moepic_destroy(moepic_ctx* ctx);                    /* NULL is a no-op; syncs the device  */

#ifdef __cplusplus
}
#endif
#endif /* MOEPIC_H */
