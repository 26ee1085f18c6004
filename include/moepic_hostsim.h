/* moepic_hostsim.h — the library's host control plane without a GPU.
 *
 * Exposes the exact C++ objects moepic_layer_forward / moepic_predict_prefetch / moepic_configure
 * drive (cache manager, classification, admission, prefetch planner, statistics, Alg. 1), fed
 * with routing decisions supplied by the caller instead of the router kernel.  It exists so
 * the control plane can be checked bit-for-bit against the oracle on a machine without a GPU
 * (tests/test_hostsim_vs_oracle.py).  No CUDA call is made by any function in this header.
 *
 * Argument conventions, errors and trace semantics are those of moepic.h.
 */
#ifndef MOEPIC_HOSTSIM_H
#define MOEPIC_HOSTSIM_H

#include "moepic.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct moepic_hostsim moepic_hostsim;

/* desc as for moepic_create (v_e_max sizes the simulated slot pool). */
moepic_status moepic_hostsim_create(const moepic_model_desc* desc, moepic_hostsim** out);

/* as moepic_configure. */
moepic_status moepic_hostsim_configure(moepic_hostsim* hs, const moepic_cache_config* cfg,
                                       moepic_config_out* out);

/* One layer step with routing supplied by the caller:
 *   ids: host [B][K] routed experts of layer `layer` in key order;
 *   ranking_next: host [N] predicted ranking R' for layer next_layer, or NULL (no prediction);
 *   next_layer: layer the plan targets (ignored when ranking_next is NULL).
 * trace receives act / adm / plan / byte fields (ids and w are not written).                 */
moepic_status moepic_hostsim_step(moepic_hostsim* hs, int32_t layer, const int32_t* ids, int32_t B,
                                  int32_t next_layer, const int32_t* ranking_next,
                                  moepic_trace* trace);

/* as moepic_predict_prefetch with the ranking supplied by the caller. */
moepic_status moepic_hostsim_predict(moepic_hostsim* hs, int32_t next_layer, const int32_t* ranking,
                                     moepic_trace* trace);

/* cached set of a layer: writes up to N expert ids (ascending) into out, count into *n. */
moepic_status moepic_hostsim_cached(moepic_hostsim* hs, int32_t layer, int32_t* out, int32_t* n);

/* as moepic_get_stats / moepic_set_stats (same snapshot format, interchangeable with a
 * context of the same (L, N, K)): statistics H/P/PH accumulators and the cache
 * counters mu / nu / last (Eq. 4).                                                  */
moepic_status moepic_hostsim_get_stats(moepic_hostsim* hs, void* buf, size_t* bytes);
moepic_status moepic_hostsim_set_stats(moepic_hostsim* hs, const void* buf, size_t bytes);

const char* moepic_hostsim_last_error(const moepic_hostsim* hs);
void moepic_hostsim_destroy(moepic_hostsim* hs);

#ifdef __cplusplus
}
#endif
#endif /* MOEPIC_HOSTSIM_H */
