"""ctypes binding of include/moepic.h and include/moepic_hostsim.h — argument marshalling only.

Every function here has the name of the C entry point it calls; all work happens in
libmoepic.so (CUDA kernels for sm_100a + the C++ host control plane).  There is no Python or
CPU fallback: importing this module raises if the library is missing.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmoepic.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2509_08342_b200.build` "
                      "(there is no CPU fallback)")
lib = C.CDLL(LIB_PATH)

OK, EINVAL, ERUNTIME, ENOMEM, ESTATE = 0, 1, 2, 3, 4
LCP, LRU, LFU, RND = 0, 1, 2, 3
ALPHA, BETA, GAMMA = 0, 1, 2
ADM_FREE_SLOT, ADM_NONE = -1, -2
FUSE_PREDICT, RESIDUAL, TOKENS_SHARDED = 1, 2, 4
TRANSPORT_PEER, TRANSPORT_NCCL = 0, 1
BF16, Q4G64 = 0, 1

_i32p = C.POINTER(C.c_int32)
_f32p = C.POINTER(C.c_float)
_f64p = C.POINTER(C.c_double)
_i8p = C.POINTER(C.c_int8)
_u16p = C.POINTER(C.c_uint16)


class moepic_model_desc(C.Structure):
    _fields_ = [("L", C.c_int32), ("N", C.c_int32), ("K", C.c_int32), ("d", C.c_int32), ("I", C.c_int32),
                ("n_shared", C.c_int32), ("row_granule", C.c_int32), ("buffer_experts", C.c_int32),
                ("max_batch", C.c_int32), ("renorm_topk", C.c_int32), ("L_host", C.c_int32),
                ("v_e_max", C.c_double), ("ep_rank", C.c_int32), ("ep_size", C.c_int32),
                ("tp_rank", C.c_int32), ("tp_size", C.c_int32), ("weight_format", C.c_int32)]


class moepic_cache_config(C.Structure):
    _fields_ = [("v_e", C.c_double), ("v_i", _f64p), ("theta_i", _f64p), ("use_solver", C.c_int32),
                ("policy", C.c_int32), ("rho", C.c_double), ("omega", C.c_int32), ("zeta", C.c_double),
                ("t_att", C.c_double), ("t_moe", C.c_double), ("t_head", C.c_double),
                ("t_load_exp", C.c_double), ("y_cap_i", _i32p), ("prefetch", C.c_int32),
                ("seed", C.c_uint64), ("cancel_prefetch", C.c_int32), ("prefetch_rows_i", C.POINTER(C.c_int64))]


class moepic_config_out(C.Structure):
    _fields_ = [("C_i", _i32p), ("I_top_i", _i32p), ("theta_eff_i", _f64p), ("V_i", _f64p)]


class moepic_trace(C.Structure):
    _fields_ = [("ids", _i32p), ("w", _f32p),
                ("act_expert", _i32p), ("act_class", _i8p), ("n_act", C.c_int32),
                ("adm_expert", _i32p), ("adm_victim", _i32p), ("n_adm", C.c_int32),
                ("plan_expert", _i32p), ("plan_full", _i8p), ("n_plan", C.c_int32),
                ("plan_layer", C.c_int32),
                ("pcie_ondemand_bytes", C.c_uint64), ("pcie_prefetch_bytes", C.c_uint64),
                ("hbm_bytes", C.c_uint64), ("kernel_launches", C.c_int32), ("ranking", _i32p)]


class moepic_counters(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "layer_steps", "kernel_launches", "h2d_copies", "pcie_ondemand_bytes", "pcie_prefetch_bytes",
        "hbm_bytes", "act_alpha", "act_beta", "act_gamma", "pred_hits", "pred_total",
        "pcie_prefetch_planned_bytes")]


class moepic_kernel_stats(C.Structure):
    _fields_ = [("launches", C.c_uint64), ("total_ms", C.c_double), ("bytes", C.c_uint64),
                ("kernel_ms", C.c_double)]


KERNEL_ROUTER, KERNEL_EXPERT, KERNEL_COMBINE, KERNEL_GEMM = 0, 1, 2, 3
PROFILE_CLASSES = 0x100   # moepic_profile: time only the classes whose bits are set

_ctxp = C.c_void_p
_sig = {
    "moepic_arena_bytes": (C.c_int, [C.POINTER(moepic_model_desc), C.POINTER(C.c_size_t)]),
    "moepic_create": (C.c_int, [C.POINTER(moepic_model_desc), C.c_void_p, C.c_size_t, C.POINTER(_ctxp)]),
    "moepic_pack_expert": (C.c_int, [C.POINTER(moepic_model_desc), _u16p, _u16p, _u16p, C.c_void_p,
                                     C.POINTER(C.c_size_t)]),
    "moepic_load_router": (C.c_int, [_ctxp, C.c_int32, _u16p]),
    "moepic_load_expert": (C.c_int, [_ctxp, C.c_int32, C.c_int32, _u16p, _u16p, _u16p]),
    "moepic_configure": (C.c_int, [_ctxp, C.POINTER(moepic_cache_config), C.POINTER(moepic_config_out)]),
    "moepic_layer_forward": (C.c_int, [_ctxp, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                       C.c_uint32, C.POINTER(moepic_trace)]),
    "moepic_layer_forward_host": (C.c_int, [_ctxp, C.c_int32, _u16p, C.c_int32, _f32p, C.c_void_p,
                                            C.c_uint32, C.POINTER(moepic_trace)]),
    "moepic_predict_prefetch": (C.c_int, [_ctxp, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p,
                                          C.POINTER(moepic_trace)]),
    "moepic_get_stats": (C.c_int, [_ctxp, C.c_void_p, C.POINTER(C.c_size_t)]),
    "moepic_set_stats": (C.c_int, [_ctxp, C.c_void_p, C.c_size_t]),
    "moepic_get_counters": (C.c_int, [_ctxp, C.POINTER(moepic_counters)]),
    "moepic_profile": (C.c_int, [_ctxp, C.c_int32]),
    "moepic_profile_read": (C.c_int, [_ctxp, C.c_int32, C.POINTER(moepic_kernel_stats)]),
    "moepic_attention_ws_bytes": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                            C.POINTER(C.c_size_t)]),
    "moepic_attention_decode": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                          C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_size_t,
                                          C.c_void_p]),
    "moepic_group_handle": (C.c_int, [_ctxp, C.c_int32, C.c_void_p, C.POINTER(C.c_size_t)]),
    "moepic_group_join": (C.c_int, [_ctxp, C.c_void_p, C.c_size_t]),
    "moepic_ep_plan": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _i32p,
                                 _i32p, _i32p, _i32p, _i32p, _i32p, _i32p, _i32p, _i32p, _i32p, _i32p]),
    "moepic_last_error": (C.c_char_p, [_ctxp]),
    "moepic_destroy": (None, [_ctxp]),
    "moepic_hostsim_create": (C.c_int, [C.POINTER(moepic_model_desc), C.POINTER(_ctxp)]),
    "moepic_hostsim_configure": (C.c_int, [_ctxp, C.POINTER(moepic_cache_config), C.POINTER(moepic_config_out)]),
    "moepic_hostsim_step": (C.c_int, [_ctxp, C.c_int32, _i32p, C.c_int32, C.c_int32, _i32p,
                                      C.POINTER(moepic_trace)]),
    "moepic_hostsim_predict": (C.c_int, [_ctxp, C.c_int32, _i32p, C.POINTER(moepic_trace)]),
    "moepic_hostsim_cached": (C.c_int, [_ctxp, C.c_int32, _i32p, _i32p]),
    "moepic_hostsim_last_error": (C.c_char_p, [_ctxp]),
    "moepic_hostsim_get_stats": (C.c_int, [_ctxp, C.c_void_p, C.POINTER(C.c_size_t)]),
    "moepic_hostsim_set_stats": (C.c_int, [_ctxp, C.c_void_p, C.c_size_t]),
    "moepic_hostsim_destroy": (None, [_ctxp]),
}

for _name, (_res, _args) in _sig.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args
    globals()[_name] = _f

EXPORTED = tuple(_sig)
