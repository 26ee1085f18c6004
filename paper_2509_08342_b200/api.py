"""Thin Python wrappers over the C ABI (marshalling of torch / numpy buffers only).

`MoEpic` wraps one moepic_ctx (one GPU); `HostSim` wraps the GPU-free control plane.  No
arithmetic of the method happens here — every step runs in libmoepic.so.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _moepic as M


class MoEpicError(RuntimeError):
    pass


def _check(st, who, errfn=None, h=None):
    if st != M.OK:
        msg = errfn(h).decode() if (errfn and h) else ""
        raise MoEpicError(f"{who} failed with status {st}: {msg}")


def _ptr(a, t):
    return a.ctypes.data_as(C.POINTER(t)) if a is not None else None


def model_desc(L, N, K, d, I, n_shared=0, row_granule=64, buffer_experts=None, max_batch=1,
               renorm_topk=1, L_host=None, v_e_max=None, ep_rank=0, ep_size=1, tp_rank=0, tp_size=1,
               weight_format=0):
    """Model shape (include/moepic.h moepic_model_desc).  With tp_size > 1 the context holds rows
    [tp_rank*I/tp_size, (tp_rank+1)*I/tp_size) of every expert; v_e_max is then in units of that
    local slice, and load_expert still takes the full HF tensors.  weight_format = M.Q4G64 stores
    the experts as 4-bit group-quantised rows (include/moepic.h)."""
    return M.moepic_model_desc(L=L, N=N, K=K, d=d, I=I, n_shared=n_shared, row_granule=row_granule,
                               buffer_experts=K if buffer_experts is None else buffer_experts,
                               max_batch=max_batch, renorm_topk=renorm_topk,
                               L_host=L if L_host is None else L_host,
                               v_e_max=float(L * N if v_e_max is None else v_e_max),
                               ep_rank=ep_rank, ep_size=ep_size, tp_rank=tp_rank, tp_size=tp_size,
                               weight_format=weight_format)


def pack_expert(desc, gate_bits, up_bits, down_bits) -> np.ndarray:
    """moepic_pack_expert: the library's stored image of one expert ([rows][row bytes] uint8)."""
    g = np.ascontiguousarray(gate_bits, dtype=np.uint16)
    u = np.ascontiguousarray(up_bits, dtype=np.uint16)
    dn = np.ascontiguousarray(down_bits, dtype=np.uint16)
    n = C.c_size_t()
    _check(M.moepic_pack_expert(C.byref(desc), _ptr(g, C.c_uint16), _ptr(u, C.c_uint16), _ptr(dn, C.c_uint16),
                                None, C.byref(n)), "moepic_pack_expert")
    out = np.zeros(n.value, np.uint8)
    _check(M.moepic_pack_expert(C.byref(desc), _ptr(g, C.c_uint16), _ptr(u, C.c_uint16), _ptr(dn, C.c_uint16),
                                out.ctypes.data_as(C.c_void_p), C.byref(n)), "moepic_pack_expert")
    return out


def ep_plan(N, K, G, me, Bl, ids_all):
    """moepic_ep_plan: the token-sharded EP exchange lists of rank `me` (include/moepic.h)."""
    ids = np.ascontiguousarray(ids_all, dtype=np.int32).reshape(G * Bl, K)
    cd, cs = Bl * min(G, K), G * Bl
    a = {k: np.zeros(n, np.int32) for k, n in (("d_tok", cd), ("d_dst", cd), ("d_row", cd), ("sub", cs),
                                                ("c_dst", cs), ("c_row", cs), ("r_off", Bl + 1), ("r_row", cd))}
    nd, ns = C.c_int32(), C.c_int32()
    _check(M.moepic_ep_plan(N, K, G, me, Bl, _ptr(ids, C.c_int32), _ptr(a["d_tok"], C.c_int32),
                            _ptr(a["d_dst"], C.c_int32), _ptr(a["d_row"], C.c_int32), C.byref(nd),
                            _ptr(a["sub"], C.c_int32), _ptr(a["c_dst"], C.c_int32), _ptr(a["c_row"], C.c_int32),
                            C.byref(ns), _ptr(a["r_off"], C.c_int32), _ptr(a["r_row"], C.c_int32)), "moepic_ep_plan")
    for k in ("d_tok", "d_dst", "d_row"):
        a[k] = a[k][:nd.value]
    for k in ("sub", "c_dst", "c_row"):
        a[k] = a[k][:ns.value]
    a["r_row"] = a["r_row"][:a["r_off"][-1]]
    return a


class _Cfg:
    """Keeps the numpy arrays behind a moepic_cache_config alive."""

    def __init__(self, L, v_e, v_i=None, theta_i=None, use_solver=False, policy=M.LCP, rho=0.25,
                 omega=128, zeta=0.01, t_att=0.0, t_moe=0.0, t_head=0.0, t_load_exp=0.0, y_cap_i=None,
                 prefetch=True, seed=0, cancel_prefetch=True, prefetch_rows_i=None):
        self.v_i = None if v_i is None else np.ascontiguousarray(v_i, dtype=np.float64)
        self.th = None if theta_i is None else np.ascontiguousarray(theta_i, dtype=np.float64)
        self.yc = None if y_cap_i is None else np.ascontiguousarray(y_cap_i, dtype=np.int32)
        self.pw = None if prefetch_rows_i is None else np.ascontiguousarray(prefetch_rows_i, dtype=np.int64)
        self.c = M.moepic_cache_config(
            v_e=float(v_e), v_i=_ptr(self.v_i, C.c_double), theta_i=_ptr(self.th, C.c_double),
            use_solver=int(use_solver), policy=int(policy), rho=float(rho), omega=int(omega),
            zeta=float(zeta), t_att=float(t_att), t_moe=float(t_moe), t_head=float(t_head),
            t_load_exp=float(t_load_exp), y_cap_i=_ptr(self.yc, C.c_int32), prefetch=int(prefetch),
            seed=int(seed), cancel_prefetch=int(cancel_prefetch), prefetch_rows_i=_ptr(self.pw, C.c_int64))
        self.C_i = np.zeros(L, np.int32)
        self.I_top = np.zeros(L, np.int32)
        self.theta_eff = np.zeros(L, np.float64)
        self.V_i = np.zeros(L, np.float64)
        self.out = M.moepic_config_out(_ptr(self.C_i, C.c_int32), _ptr(self.I_top, C.c_int32),
                                       _ptr(self.theta_eff, C.c_double), _ptr(self.V_i, C.c_double))

    def result(self):
        return dict(C_i=self.C_i.tolist(), I_top_i=self.I_top.tolist(), theta_eff_i=self.theta_eff.tolist(),
                    V_i=self.V_i.tolist())


@dataclass
class Trace:
    ids: np.ndarray = None
    w: np.ndarray = None
    act: list = field(default_factory=list)      # [(expert, class)]
    adm: list = field(default_factory=list)      # [(expert, victim)]
    plan: list = field(default_factory=list)     # [(expert, full)]
    plan_layer: int = -1
    pcie_ondemand: int = 0
    pcie_prefetch: int = 0
    hbm: int = 0
    launches: int = 0
    ranking: np.ndarray = None


class _TraceBuf:
    def __init__(self, N, BK):
        self.ids = np.zeros(max(BK, 1), np.int32)
        self.w = np.zeros(max(BK, 1), np.float32)
        self.ae = np.zeros(N, np.int32)
        self.ac = np.zeros(N, np.int8)
        self.me = np.zeros(N, np.int32)
        self.mv = np.zeros(N, np.int32)
        self.pe = np.zeros(N, np.int32)
        self.pf = np.zeros(N, np.int8)
        self.rk = np.zeros(N, np.int32)
        self.t = M.moepic_trace(ids=_ptr(self.ids, C.c_int32), w=_ptr(self.w, C.c_float),
                                act_expert=_ptr(self.ae, C.c_int32), act_class=_ptr(self.ac, C.c_int8),
                                adm_expert=_ptr(self.me, C.c_int32), adm_victim=_ptr(self.mv, C.c_int32),
                                plan_expert=_ptr(self.pe, C.c_int32), plan_full=_ptr(self.pf, C.c_int8),
                                ranking=_ptr(self.rk, C.c_int32))

    def result(self, B, K):
        t = self.t
        return Trace(ids=self.ids[:B * K].reshape(B, K).copy(), w=self.w[:B * K].reshape(B, K).copy(),
                     act=[(int(self.ae[i]), int(self.ac[i])) for i in range(t.n_act)],
                     adm=[(int(self.me[i]), int(self.mv[i])) for i in range(t.n_adm)],
                     plan=[(int(self.pe[i]), bool(self.pf[i])) for i in range(t.n_plan)],
                     plan_layer=int(t.plan_layer), pcie_ondemand=int(t.pcie_ondemand_bytes),
                     pcie_prefetch=int(t.pcie_prefetch_bytes), hbm=int(t.hbm_bytes),
                     launches=int(t.kernel_launches),
                     ranking=self.rk.copy() if t.plan_layer >= 0 else None)


class MoEpic:
    """One library context on the current CUDA device.  Device memory for the arena is a torch
    uint8 tensor (PyTorch is plumbing for memory and streams only)."""

    def __init__(self, desc: M.moepic_model_desc, device=None):
        import torch
        self.desc = desc
        nbytes = C.c_size_t()
        _check(M.moepic_arena_bytes(C.byref(desc), C.byref(nbytes)), "moepic_arena_bytes")
        self.arena = torch.empty(int(nbytes.value) + 256, dtype=torch.uint8, device=device or "cuda")
        base = self.arena.data_ptr()
        aligned = (base + 255) // 256 * 256
        self.h = C.c_void_p()
        _check(M.moepic_create(C.byref(desc), C.c_void_p(aligned), int(nbytes.value), C.byref(self.h)),
               "moepic_create")
        self._tb = _TraceBuf(desc.N, desc.max_batch * desc.K)

    def close(self):
        if self.h:
            M.moepic_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _err(self, st, who):
        _check(st, who, M.moepic_last_error, self.h)

    def load_router(self, layer, w_bits: np.ndarray):
        a = np.ascontiguousarray(w_bits, dtype=np.uint16)
        self._err(M.moepic_load_router(self.h, layer, _ptr(a, C.c_uint16)), "moepic_load_router")

    def load_expert(self, layer, expert, gate_bits, up_bits, down_bits):
        g = np.ascontiguousarray(gate_bits, dtype=np.uint16)
        u = np.ascontiguousarray(up_bits, dtype=np.uint16)
        dn = np.ascontiguousarray(down_bits, dtype=np.uint16)
        self._err(M.moepic_load_expert(self.h, layer, expert, _ptr(g, C.c_uint16), _ptr(u, C.c_uint16),
                                       _ptr(dn, C.c_uint16)), "moepic_load_expert")

    def configure(self, **kw):
        cfg = _Cfg(self.desc.L, **kw)
        self._err(M.moepic_configure(self.h, C.byref(cfg.c), C.byref(cfg.out)), "moepic_configure")
        return cfg.result()

    def layer_forward(self, layer, h, y, stream=None, flags=0, trace=True):
        """h: torch bf16 [B][d] cuda; y: torch fp32 [B][d] cuda; stream: torch.cuda.Stream or None."""
        B = h.shape[0]
        sp = C.c_void_p(stream.cuda_stream if stream is not None else None)
        tp = C.byref(self._tb.t) if trace else None
        self._err(M.moepic_layer_forward(self.h, layer, C.c_void_p(h.data_ptr()), B, C.c_void_p(y.data_ptr()),
                                         sp, flags, tp), "moepic_layer_forward")
        return self._tb.result(B, self.desc.K) if trace else None

    def layer_forward_host(self, layer, h_bits: np.ndarray, stream=None, flags=0, trace=True):
        a = np.ascontiguousarray(h_bits, dtype=np.uint16)
        B = a.shape[0]
        y = np.empty((B, self.desc.d), np.float32)   # fully written by the call
        sp = C.c_void_p(stream.cuda_stream if stream is not None else None)
        tp = C.byref(self._tb.t) if trace else None
        self._err(M.moepic_layer_forward_host(self.h, layer, _ptr(a, C.c_uint16), B, _ptr(y, C.c_float), sp,
                                              flags, tp), "moepic_layer_forward_host")
        return y, (self._tb.result(B, self.desc.K) if trace else None)

    def predict_prefetch(self, next_layer, h, stream=None, trace=True):
        B = h.shape[0]
        sp = C.c_void_p(stream.cuda_stream if stream is not None else None)
        tp = C.byref(self._tb.t) if trace else None
        self._err(M.moepic_predict_prefetch(self.h, next_layer, C.c_void_p(h.data_ptr()), B, sp, tp),
                  "moepic_predict_prefetch")
        return self._tb.result(0, self.desc.K) if trace else None

    def counters(self):
        c = M.moepic_counters()
        self._err(M.moepic_get_counters(self.h, C.byref(c)), "moepic_get_counters")
        return {n: int(getattr(c, n)) for n, _ in M.moepic_counters._fields_}

    def profile(self, enable=True):
        self._err(M.moepic_profile(self.h, int(enable)), "moepic_profile")

    def profile_read(self, kernel_class):
        k = M.moepic_kernel_stats()
        self._err(M.moepic_profile_read(self.h, kernel_class, C.byref(k)), "moepic_profile_read")
        return dict(launches=int(k.launches), total_ms=float(k.total_ms), bytes=int(k.bytes),
                    kernel_ms=float(k.kernel_ms))

    def group_handle(self, transport=M.TRANSPORT_PEER) -> bytes:
        """moepic_group_handle: this rank's opaque handle (exchange region IPC handle, NCCL id)."""
        n = C.c_size_t()
        self._err(M.moepic_group_handle(self.h, transport, None, C.byref(n)), "moepic_group_handle")
        buf = C.create_string_buffer(n.value)
        self._err(M.moepic_group_handle(self.h, transport, buf, C.byref(n)), "moepic_group_handle")
        return buf.raw

    def group_join(self, handles):
        """moepic_group_join with the G handles in rank order (collective)."""
        blob = b"".join(handles)
        buf = C.create_string_buffer(blob, len(blob))
        self._err(M.moepic_group_join(self.h, buf, len(handles[0])), "moepic_group_join")

    def join_process_group(self, transport=M.TRANSPORT_PEER, group=None):
        """Exchange handles over an initialised torch.distributed process group (plumbing), then
        join.  The group's rank order must match ep_rank / tp_rank."""
        import torch
        import torch.distributed as dist
        mine = self.group_handle(transport)
        out = [None] * dist.get_world_size(group)
        dist.all_gather_object(out, mine, group=group)
        self.group_join(out)

    def get_stats(self) -> bytes:
        n = C.c_size_t()
        self._err(M.moepic_get_stats(self.h, None, C.byref(n)), "moepic_get_stats")
        buf = C.create_string_buffer(n.value)
        self._err(M.moepic_get_stats(self.h, buf, C.byref(n)), "moepic_get_stats")
        return buf.raw

    def set_stats(self, blob: bytes):
        buf = C.create_string_buffer(blob, len(blob))
        self._err(M.moepic_set_stats(self.h, buf, len(blob)), "moepic_set_stats")


class HostSim:
    """The library's host control plane fed with caller-supplied routing (no GPU)."""

    def __init__(self, desc: M.moepic_model_desc):
        self.desc = desc
        self.h = C.c_void_p()
        _check(M.moepic_hostsim_create(C.byref(desc), C.byref(self.h)), "moepic_hostsim_create")
        self._tb = _TraceBuf(desc.N, 0)

    def __del__(self):
        try:
            if self.h:
                M.moepic_hostsim_destroy(self.h)
        except Exception:
            pass

    def _err(self, st, who):
        _check(st, who, M.moepic_hostsim_last_error, self.h)

    def configure(self, **kw):
        cfg = _Cfg(self.desc.L, **kw)
        self._err(M.moepic_hostsim_configure(self.h, C.byref(cfg.c), C.byref(cfg.out)), "moepic_hostsim_configure")
        return cfg.result()

    def step(self, layer, ids, next_layer=None, ranking_next=None):
        a = np.ascontiguousarray(ids, dtype=np.int32)
        B = a.shape[0]
        r = None if ranking_next is None else np.ascontiguousarray(ranking_next, dtype=np.int32)
        self._err(M.moepic_hostsim_step(self.h, layer, _ptr(a, C.c_int32), B,
                                        -1 if next_layer is None else next_layer, _ptr(r, C.c_int32),
                                        C.byref(self._tb.t)), "moepic_hostsim_step")
        return self._tb.result(0, self.desc.K)

    def predict(self, next_layer, ranking):
        r = np.ascontiguousarray(ranking, dtype=np.int32)
        self._err(M.moepic_hostsim_predict(self.h, next_layer, _ptr(r, C.c_int32), C.byref(self._tb.t)),
                  "moepic_hostsim_predict")
        return self._tb.result(0, self.desc.K)

    def get_stats(self) -> bytes:
        n = C.c_size_t()
        self._err(M.moepic_hostsim_get_stats(self.h, None, C.byref(n)), "moepic_hostsim_get_stats")
        buf = C.create_string_buffer(n.value)
        self._err(M.moepic_hostsim_get_stats(self.h, buf, C.byref(n)), "moepic_hostsim_get_stats")
        return buf.raw

    def set_stats(self, blob: bytes):
        buf = C.create_string_buffer(blob, len(blob))
        self._err(M.moepic_hostsim_set_stats(self.h, buf, len(blob)), "moepic_hostsim_set_stats")

    def cached(self, layer):
        out = np.zeros(self.desc.N, np.int32)
        n = C.c_int32()
        self._err(M.moepic_hostsim_cached(self.h, layer, _ptr(out, C.c_int32), C.byref(n)), "moepic_hostsim_cached")
        return set(out[:n.value].tolist())


class Attention:
    """moepic_attention_decode (attention stand-in) with its scratch held in a
    torch tensor.  q bf16 [B][Hq][128], caches bf16 [B][S_max][Hkv][128] (cuda)."""

    def __init__(self, B, S_max, Hq, Hkv, dh=128, device="cuda"):
        import torch
        n = C.c_size_t()
        _check(M.moepic_attention_ws_bytes(B, S_max, Hq, Hkv, dh, C.byref(n)), "moepic_attention_ws_bytes")
        self.ws = torch.empty(int(n.value), dtype=torch.uint8, device=device)
        self.B, self.S_max, self.Hq, self.Hkv, self.dh = B, S_max, Hq, Hkv, dh

    def __call__(self, q, k_cache, v_cache, S, out, stream=None):
        sp = C.c_void_p(stream.cuda_stream if stream is not None else None)
        _check(M.moepic_attention_decode(C.c_void_p(q.data_ptr()), C.c_void_p(k_cache.data_ptr()),
                                         C.c_void_p(v_cache.data_ptr()), q.shape[0], S, k_cache.shape[1],
                                         self.Hq, self.Hkv, self.dh, C.c_void_p(out.data_ptr()),
                                         C.c_void_p(self.ws.data_ptr()), self.ws.numel(), sp),
               "moepic_attention_decode")
        return out
