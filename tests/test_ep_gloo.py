"""Expert-parallel path on CPU with torch.distributed gloo, world size 2.

Each rank runs the library's host control plane (moepic_hostsim, ep_rank / ep_size) and the
oracle's per-rank state machine on the same routing: per-rank traces must be bit-identical
(C-P16 "per-rank cache traces match the oracle run with G simulated ranks").  The decode combine
is an all-reduce of per-rank partial outputs: the sum over ranks of the oracle's partials
(routed experts owned by the rank + its rows of the shared experts) must equal the
single-device layer output (decomposition identity, C-P16)."""
import os
import socket
import zlib

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import synth
        from oracle import numeric as ON
        from oracle.replay import OracleEngine, CacheConfig
        from paper_2509_08342_b200 import api
        L, N, K, d, I = 2, 8, 2, 64, 128
        routers = [synth.bf16_bits(synth.router_weights(3, i, N, d)) for i in range(L)]
        experts = {(i, e): tuple(synth.bf16_bits(x) for x in synth.expert_weights(3, i, e, d, I))
                   for i in range(L) for e in range(N)}
        shared = {(i, s): tuple(synth.bf16_bits(x) for x in synth.shared_expert_weights(3, i, s, d, I))
                  for i in range(L) for s in range(1)}
        desc = api.model_desc(L, N, K, d, I, n_shared=1, row_granule=16, max_batch=2, v_e_max=8,
                              ep_rank=rank, ep_size=world)
        hs = api.HostSim(desc)
        orc = OracleEngine(L, N, K, d, I, row_granule=16, n_shared=1, ep_rank=rank, ep_size=world)
        cfg = dict(v_e=2.0, seed=4)
        a = hs.configure(**cfg)
        C, It, _, V = orc.configure(CacheConfig(**cfg))
        assert a["C_i"] == C and a["I_top_i"] == It
        H = synth.hidden_states(3, 12, L, d)
        worst = 0.0
        for t in range(12):
            for i in range(L):
                hb = synth.bf16_bits(H[t, i][None])
                y_full, ids, w, _ = ON.moe_layer(hb, routers[i], lambda e: experts[(i, e)], K,
                                                 shared=[shared[(i, 0)]])
                # routing is replicated: every rank derives identical ids
                g_ids = [torch.zeros_like(torch.from_numpy(ids)) for _ in range(world)]
                dist.all_gather(g_ids, torch.from_numpy(ids))
                assert all(torch.equal(g_ids[0], x) for x in g_ids)
                nxt = (i + 1) % L
                rank_next = ON.predicted_ranking(ON.router_logits(hb, routers[nxt]), K)
                x = hs.step(i, ids, nxt, rank_next)
                o = orc.step(i, ids, nxt, rank_next)
                assert x.act == o.act and x.adm == o.adm and x.plan == o.plan
                assert (x.pcie_ondemand, x.pcie_prefetch, x.hbm) == (o.pcie_ondemand, o.pcie_prefetch, o.hbm)
                assert all(e * world // N == rank for e, _ in x.act)
                part = torch.from_numpy(ON.moe_layer_ep_partial(hb, routers[i], lambda e: experts[(i, e)], K,
                                                                rank, world, shared=[shared[(i, 0)]]))
                dist.all_reduce(part)                         # the decode combine
                worst = max(worst, float(np.abs(part.numpy() - y_full).max() / np.abs(y_full).max()))
        assert worst < 1e-12, worst
        q.put((rank, "ok"))
    except Exception as e:   # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_ep_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


def _tp_worker(rank, world, port, q):
    """Tensor parallel along I: each rank's control plane works on its
    I / G rows of every expert.  Routing is replicated, so every rank must take the SAME cache
    decisions, and they must equal the oracle's state machine run on the I / G-row shape; the
    all-reduce of the per-rank partial outputs (oracle) must equal the single-device layer."""
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import synth
        from oracle import numeric as ON
        from oracle.replay import OracleEngine, CacheConfig
        from paper_2509_08342_b200 import api
        L, N, K, d, I = 2, 8, 2, 64, 128
        routers = [synth.bf16_bits(synth.router_weights(5, i, N, d)) for i in range(L)]
        experts = {(i, e): tuple(synth.bf16_bits(x) for x in synth.expert_weights(5, i, e, d, I))
                   for i in range(L) for e in range(N)}
        shared = {(i, 0): tuple(synth.bf16_bits(x) for x in synth.shared_expert_weights(5, i, 0, d, I))
                  for i in range(L)}
        desc = api.model_desc(L, N, K, d, I, n_shared=1, row_granule=16, max_batch=2, v_e_max=8,
                              tp_rank=rank, tp_size=world)
        hs = api.HostSim(desc)
        orc = OracleEngine(L, N, K, d, I // world, row_granule=16, n_shared=1)
        cfg = dict(v_e=3.0, theta_i=[0.5, 0.75], seed=2)
        a = hs.configure(**cfg)
        C, It, _, V = orc.configure(CacheConfig(**cfg))
        assert a["C_i"] == C and a["I_top_i"] == It
        H = synth.hidden_states(5, 12, L, d)
        worst = 0.0
        for t in range(12):
            for i in range(L):
                hb = synth.bf16_bits(H[t, i][None])
                y_full, ids, w, _ = ON.moe_layer(hb, routers[i], lambda e: experts[(i, e)], K,
                                                 shared=[shared[(i, 0)]])
                nxt = (i + 1) % L
                rank_next = ON.predicted_ranking(ON.router_logits(hb, routers[nxt]), K)
                x = hs.step(i, ids, nxt, rank_next)
                o = orc.step(i, ids, nxt, rank_next)
                assert x.act == o.act and x.adm == o.adm and x.plan == o.plan
                assert (x.pcie_ondemand, x.pcie_prefetch, x.hbm) == (o.pcie_ondemand, o.pcie_prefetch, o.hbm)
                # identical decisions on every rank
                tr = torch.tensor([zlib.crc32(repr((x.act, x.adm, x.plan)).encode())])
                g = [torch.zeros_like(tr) for _ in range(world)]
                dist.all_gather(g, tr)
                assert all(torch.equal(g[0], v) for v in g)
                part = torch.from_numpy(ON.moe_layer_tp_partial(hb, routers[i], lambda e: experts[(i, e)], K,
                                                                rank, world, shared=[shared[(i, 0)]]))
                dist.all_reduce(part)
                worst = max(worst, float(np.abs(part.numpy() - y_full).max() / np.abs(y_full).max()))
        assert worst < 1e-12, worst
        q.put((rank, "ok"))
    except Exception as e:   # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()[-1500:]))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_tp_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_tp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
