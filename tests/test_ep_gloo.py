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


# ------------------------------------------------------------------ token-sharded EP exchange
def _emulate_sharded(N, K, d, I, G, Bl, seed):
    """Drive the library's exchange lists (moepic_ep_plan, one call per rank) through an
    emulated data plane: dispatch rows into per-rank receive buffers at the listed rows, compute
    each rank's sub-batch with the oracle's EP partial (its own experts only), return the rows to
    the listed combine-buffer rows, reduce in list order.  Must equal the dense oracle layer."""
    import synth
    from oracle import numeric as ON
    from paper_2509_08342_b200 import api
    router = synth.bf16_bits(synth.router_weights(seed, 0, N, d, 2.0))
    experts = {e: tuple(synth.bf16_bits(x) for x in synth.expert_weights(seed, 0, e, d, I)) for e in range(N)}
    T = G * Bl
    hb = synth.bf16_bits(synth.batch_hidden(seed, T, d))
    y_full, ids_all, _, _ = ON.moe_layer(hb, router, experts, K)
    lists = [api.ep_plan(N, K, G, r, Bl, ids_all) for r in range(G)]
    # every token reaches every rank owning one of its experts exactly once
    for t in range(T):
        owners = sorted({int(e) * G // N for e in ids_all[t]})
        assert [q for q in range(G) if t in set(lists[q]["sub"].tolist())] == owners
    recv = [np.full((len(lists[q]["sub"]), d), -1, np.int64) for q in range(G)]
    for r in range(G):
        for tok, q, row in zip(lists[r]["d_tok"], lists[r]["d_dst"], lists[r]["d_row"]):
            recv[q][row] = r * Bl + tok           # token index stands in for its row
    comb = [np.full((int(lists[p]["r_off"][-1]), d), np.nan) for p in range(G)]
    for q in range(G):
        L = lists[q]
        assert np.array_equal(recv[q][:, 0], L["sub"])    # rows landed in S_q order
        ysub = ON.moe_layer_ep_partial(hb[L["sub"]], router, experts, K, q, G) if len(L["sub"]) else np.zeros((0, d))
        for j, (p, row) in enumerate(zip(L["c_dst"], L["c_row"])):
            assert np.isnan(comb[p][row]).all()            # no row written twice
            comb[p][row] = ysub[j]
    y = np.zeros((T, d))
    for p in range(G):
        L = lists[p]
        assert not np.isnan(comb[p]).any()                 # every combine row filled
        for i in range(Bl):
            for r in L["r_row"][L["r_off"][i]:L["r_off"][i + 1]]:
                y[p * Bl + i] += comb[p][r]
    return float(np.abs(y - y_full).max() / np.abs(y_full).max())


@pytest.mark.parametrize("G,N,K,Bl", [(2, 8, 2, 5), (4, 8, 2, 7), (8, 64, 6, 3), (4, 128, 8, 4), (8, 8, 2, 16)])
def test_sharded_ep_lists_emulated(G, N, K, Bl):
    assert _emulate_sharded(N, K, 64, 64, G, Bl, seed=G * 100 + Bl) < 1e-12


def _sendrecv(recv, send, rank, world):
    """Grouped point-to-point exchange (the NCCL transport's ncclSend / ncclRecv pairs)."""
    reqs = []
    for p in range(world):
        if p == rank:
            recv[p].copy_(send[p])
            continue
        if send[p].numel():
            reqs.append(dist.isend(send[p].contiguous(), p))
        if recv[p].numel():
            reqs.append(dist.irecv(recv[p], p))
    for r in reqs:
        r.wait()


def _sharded_worker(rank, world, port, q):
    """world-2 gloo: each rank derives ITS lists from the library, then the exchange runs as two
    grouped send / recv rounds (dispatch rows, combine rows) with the NCCL transport's counts."""
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import synth
        from oracle import numeric as ON
        from paper_2509_08342_b200 import api
        N, K, d, I, Bl = 8, 2, 64, 128, 6
        router = synth.bf16_bits(synth.router_weights(9, 0, N, d, 2.0))
        experts = {e: tuple(synth.bf16_bits(x) for x in synth.expert_weights(9, 0, e, d, I)) for e in range(N)}
        hb_all = synth.bf16_bits(synth.batch_hidden(9, world * Bl, d))
        mine = hb_all[rank * Bl:(rank + 1) * Bl]
        # each rank routes its own tokens; the routing is all-gathered
        _, ids_mine, _, _ = ON.moe_layer(mine, router, experts, K)
        g = [torch.zeros(Bl, K, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(g, torch.from_numpy(ids_mine.astype(np.int32)))
        ids_all = torch.cat(g).numpy()
        L = api.ep_plan(N, K, world, rank, Bl, ids_all)
        # dispatch: rows grouped by destination (entry order), counts per destination
        send_cnt = [int((L["d_dst"] == q2).sum()) for q2 in range(world)]
        h64 = torch.from_numpy(mine.astype(np.int64))
        send = [h64[torch.from_numpy(L["d_tok"][L["d_dst"] == q2].astype(np.int64))] for q2 in range(world)]
        recv = [torch.zeros(int((L["sub"] // Bl == p).sum()), d, dtype=torch.int64) for p in range(world)]
        _sendrecv(recv, send, rank, world)
        hsub = torch.cat(recv).numpy().astype(np.uint16)
        assert np.array_equal(hsub, hb_all[L["sub"]])
        ysub = torch.from_numpy(ON.moe_layer_ep_partial(hsub, router, experts, K, rank, world))
        # combine: my sub rows go back grouped by owner (sub is in owner order)
        back = [ysub[torch.from_numpy(np.nonzero(L["c_dst"] == p)[0])] for p in range(world)]
        comb_in = [torch.zeros(send_cnt[q2], d, dtype=torch.float64) for q2 in range(world)]
        _sendrecv(comb_in, back, rank, world)
        comb = torch.cat(comb_in).numpy()
        y = np.zeros((Bl, d))
        for i in range(Bl):
            for r in L["r_row"][L["r_off"][i]:L["r_off"][i + 1]]:
                y[i] += comb[r]
        y_ref, _, _, _ = ON.moe_layer(mine, router, experts, K)
        err = float(np.abs(y - y_ref).max() / np.abs(y_ref).max())
        assert err < 1e-12, err
        q.put((rank, "ok"))
    except Exception:   # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()[-1500:]))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_sharded_ep_world2_gloo_sendrecv():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_sharded_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
