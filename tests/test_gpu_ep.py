"""Expert-parallel decode and prefill through the C ABI with two ranks.

gpurun exposes one GPU, so both ranks share cuda:0 (each with its own context, arena and pinned
host arena) and combine with a gloo all-reduce.  Each rank owns experts e * 2 // N == rank and
half the shared-expert rows; the sum of the partial outputs must match the single-device oracle
within 2e-3, and the routing must be identical on both ranks."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, B, fmt=0, gate=1):
    try:
        os.environ["MOEPIC_K2_GATE"] = str(gate)   # read at create
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        import synth
        from gpu_model import Model, rel_err, TOL
        from paper_2509_08342_b200 import api
        L, N, K, d, I = 2, 8, 2, 256, 512
        m = Model(L, N, K, d, I, n_shared=1, seed=17)
        if fmt:   # Q4G64: the oracle sees the dequantised experts
            from oracle import quant as Qz
            from oracle import numeric as ON
            deq = {k: Qz.dequantize_expert(Qz.quantize_expert(*w)) for k, w in m.experts.items()}
            dsh = {k: Qz.dequantize_expert(Qz.quantize_expert(*w)) for k, w in m.shared.items()}
            m.oracle_layer = lambda i, hb: ON.moe_layer(hb, m.routers[i], lambda e: deq[(i % m.L_host, e)], K,
                                                        shared=[dsh[(i, s)] for s in range(m.n_shared)])
        desc = api.model_desc(L, N, K, d, I, n_shared=1, row_granule=64, max_batch=B, v_e_max=8.0,
                              ep_rank=rank, ep_size=world, weight_format=fmt)
        ctx = api.MoEpic(desc)
        m.load_into(ctx)
        ctx.configure(v_e=2.0, seed=1)
        H = synth.hidden_states(17, 3 * B, L, d)
        worst = 0.0
        for t in range(3):
            for i in range(L):
                h = H[t * B:(t + 1) * B, i]
                y = torch.empty(B, d, dtype=torch.float32, device="cuda")
                tr = ctx.layer_forward(i, h.cuda(), y, flags=api.M.FUSE_PREDICT)
                torch.cuda.synchronize()
                ids = torch.from_numpy(tr.ids.copy())
                g_ids = [torch.zeros_like(ids) for _ in range(world)]
                dist.all_gather(g_ids, ids)
                assert all(torch.equal(g_ids[0], x) for x in g_ids)
                assert all(e * world // N == rank for e, _ in tr.act)
                yc = y.cpu()
                dist.all_reduce(yc)                          # the EP combine
                y_ref, _, _, _ = m.oracle_layer(i, synth.bf16_bits(h))
                worst = max(worst, rel_err(yc.numpy(), y_ref))
        assert worst <= TOL, worst
        ctx.close()
        q.put((rank, "ok"))
    except Exception as e:   # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()[-1500:]))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("B,fmt,gate", [(1, 0, 1), (3, 0, 1), (64, 0, 1), (3, 1, 1), (1, 0, 2), (3, 0, 2)])
def test_ep_two_ranks_one_gpu(B, fmt, gate):
    """gate 2: every decode step runs the gated K2 launch (MOEPIC_K2_GATE=2)."""
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q, B, fmt, gate)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=600) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
