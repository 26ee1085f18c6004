"""Tensor parallel along I through the C ABI with two ranks.

gpurun exposes one GPU, so both ranks share cuda:0, each with its own context holding rows
[r I / 2, (r+1) I / 2) of every routed and shared expert, and combine with a gloo all-reduce.
Each rank's partial output must match the oracle's share for its row slice, the sum must match
the single-device oracle layer within 2e-3 (MOEPIC_RESIDUAL adds h exactly once), and the
routing and cache traces must be identical on both ranks."""
import os
import socket
import zlib

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
        from oracle import numeric as ON
        from paper_2509_08342_b200 import api
        L, N, K, d, I = 2, 8, 2, 256, 512
        m = Model(L, N, K, d, I, n_shared=1, seed=23)
        expert, shared_of = m.expert, (lambda i, s: m.shared[(i, s)])
        if fmt:   # Q4G64: the oracle sees the dequantised experts (slicing rows commutes with it)
            from oracle import quant as Qz
            deq = {k: Qz.dequantize_expert(Qz.quantize_expert(*w)) for k, w in m.experts.items()}
            dsh = {k: Qz.dequantize_expert(Qz.quantize_expert(*w)) for k, w in m.shared.items()}
            expert, shared_of = (lambda i, e: deq[(i % m.L_host, e)]), (lambda i, s: dsh[(i, s)])
        desc = api.model_desc(L, N, K, d, I, n_shared=1, row_granule=64, max_batch=B, v_e_max=8.0,
                              tp_rank=rank, tp_size=world, weight_format=fmt)
        ctx = api.MoEpic(desc)
        m.load_into(ctx)
        cfg = ctx.configure(v_e=3.0, theta_i=[0.5, 0.5], seed=1)
        assert cfg["I_top_i"] == [128, 128]          # theta 0.5 of the 256-row local slice
        H = synth.hidden_states(23, 3 * B, L, d)
        worst_part = worst_sum = 0.0
        for t in range(3):
            for i in range(L):
                h = H[t * B:(t + 1) * B, i]
                hb = synth.bf16_bits(h)
                y = torch.empty(B, d, dtype=torch.float32, device="cuda")
                flags = api.M.FUSE_PREDICT | (api.M.RESIDUAL if t == 1 else 0)
                tr = ctx.layer_forward(i, h.cuda(), y, flags=flags)
                torch.cuda.synchronize()
                sig = torch.tensor([zlib.crc32(repr((tr.ids.tolist(), tr.act, tr.adm, tr.plan)).encode())])
                g = [torch.zeros_like(sig) for _ in range(world)]
                dist.all_gather(g, sig)
                assert all(torch.equal(g[0], v) for v in g), "ranks took different decisions"
                shared = [shared_of(i, s) for s in range(m.n_shared)]
                part = ON.moe_layer_tp_partial(hb, m.routers[i], lambda e: expert(i, e), K, rank, world,
                                               shared=shared)
                hres = ON.bf16_to_f64(hb) if (t == 1 and rank == 0) else 0.0
                yc = y.cpu()
                worst_part = max(worst_part, rel_err(yc.numpy(), part + hres))
                dist.all_reduce(yc)                          # the TP combine
                y_ref, _, _, _ = ON.moe_layer(hb, m.routers[i], lambda e: expert(i, e), K, shared=shared)
                if t == 1:
                    y_ref = y_ref + ON.bf16_to_f64(hb)
                worst_sum = max(worst_sum, rel_err(yc.numpy(), y_ref))
        assert worst_part <= TOL, worst_part
        assert worst_sum <= TOL, worst_sum
        ctx.close()
        q.put((rank, "ok"))
    except Exception:   # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()[-1500:]))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("B,fmt,gate", [(1, 0, 1), (5, 0, 1), (64, 0, 1), (1, 1, 1), (5, 1, 1), (1, 0, 2), (1, 1, 2)])
def test_tp_two_ranks_one_gpu(B, fmt, gate):
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
