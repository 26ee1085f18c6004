"""GPU parity tests (T2-T4 of SURVEY §4): the CUDA path through the C ABI vs the oracle.

Bar (BASELINE north_star): routing ids, predicted rankings and cache traces bit-exact;
gate weights within 1e-6; layer outputs max|gpu-ref|/max|ref| <= 2e-3.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import numeric as ON
from oracle.replay import OracleEngine, CacheConfig
from gpu_model import Model, rel_err, TOL

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    from paper_2509_08342_b200 import build
    build.build()


def _api():
    from paper_2509_08342_b200 import api
    return api


def _ctx(model, max_batch=1, v_e_max=None, renorm=1, g=64, Ub=None):
    api = _api()
    desc = api.model_desc(model.L, model.N, model.K, model.d, model.I, n_shared=model.n_shared,
                          row_granule=g, buffer_experts=Ub, max_batch=max_batch, renorm_topk=renorm,
                          L_host=model.L_host, v_e_max=v_e_max if v_e_max is not None else model.L * model.N)
    ctx = api.MoEpic(desc)
    model.load_into(ctx)
    return ctx


def _replay(model, ctx, orc, h_tokens, flags, renorm=True, check_y=True, predict_first=False):
    """Run tokens x layers through both; compare traces bit-exactly and y within TOL."""
    api = _api()
    L, K = model.L, model.K
    worst = 0.0
    stream = torch.cuda.Stream()
    for t, hl in enumerate(h_tokens):            # hl: [L][B][d] bf16 torch (cpu)
        for i in range(L):
            h_bits = synth.bf16_bits(hl[i])
            h_dev = hl[i].to("cuda")
            y = torch.empty(h_dev.shape[0], model.d, dtype=torch.float32, device="cuda")
            tr = ctx.layer_forward(i, h_dev, y, stream=stream, flags=flags)
            stream.synchronize()
            y_ref, ids, w, logits = model.oracle_layer(i, h_bits, renorm=renorm)
            assert np.array_equal(tr.ids, ids), (t, i, tr.ids, ids)
            np.testing.assert_allclose(tr.w, w, rtol=0, atol=1e-6)
            nxt, rank = None, None
            if flags & api.M.FUSE_PREDICT:
                nxt = (i + 1) % L
                rank = ON.predicted_ranking(ON.router_logits(h_bits, model.routers[nxt]), K)
                assert np.array_equal(tr.ranking, rank), (t, i)
            o = orc.step(i, ids, nxt, rank)
            assert tr.act == o.act, (t, i, tr.act, o.act)
            assert tr.adm == o.adm, (t, i, tr.adm, o.adm)
            assert tr.plan == o.plan, (t, i)
            assert (tr.pcie_ondemand, tr.pcie_prefetch, tr.hbm) == (o.pcie_ondemand, o.pcie_prefetch, o.hbm)
            if check_y:
                e = rel_err(y.cpu().numpy(), y_ref)
                worst = max(worst, e)
                assert e <= TOL, (t, i, e)
    return worst


# ------------------------------------------------------------------ T2 router
@pytest.mark.parametrize("shape,B", [("toy", 1), ("toy", 16), ("qwen3", 1), ("qwen3", 5), ("qwen3", 16),
                                     ("deepseek", 3), ("mixtral", 1), ("mixtral", 7)])
def test_router_ids_weights_ranking_bit_exact(shape, B):
    api = _api()
    S = synth.SHAPES[shape]
    for seed in range(3):
        m = Model(2, S.N, S.K, S.d, 64, L_host=1, seed=seed)    # I irrelevant for routing
        ctx = _ctx(m, max_batch=B, v_e_max=1.0)
        ctx.configure(v_e=0.0, prefetch=True)
        h = synth.batch_hidden(seed + 11, B, S.d)
        y = torch.empty(B, S.d, dtype=torch.float32, device="cuda")
        tr = ctx.layer_forward(0, h.to("cuda"), y, flags=api.M.FUSE_PREDICT)
        torch.cuda.synchronize()
        hb = synth.bf16_bits(h)
        lg = ON.router_logits(hb, m.routers[0])
        ids = np.stack([ON.topk_ids(lg[b], S.K) for b in range(B)])
        w = np.stack([ON.gate_weights(lg[b], ids[b]) for b in range(B)])
        assert np.array_equal(tr.ids, ids)
        np.testing.assert_allclose(tr.w, w, rtol=0, atol=1e-6)
        np.testing.assert_allclose(tr.w.sum(axis=1), 1.0, atol=1e-6)
        rank = ON.predicted_ranking(ON.router_logits(hb, m.routers[1]), S.K)
        assert np.array_equal(tr.ranking, rank)
        ctx.close()


# ------------------------------------------------------------------ T3/T4 toy replay
def test_toy_full_replay():
    """BJ config 0: 2 layers, 8 experts top-2, d 64, I 128, r = 0.5, 16 tokens, 4-expert budget."""
    api = _api()
    S = synth.SHAPES["toy"]
    m = Model(S.L, S.N, S.K, S.d, S.I, seed=0)
    ctx = _ctx(m, max_batch=16, v_e_max=4.0, g=16)
    orc = OracleEngine(S.L, S.N, S.K, S.d, S.I, row_granule=16)
    cfg = dict(v_e=4.0, theta_i=[0.5, 0.5], seed=0)
    assert ctx.configure(**cfg)["C_i"] == list(orc.configure(CacheConfig(**cfg))[0])
    H = synth.hidden_states(0, 16, S.L, S.d)                         # [T][L][d]
    toks = [[H[t, i][None] for i in range(S.L)] for t in range(16)]
    worst = _replay(m, ctx, orc, toks, api.M.FUSE_PREDICT)
    # one batch step of all 16 tokens (B = 16)
    batch = [[H[:, i] for i in range(S.L)]]
    worst = max(worst, _replay(m, ctx, orc, batch, api.M.FUSE_PREDICT))
    assert worst <= TOL


@pytest.mark.parametrize("theta,v_e,prefetch", [(0.5, 4.0, True), (0.25, 4.0, True), (1.0, 4.0, False),
                                                (1.0, 4.0, True), (0.5, 0.0, True), (0.75, 6.0, True)])
def test_split_identity_every_mode(theta, v_e, prefetch):
    """C-P1 on the GPU: the output does not depend on theta / budget / prefetch."""
    api = _api()
    m = Model(2, 8, 2, 256, 512, seed=3)
    ctx = _ctx(m, max_batch=4, v_e_max=8.0, g=64)
    orc = OracleEngine(2, 8, 2, 256, 512, row_granule=64)
    cfg = dict(v_e=v_e, theta_i=[theta, theta], prefetch=prefetch, seed=5)
    ctx.configure(**cfg)
    orc.configure(CacheConfig(**cfg))
    H = synth.hidden_states(7, 6, 2, 256)
    toks = [[H[t, i][None] for i in range(2)] for t in range(6)]
    _replay(m, ctx, orc, toks, api.M.FUSE_PREDICT if prefetch else 0)


@pytest.mark.parametrize("policy", [0, 1, 2, 3])
def test_policies_replay_qwen_small(policy):
    """Multi-layer multi-token replay with admissions and evictions (tight budget)."""
    api = _api()
    m = Model(3, 32, 4, 256, 256, seed=policy)
    ctx = _ctx(m, max_batch=3, v_e_max=6.0, g=64)
    orc = OracleEngine(3, 32, 4, 256, 256, row_granule=64)
    cfg = dict(v_e=6.0, theta_i=[0.5, 0.25, 0.75], policy=policy, seed=13)
    ctx.configure(**cfg)
    orc.configure(CacheConfig(**cfg))
    H = synth.hidden_states(policy, 12, 3, 256)
    toks = [[H[t, i][None] for i in range(3)] for t in range(8)]
    toks += [[H[8:11, i] for i in range(3)]]                      # B = 3 step
    _replay(m, ctx, orc, toks, api.M.FUSE_PREDICT)


def test_solver_reconfigure_on_gpu():
    api = _api()
    m = Model(4, 16, 2, 128, 256, seed=21)
    ctx = _ctx(m, v_e_max=16.0, g=64)
    orc = OracleEngine(4, 16, 2, 128, 256, row_granule=64)
    cfg = dict(v_e=12.0, t_att=20.0, t_moe=40.0, t_head=10.0, t_load_exp=35.0, zeta=0.02)
    ctx.configure(**cfg)
    orc.configure(CacheConfig(**cfg))
    H = synth.hidden_states(21, 30, 4, 128)
    toks = [[H[t, i][None] for i in range(4)] for t in range(20)]
    _replay(m, ctx, orc, toks, api.M.FUSE_PREDICT)
    a = ctx.configure(use_solver=True, **cfg)
    C, It, th, V = orc.configure(CacheConfig(use_solver=True, **cfg))
    assert a["C_i"] == C and a["I_top_i"] == It and a["V_i"] == V
    toks = [[H[t, i][None] for i in range(4)] for t in range(20, 30)]
    _replay(m, ctx, orc, toks, api.M.FUSE_PREDICT)


# ------------------------------------------------------------------ BJ shapes
@pytest.mark.parametrize("B", [1, 4, 16])
def test_qwen3_shape(B):
    """BJ config 2 shape (d 2048, I 768, 128 experts top-8), 2 layers, 50% budget."""
    api = _api()
    S = synth.SHAPES["qwen3"]
    m = Model(2, S.N, S.K, S.d, S.I, seed=1, gen_device="cuda")
    ctx = _ctx(m, max_batch=B, v_e_max=128.0)
    orc = OracleEngine(2, S.N, S.K, S.d, S.I)
    cfg = dict(v_e=128.0, seed=2)
    ctx.configure(**cfg)
    orc.configure(CacheConfig(**cfg))
    H = synth.hidden_states(5, 3 * B, 2, S.d)
    toks = [[H[t * B:(t + 1) * B, i] for i in range(2)] for t in range(3)]
    _replay(m, ctx, orc, toks, api.M.FUSE_PREDICT)


@pytest.mark.parametrize("B,tail_kb", [(1, 256), (4, 256), (16, 1024), (4, 4000)])
def test_od_tail_split(B, tail_kb, monkeypatch):
    """The layer's last on-demand copy split into head + tail (MOEPIC_OD_TAIL_KB, read at create):
    one K2 launch over the resident, prefetched and head rows, then the tail with the fused
    combine.  Qwen3 shape, where bottoms are 4.7 MB: 256 KB / 1 MB tails split every layer; a
    4000 KB tail is over half a bottom, so nothing is split.  Same traces, y within TOL."""
    api = _api()
    S = synth.SHAPES["qwen3"]
    m = Model(2, S.N, S.K, S.d, S.I, seed=3, gen_device="cuda")
    H = synth.hidden_states(6, 3 * B, 2, S.d)
    toks = [[H[t * B:(t + 1) * B, i] for i in range(2)] for t in range(3)]
    copies = {}
    for kb in (tail_kb, 0):      # 0: no split (the reference count of copies)
        monkeypatch.setenv("MOEPIC_OD_TAIL_KB", str(kb))
        ctx = _ctx(m, max_batch=B, v_e_max=128.0)
        orc = OracleEngine(2, S.N, S.K, S.d, S.I)
        cfg = dict(v_e=128.0, seed=5)
        ctx.configure(**cfg, cancel_prefetch=False)   # every planned chunk issued: a timing-free count
        orc.configure(CacheConfig(**cfg))
        c0 = ctx.counters()
        _replay(m, ctx, orc, toks, api.M.FUSE_PREDICT)
        copies[kb] = ctx.counters()["h2d_copies"] - c0["h2d_copies"]
        del ctx
    extra = copies[tail_kb] - copies[0]      # one extra copy per split layer step (6 steps)
    if tail_kb < 2000:
        assert 0 < extra <= 6, copies
    else:
        assert extra == 0, copies


def test_deepseek_shape_shared_no_renorm():
    """BJ config 3 shape: 64 routed + 2 shared experts top-6, d 2048, I 1408, renorm off (Q4)."""
    api = _api()
    S = synth.SHAPES["deepseek"]
    m = Model(2, S.N, S.K, S.d, S.I, n_shared=2, seed=4, gen_device="cuda")
    ctx = _ctx(m, max_batch=2, v_e_max=64.0, renorm=0)
    orc = OracleEngine(2, S.N, S.K, S.d, S.I, n_shared=2)
    cfg = dict(v_e=64.0, seed=1)
    ctx.configure(**cfg)
    orc.configure(CacheConfig(**cfg))
    H = synth.hidden_states(9, 4, 2, S.d)
    toks = [[H[t:t + 1, i] for i in range(2)] for t in range(3)] + [[H[2:4, i] for i in range(2)]]
    _replay(m, ctx, orc, toks, api.M.FUSE_PREDICT, renorm=False)


def test_mixtral_full_size_layer():
    """BJ config 1 layer at full size (d 4096, I 14336, 8 experts top-2), 50% budget, B = 1."""
    api = _api()
    S = synth.SHAPES["mixtral"]
    m = Model(2, S.N, S.K, S.d, S.I, L_host=1, seed=0, gen_device="cuda")
    ctx = _ctx(m, v_e_max=8.0)
    orc = OracleEngine(2, S.N, S.K, S.d, S.I)
    cfg = dict(v_e=8.0, seed=0)
    ctx.configure(**cfg)
    orc.configure(CacheConfig(**cfg))
    H = synth.hidden_states(1, 3, 2, S.d)
    toks = [[H[t, i][None] for i in range(2)] for t in range(3)]
    _replay(m, ctx, orc, toks, api.M.FUSE_PREDICT)


# ------------------------------------------------------------------ API paths
def test_host_buffers_and_predict_prefetch():
    api = _api()
    m = Model(2, 8, 2, 128, 256, seed=8)
    ctx = _ctx(m, max_batch=2, v_e_max=8.0)
    orc = OracleEngine(2, 8, 2, 128, 256)
    cfg = dict(v_e=2.0, seed=0)
    ctx.configure(**cfg)
    orc.configure(CacheConfig(**cfg))
    H = synth.hidden_states(8, 4, 2, 128)
    # predict layer 0 from the "previous token's last layer"
    hp = H[0, 1][None]
    tr = ctx.predict_prefetch(0, hp.to("cuda"))
    rank = ON.predicted_ranking(ON.router_logits(synth.bf16_bits(hp), m.routers[0]), 2)
    o = orc.predict_prefetch(0, rank)
    assert tr.plan == o.plan and np.array_equal(tr.ranking, rank)
    for t in range(1, 4):
        for i in range(2):
            hb = synth.bf16_bits(H[t, i][None])
            y, tr = ctx.layer_forward_host(i, hb, flags=api.M.FUSE_PREDICT)
            y_ref, ids, _, _ = m.oracle_layer(i, hb)
            nrank = ON.predicted_ranking(ON.router_logits(hb, m.routers[(i + 1) % 2]), 2)
            o = orc.step(i, ids, (i + 1) % 2, nrank)
            assert tr.act == o.act and tr.adm == o.adm and tr.plan == o.plan
            assert rel_err(y, y_ref) <= TOL


@pytest.mark.parametrize("B", [3, 40])
def test_host_buffers_batches(B):
    """Host-buffer entry for a decode batch and a prefill batch (h staged by SM loads from mapped
    pinned memory, y stored zero-copy into mapped pinned memory)."""
    api = _api()
    m = Model(2, 8, 2, 256, 512, n_shared=1, seed=18)
    ctx = _ctx(m, max_batch=B, v_e_max=8.0)
    orc = OracleEngine(2, 8, 2, 256, 512, n_shared=1)
    cfg = dict(v_e=4.0, seed=2)
    ctx.configure(**cfg)
    orc.configure(CacheConfig(**cfg))
    H = synth.hidden_states(19, 2 * B, 2, 256)
    for t in range(2):
        for i in range(2):
            hb = synth.bf16_bits(H[t * B:(t + 1) * B, i])
            y, tr = ctx.layer_forward_host(i, hb, flags=api.M.FUSE_PREDICT)
            y_ref, ids, _, _ = m.oracle_layer(i, hb)
            assert np.array_equal(tr.ids, ids)
            nrank = ON.predicted_ranking(ON.router_logits(hb, m.routers[(i + 1) % 2]), 2)
            o = orc.step(i, ids, (i + 1) % 2, nrank)
            assert tr.act == o.act and tr.adm == o.adm and tr.plan == o.plan
            assert rel_err(y, y_ref) <= TOL


def test_residual_flag_and_errors():
    api = _api()
    m = Model(2, 8, 2, 64, 128, seed=2)
    ctx = _ctx(m, v_e_max=4.0, g=16)
    h = synth.batch_hidden(1, 1, 64)
    y = torch.empty(1, 64, dtype=torch.float32, device="cuda")
    with pytest.raises(api.MoEpicError):
        ctx.layer_forward(0, h.cuda(), y)          # not configured yet
    ctx.configure(v_e=4.0)
    ctx.layer_forward(0, h.cuda(), y, flags=api.M.RESIDUAL)
    torch.cuda.synchronize()
    y_ref, _, _, _ = m.oracle_layer(0, synth.bf16_bits(h))
    y_ref = y_ref + ON.bf16_to_f64(synth.bf16_bits(h))
    assert rel_err(y.cpu().numpy(), y_ref) <= TOL
    with pytest.raises(api.MoEpicError):
        ctx.layer_forward(5, h.cuda(), y)          # layer out of range
    with pytest.raises(api.MoEpicError):
        ctx.configure(v_e=5.0)                     # exceeds v_e_max
    ctx.layer_forward(1, h.cuda(), y)              # still usable after EINVAL


def test_cancel_prefetch_same_results_fewer_bytes():
    """P:291 "terminates the prefetch": dropping the unissued chunks of mispredicted experts
    changes neither traces nor outputs, only the bytes moved (<= planned)."""
    api = _api()
    S = synth.SHAPES["qwen3"]
    runs = {}
    for cancel in (True, False):
        m = Model(3, S.N, S.K, S.d, S.I, L_host=1, seed=2, gen_device="cuda")
        ctx = _ctx(m, v_e_max=96.0)
        ctx.configure(v_e=96.0, seed=1, cancel_prefetch=cancel, y_cap_i=[16] * 3)
        H = synth.hidden_states(2, 12, 3, S.d)
        ys, trs = [], []
        for t in range(12):
            for i in range(3):
                y = torch.empty(1, S.d, dtype=torch.float32, device="cuda")
                tr = ctx.layer_forward(i, H[t, i][None].cuda(), y, flags=api.M.FUSE_PREDICT)
                torch.cuda.synchronize()
                ys.append(y.cpu().numpy())
                trs.append((tr.act, tr.adm, tr.plan, tr.pcie_prefetch))
        runs[cancel] = (ys, trs, ctx.counters())
        ctx.close()
    assert runs[True][1] == runs[False][1]
    for a, b in zip(runs[True][0], runs[False][0]):
        np.testing.assert_array_equal(a, b)            # deterministic kernels: bit-identical
    c_on, c_off = runs[True][2], runs[False][2]
    assert c_off["pcie_prefetch_bytes"] == c_off["pcie_prefetch_planned_bytes"]
    assert c_on["pcie_prefetch_planned_bytes"] == c_off["pcie_prefetch_planned_bytes"]
    assert c_on["pcie_prefetch_bytes"] < c_on["pcie_prefetch_planned_bytes"]


@pytest.mark.parametrize("B,W,th", [(1, 64, 0.5), (1, 192, 0.5), (3, 128, 0.5), (40, 192, 0.5), (1, 320, 1.0),
                                    (2, 128, 1.0), (40, 448, 1.0)])
def test_window_cut_prefetch(B, W, th):
    """Reading Q30 on the GPU: plans cut at W rows; a cut item's prefix (of a bottom, or of a
    full expert) is computed from the plan buffer (after the plan event) and the rest of it
    from the on-demand region -- two segments of one expert, on K2 (B <= 32) and on the tcgen05
    prefill path (B = 40); an admitted gamma with a prefix fills its slot by D2D from both.
    Traces and bytes bit-exact, y within 2e-3 (split identity)."""
    api = _api()
    m = Model(3, 8, 2, 256, 512, seed=29)
    ctx = _ctx(m, max_batch=B, v_e_max=12.0, g=64)
    orc = OracleEngine(3, 8, 2, 256, 512, row_granule=64)
    cfg = dict(v_e=6.0 if th < 1 else 3.0, theta_i=[th, th / 2, th], prefetch_rows_i=[W] * 3, seed=2)
    ctx.configure(**cfg)
    orc.configure(CacheConfig(**cfg))
    H = synth.hidden_states(41, 4 * B, 3, 256)
    toks = [[H[t * B:(t + 1) * B, i] for i in range(3)] for t in range(4)]
    _replay(m, ctx, orc, toks, api.M.FUSE_PREDICT)
    c = ctx.counters()
    assert c["pred_hits"] > 0 and c["pcie_prefetch_planned_bytes"] > 0


@pytest.mark.parametrize("env", [{"MOEPIC_COPY_STREAMS": "2"}, {"MOEPIC_PDL": "0", "MOEPIC_OD_SPLIT_BOUNDARY": "0"}])
def test_transfer_engine_variants_bit_identical(env, monkeypatch):
    """The transfer-engine / launch variants change only when things run, never what: traces equal;
    two copy streams keep the K2 launch grouping, so y is bit-identical; without the PDL router and
    the boundary split the rows are grouped into launches differently, so y agrees to fp32
    rounding of the partial sums."""
    api = _api()
    S = synth.SHAPES["qwen3"]
    m = Model(2, S.N, S.K, S.d, S.I, seed=6, gen_device="cuda")
    H = synth.hidden_states(8, 6, 2, S.d)
    toks = [[H[t, i][None] for i in range(2)] for t in range(6)]
    out = []
    for variant in (None, env):
        for k in ("MOEPIC_COPY_STREAMS", "MOEPIC_PDL", "MOEPIC_OD_SPLIT_BOUNDARY"):
            monkeypatch.delenv(k, raising=False)
        for k, v in (variant or {}).items():
            monkeypatch.setenv(k, v)
        ctx = _ctx(m, v_e_max=64.0)
        ctx.configure(v_e=48.0, seed=4, prefetch_rows_i=[256, 256])
        ys, trs = [], []
        for t in toks:
            for i in range(2):
                y = torch.empty(1, S.d, dtype=torch.float32, device="cuda")
                tr = ctx.layer_forward(i, t[i].cuda(), y, flags=api.M.FUSE_PREDICT)
                torch.cuda.synchronize()
                ys.append(y.cpu().numpy())
                trs.append((tr.act, tr.adm, tr.plan, tr.pcie_ondemand))
        out.append((ys, trs))
        ctx.close()
    assert out[0][1] == out[1][1]
    for a, b in zip(out[0][0], out[1][0]):
        if "MOEPIC_COPY_STREAMS" in env:
            np.testing.assert_array_equal(a, b)
        else:
            assert rel_err(b, a) <= 1e-5


def test_profile_class_mask():
    """moepic_profile(MOEPIC_PROFILE_CLASSES | 1 << class): only that class is event-timed."""
    api = _api()
    S = synth.SHAPES["qwen3"]
    m = Model(2, S.N, S.K, S.d, S.I, L_host=1, seed=1, gen_device="cuda")
    ctx = _ctx(m, v_e_max=64.0)
    ctx.configure(v_e=32.0, seed=1)
    H = synth.hidden_states(3, 4, 2, S.d)
    ctx.profile(api.M.PROFILE_CLASSES | (1 << api.M.KERNEL_EXPERT))
    for t in range(4):
        for i in range(2):
            y = torch.empty(1, S.d, dtype=torch.float32, device="cuda")
            ctx.layer_forward(i, H[t, i][None].cuda(), y, flags=api.M.FUSE_PREDICT)
    torch.cuda.synchronize()
    k1, k2 = ctx.profile_read(api.M.KERNEL_ROUTER), ctx.profile_read(api.M.KERNEL_EXPERT)
    assert k1["launches"] == 0 and k2["launches"] >= 8 and k2["kernel_ms"] > 0
    ctx.profile(True)
    for i in range(2):
        y = torch.empty(1, S.d, dtype=torch.float32, device="cuda")
        ctx.layer_forward(i, H[0, i][None].cuda(), y, flags=api.M.FUSE_PREDICT)
    torch.cuda.synchronize()
    assert ctx.profile_read(api.M.KERNEL_ROUTER)["launches"] == 2
    ctx.close()
