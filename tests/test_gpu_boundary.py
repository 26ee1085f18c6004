"""GPU checks of the boundary's less-travelled paths, all through the C ABI:

* stats checkpoint: get_stats -> set_stats into a fresh context -> identical Alg. 1 config
   and identical traces afterwards, equal to the oracle that never restarted;
* exact logit ties in the router: duplicated router rows, h = 0, duplicated tokens at B > 1
  (keys (logit desc, id asc), reading Q4 / Q9 / Q25);
* C-P1 split identity at every granule I_top in {0, g, ..., I}, including I_top = 0 with C > 0
  (P:231);
* a real CUDA fault (MOEPIC_FAULT_AT_STEP) -> ERUNTIME, then ESTATE on every later call;
* poison mode (MOEPIC_POISON=1): freed ping-pong halves, the workspace, the slot pool and
  evicted slots are NaN-filled; the parity replays must be unchanged.
"""
import os
import subprocess
import sys
import textwrap

import numpy as np
import pytest
import torch

import synth
from oracle import numeric as ON
from oracle.replay import OracleEngine, CacheConfig
from gpu_model import Model, rel_err, TOL

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    from paper_2509_08342_b200 import build
    build.build()


def _api():
    from paper_2509_08342_b200 import api
    return api


def _ctx(m, max_batch=1, v_e_max=None, g=64, Ub=None):
    api = _api()
    desc = api.model_desc(m.L, m.N, m.K, m.d, m.I, n_shared=m.n_shared, row_granule=g, buffer_experts=Ub,
                          max_batch=max_batch, L_host=m.L_host, v_e_max=v_e_max or m.L * m.N)
    ctx = api.MoEpic(desc)
    m.load_into(ctx)
    return ctx


def _step_both(m, ctx, orc, i, h, flags):
    api = _api()
    hb = synth.bf16_bits(h)
    y = torch.empty(h.shape[0], m.d, dtype=torch.float32, device="cuda")
    tr = ctx.layer_forward(i, h.cuda(), y, flags=flags)
    torch.cuda.synchronize()
    y_ref, ids, w, _ = m.oracle_layer(i, hb)
    assert np.array_equal(tr.ids, ids)
    nxt, rank = None, None
    if flags & api.M.FUSE_PREDICT:
        nxt = (i + 1) % m.L
        rank = ON.predicted_ranking(ON.router_logits(hb, m.routers[nxt]), m.K)
        assert np.array_equal(tr.ranking, rank)
    o = orc.step(i, ids, nxt, rank)
    assert (tr.act, tr.adm, tr.plan) == (o.act, o.adm, o.plan)
    assert (tr.pcie_ondemand, tr.pcie_prefetch, tr.hbm) == (o.pcie_ondemand, o.pcie_prefetch, o.hbm)
    assert rel_err(y.cpu().numpy(), y_ref) <= TOL
    return tr


def test_stats_checkpoint_round_trip_gpu():
    api = _api()
    F = api.M.FUSE_PREDICT
    m = Model(3, 16, 2, 256, 256, seed=17)
    a = _ctx(m, max_batch=2, v_e_max=12.0)
    orc = OracleEngine(3, 16, 2, 256, 256)
    kw = dict(v_e=9.0, t_att=20.0, t_moe=40.0, t_head=10.0, t_load_exp=35.0, zeta=0.02, seed=4)
    a.configure(**kw)
    orc.configure(CacheConfig(**kw))
    H = synth.hidden_states(13, 40, 3, 256)
    for t in range(30):
        for i in range(3):
            _step_both(m, a, orc, i, H[t, i][None], F)
    blob = a.get_stats()
    b = _ctx(m, max_batch=2, v_e_max=12.0)
    b.configure(**kw)
    b.set_stats(blob)
    assert b.get_stats() == blob
    skw = dict(kw, use_solver=True)
    ra, rb = a.configure(**skw), b.configure(**skw)
    C, It, th, V = orc.configure(CacheConfig(**skw))
    assert ra == rb and ra["C_i"] == C and ra["I_top_i"] == It and ra["V_i"] == V
    import copy
    orc_b = copy.deepcopy(orc)   # b's future = a's future: replay both against copies of the oracle
    for t in range(30, 40):
        for i in range(3):
            _step_both(m, a, orc, i, H[t, i][None], F)
            _step_both(m, b, orc_b, i, H[t, i][None], F)
    a.close()
    b.close()


def _route_check(ctx, m, h, B):
    api = _api()
    y = torch.empty(B, m.d, dtype=torch.float32, device="cuda")
    tr = ctx.layer_forward(0, h.cuda(), y, flags=api.M.FUSE_PREDICT)
    torch.cuda.synchronize()
    hb = synth.bf16_bits(h)
    lg = ON.router_logits(hb, m.routers[0])
    ids = np.stack([ON.topk_ids(lg[b], m.K) for b in range(B)])
    w = np.stack([ON.gate_weights(lg[b], ids[b]) for b in range(B)])
    assert np.array_equal(tr.ids, ids), (tr.ids, ids)
    np.testing.assert_allclose(tr.w, w, rtol=0, atol=1e-6)
    rank = ON.predicted_ranking(ON.router_logits(hb, m.routers[1]), m.K)
    assert np.array_equal(tr.ranking, rank), (tr.ranking, rank)
    return tr, lg, ids, rank


@pytest.mark.parametrize("shape", ["toy", "qwen3", "mixtral"])
def test_router_exact_ties(shape):
    """Exact logit ties: the id-ascending tie rules hold on the GPU as in the oracle (where they
    are pinned against brute force, tests/test_oracle_numeric.py)."""
    S = synth.SHAPES[shape]
    m = Model(2, S.N, S.K, S.d, 64, L_host=1, seed=5)
    # duplicate router rows: every expert j >= N/2 copies row j - N/2 in both routers, so each
    # logit of the upper half ties exactly with one of the lower half
    for i in range(2):
        r = m.routers[i].copy()
        r[S.N // 2:] = r[:S.N // 2]
        m.routers[i] = r
    for B in (1, 3):
        ctx = _ctx(m, max_batch=B, v_e_max=1.0)
        ctx.configure(v_e=0.0)
        h = synth.batch_hidden(23, B, S.d)
        tr, lg, ids, rank = _route_check(ctx, m, h, B)
        # the tie is real: the winner's twin has the same logit and a larger id
        e0 = int(ids[0, 0])
        twin = e0 + S.N // 2 if e0 < S.N // 2 else e0 - S.N // 2
        assert lg[0, e0] == lg[0, twin] and e0 < twin
        # h = 0: every logit is +0 -> ids 0..K-1, w = 1/K, ranking 0..N-1
        z = torch.zeros(B, S.d, dtype=torch.bfloat16)
        tr, lg, ids, rank = _route_check(ctx, m, z, B)
        assert np.array_equal(ids, np.tile(np.arange(S.K), (B, 1)))
        assert np.array_equal(rank, np.arange(S.N))
        np.testing.assert_allclose(tr.w, 1.0 / S.K, atol=1e-7)
        ctx.close()
    # B > 1 with duplicated tokens: prediction counts and max logits tie in pairs (Q9 keys)
    ctx = _ctx(m, max_batch=4, v_e_max=1.0)
    ctx.configure(v_e=0.0)
    h = synth.batch_hidden(29, 2, S.d)
    _route_check(ctx, m, torch.cat([h, h]), 4)
    ctx.close()


def test_split_identity_every_granule():
    """C-P1 at every I_top in {0, g, ..., I} (g = 64, I = 256): theta 0.2 gives I_top = 0 with
    C > 0 (a cache that holds nothing, reading Q2 / Q21), 0.25 / 0.5 / 0.75 / 1 the others;
    per-layer mixes too.  Output within 2e-3 of the unsplit oracle layer, traces bit-exact."""
    api = _api()
    m = Model(2, 8, 2, 256, 256, seed=8)
    H = synth.hidden_states(4, 6, 2, 256)
    for th in ([0.2, 0.2], [0.25, 0.25], [0.5, 0.5], [0.75, 0.75], [1.0, 1.0], [0.2, 1.0], [0.75, 0.25]):
        ctx = _ctx(m, max_batch=1, v_e_max=8.0)
        orc = OracleEngine(2, 8, 2, 256, 256)
        cfg = dict(v_e=2.0, theta_i=th, seed=1)
        r = ctx.configure(**cfg)
        C, It, _, _ = orc.configure(CacheConfig(**cfg))
        assert r["C_i"] == C and r["I_top_i"] == It
        if th[0] == 0.2:
            assert It[0] == 0 and C[0] > 0
        for t in range(6):
            for i in range(2):
                _step_both(m, ctx, orc, i, H[t, i][None], api.M.FUSE_PREDICT)
        ctx.close()


def _child(code, env_extra, timeout=300):
    env = dict(os.environ, **env_extra)
    env["PYTHONPATH"] = ROOT + os.pathsep + os.path.join(ROOT, "tests") + os.pathsep + env.get("PYTHONPATH", "")
    return subprocess.run([sys.executable, "-c", textwrap.dedent(code)], env=env, capture_output=True, text=True,
                          timeout=timeout, cwd=ROOT)


def test_injected_cuda_fault_poisons_context():
    """A real kernel fault (a trap on the caller's stream at the 3rd layer_forward) returns
    MOEPIC_ERUNTIME with the CUDA error in last_error; every later call returns MOEPIC_ESTATE
    (moepic.h conventions).  Runs in a child process: the fault leaves the CUDA context unusable."""
    code = """
        import ctypes as C, torch, synth
        from gpu_model import Model
        from paper_2509_08342_b200 import api, _moepic as M
        m = Model(2, 8, 2, 128, 128, seed=1)
        desc = api.model_desc(2, 8, 2, 128, 128, max_batch=1, v_e_max=4.0)
        ctx = api.MoEpic(desc)
        m.load_into(ctx)
        ctx.configure(v_e=2.0)
        h = synth.batch_hidden(1, 1, 128).cuda()
        y = torch.empty(1, 128, dtype=torch.float32, device="cuda")
        st = []
        for k in range(5):
            st.append(M.moepic_layer_forward(ctx.h, k % 2, C.c_void_p(h.data_ptr()), 1, C.c_void_p(y.data_ptr()),
                                             None, 0, None))
            if k == 2:
                print("ERR", M.moepic_last_error(ctx.h).decode())
        st.append(M.moepic_configure(ctx.h, None, None))
        print("STATUS", st)
    """
    r = _child(code, {"MOEPIC_FAULT_AT_STEP": "3"})
    assert r.returncode == 0, r.stderr[-2000:]
    line = [x for x in r.stdout.splitlines() if x.startswith("STATUS")][0]
    st = eval(line.split(" ", 1)[1])
    assert st == [0, 0, 2, 4, 4, 4], st
    err = [x for x in r.stdout.splitlines() if x.startswith("ERR")][0]
    assert "cudaStreamSynchronize" in err


def test_poison_mode_parity_unchanged():
    """the replay / edge parity tests rerun with MOEPIC_POISON=1 (dead buffers and
    evicted slots NaN-filled): a stale or early read would surface as NaN."""
    sel = ("test_toy_full_replay or test_split_identity_every_mode or test_policies_replay_qwen_small "
           "or test_od_tail_split or test_cancel_prefetch or test_prefill_smallest_batches "
           "or test_configure_drops_pending_prefetch or test_decode_max_batch_32 or test_deepseek_shape "
           "or test_window_cut_prefetch or test_k2t or test_q4_prefill_parity")
    env = dict(os.environ, MOEPIC_POISON="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-k", sel,
                        "tests/test_gpu_parity.py", "tests/test_gpu_edges.py", "tests/test_gpu_k2t.py",
                        "tests/test_gpu_q4.py"],
                       env=env, capture_output=True, text=True, timeout=1200, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout
