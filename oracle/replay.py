"""C-S: the MoEpic control-plane state machine, step by step (TEST INFRASTRUCTURE).

One `step()` is one `moepic_layer_forward` (layer i, one batch of B tokens); one
`predict_prefetch()` is one `moepic_predict_prefetch`; `configure()` is one
`moepic_configure`.  The algorithm follows the paper in its order; every choice the
paper leaves open is a numbered reading in DESIGN.md (Q-numbers below).

Per step, in order:
  1. A = distinct activated experts, ordered (B_e desc, id asc)                    (Q9)
  2. stats observe (pre-step frequency ranks; prediction = the ranking that planned
     this layer's prefetch, if any)                                                (Q15)
  3. classify against the state before the step:
       alpha: all rows resident — (top cached and (theta_eff = 1 or bottom prefetched))
              or full expert prefetched
       beta : top cached, bottom missing          gamma: otherwise
  4. counters: e in A: mu += B_e, nu = 0, last = step; else nu += 1  (Q12)
  5. admission (Q11): each e in A whose top is not cached, in A order: free slot
     if |cache| < C_i, else victim = min over cache \\ A of (key asc, nu desc, id asc)
     (RND: splitmix64 draw over the id-sorted candidates); no candidate -> not admitted
  6. bytes: PCIe on-demand = sum_beta (I - I_top) 6d + sum_gamma I 6d
  7. plan for the next layer (Q7/Q8): walk R'; rows = I - I_top if the top is
     cached there (skip if 0) else I (full); stop at the first item that does not fit
     U_b * I rows or when the count reaches the Y cap.
     Reading Q30 (window-capped plan): with a per-layer prefetch window W_j in rows
     (prefetch_rows_i), the plan is cut at min(U_b * I, W_j) rows; the count cap is then
     y_cap only (Alg. 1's Y stays inside the solver).  The item at the cut (bottom or full
     expert) keeps its first g * floor(remaining / g) rows: "the router terminates the
     prefetch" mid-item, deterministically at W_j.  An activated expert with a
     prefetched prefix is not fully resident: beta (bottom prefix) or gamma (prefix of
     a full expert), and loads only the rest; an admitted gamma-with-prefix fills its slot
     on the device (D2D of its top rows, as for a fully prefetched expert).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import policy as P
from .stats import LayerStats
from .configurator import vram_allocation

ALPHA, BETA, GAMMA = 0, 1, 2
ADM_FREE, ADM_NONE = -1, -2


@dataclass
class CacheConfig:
    v_e: float
    v_i: list | None = None
    theta_i: list | None = None
    use_solver: bool = False
    policy: int = P.LCP
    rho: float = 0.25
    omega: int = 128
    zeta: float = 0.01
    tau: int = 5000
    t_att: float = 0.0
    t_moe: float = 0.0
    t_head: float = 0.0
    t_load_exp: float = 0.0
    y_cap_i: list | None = None
    prefetch: bool = True
    seed: int = 0
    prefetch_rows_i: list | None = None   # reading Q30: per-layer window W_j in rows


@dataclass
class Plan:
    target: int
    items: list            # [(expert, full: bool, rows)]
    ranking: np.ndarray | None


@dataclass
class StepTrace:
    act: list = field(default_factory=list)       # [(expert, class)] in A order
    adm: list = field(default_factory=list)       # [(expert, victim)]
    plan: list = field(default_factory=list)      # [(expert, full)]
    pcie_ondemand: int = 0
    pcie_prefetch: int = 0
    hbm: int = 0


class OracleEngine:
    def __init__(self, L, N, K, d, I, row_granule=64, buffer_experts=None, n_shared=0, I_shared=None,
                 ep_rank=0, ep_size=1):
        self.L, self.N, self.K, self.d, self.I = L, N, K, d, I
        # expert parallelism: this engine is rank ep_rank of ep_size; it owns
        # experts e with e * ep_size // N == ep_rank and the shared-expert rows
        # [ep_rank * I // ep_size, (ep_rank + 1) * I // ep_size)
        self.ep_rank, self.ep_size = ep_rank, ep_size
        self.g = row_granule
        self.U_b = K if buffer_experts is None else buffer_experts
        self.n_shared = n_shared
        self.I_shared = I if I_shared is None else I_shared
        self.row_bytes = 6 * d
        self.mu = [[0] * N for _ in range(L)]
        self.nu = [[0] * N for _ in range(L)]
        self.last = [[-1] * N for _ in range(L)]
        self.step_no = [0] * L
        self.cache = [set() for _ in range(L)]
        self.C = [0] * L
        self.I_top = [0] * L
        self.V = None
        self.Y = None
        self.stats = [LayerStats(N, K) for _ in range(L)]
        self.rnd = [0] * L
        self.cfg = None
        self.pending = None

    # ------------------------------------------------------------------ configure
    def is_local(self, e) -> bool:
        return e * self.ep_size // self.N == self.ep_rank

    def shared_rows(self) -> int:
        return (self.ep_rank + 1) * self.I_shared // self.ep_size - self.ep_rank * self.I_shared // self.ep_size

    def cache_on(self, i) -> bool:
        return self.C[i] > 0 and self.I_top[i] > 0

    def configure(self, cfg: CacheConfig):
        """moepic_configure.  Returns (C_i, I_top_i, theta_eff_i, V_i)."""
        L, N, K = self.L, self.N, self.K
        if cfg.v_e < 0:
            raise ValueError("v_e must be >= 0")
        first = self.cfg is None
        if first:
            for i in range(L):
                self.rnd[i] = P.layer_stream_seed(cfg.seed, i, 1)
        self.cfg = cfg
        if cfg.use_solver:
            if any(s.q == 0 for s in self.stats):
                raise ValueError("empty accumulator")
            V0 = self.V if self.V is not None else (
                list(cfg.v_i) if cfg.v_i is not None else [cfg.v_e / L] * L)
            V, th, C, _, _ = vram_allocation(self.stats, V0, cfg.v_e, cfg.zeta, K, N, float(self.U_b),
                                             cfg.t_att, cfg.t_moe, cfg.t_head, cfg.t_load_exp)
            thetas = th
            Cs = C
            self.Y = list(vram_allocation.last_Y)   # Eq. 10's Y caps the planner (reading Q27)
        else:
            self.Y = None
            V = list(cfg.v_i) if cfg.v_i is not None else [cfg.v_e / L] * L
            thetas = list(cfg.theta_i) if cfg.theta_i is not None else [0.5] * L
            s = 0.0
            for v in V:
                s = s + v
            if s > cfg.v_e + 1e-9:
                raise ValueError("sum V_i > V_e")
            Cs = []
            for i in range(L):
                if not (0.0 < thetas[i] <= 1.0):
                    raise ValueError("theta must be in (0, 1]")
                if V[i] < 0:
                    raise ValueError("V_i must be >= 0")
                c = int(math.floor(V[i] / thetas[i] + 1e-9))
                Cs.append(min(N, c))
        self.V = list(V)
        for i in range(L):
            self.C[i] = Cs[i]
            it = self.g * int(math.floor(thetas[i] * self.I / self.g + 1e-9))
            self.I_top[i] = min(self.I, it)
            self.cache[i] = set(self._relayout_set(i, cfg))
        self.pending = None
        theta_eff = [self.I_top[i] / self.I for i in range(L)]
        return list(self.C), list(self.I_top), theta_eff, list(self.V)

    def _relayout_set(self, i, cfg):
        """rank all N experts by cache priority, keep the top C_i.
        Cold start (no stats yet, "selected randomly", Q14): seed 0 -> ids 0..C-1,
        else the first C_i of a splitmix64 Fisher-Yates permutation."""
        N, C = self.N, self.C[i]
        if not self.cache_on(i):
            return []
        if self.stats[i].q == 0:
            if cfg.seed == 0:
                order = list(range(N))
            else:
                order, _ = P.fisher_yates(N, P.layer_stream_seed(cfg.seed, i, 2))
        elif cfg.policy == P.RND:
            order, self.rnd[i] = P.fisher_yates(N, self.rnd[i])
        else:
            keyf = lambda e: P.policy_key(cfg.policy, self.mu[i][e], self.nu[i][e], self.last[i][e], cfg.rho,
                                          cfg.omega)
            order = sorted(range(N), key=lambda e: (-keyf(e), self.nu[i][e], e))
        return [e for e in order if self.is_local(e)][:C]

    # ------------------------------------------------------------------ planning
    def _plan(self, j, ranking):
        cfg = self.cfg
        if not cfg.prefetch:
            return Plan(j, [], ranking)
        cap_rows = self.U_b * self.I
        ycap = self.N if cfg.y_cap_i is None else cfg.y_cap_i[j]
        window = cfg.prefetch_rows_i is not None
        if window:
            cap_rows = min(cap_rows, cfg.prefetch_rows_i[j])
        elif self.Y is not None:
            ycap = min(ycap, self.Y[j])
        items, used = [], 0
        for e in ranking:
            e = int(e)
            if len(items) >= ycap:
                break
            if not self.is_local(e):
                continue
            if self.cache_on(j) and e in self.cache[j]:
                rows = self.I - self.I_top[j]
                if rows == 0:
                    continue
                full = False
            else:
                rows, full = self.I, True
            if used + rows > cap_rows:
                part = self.g * ((cap_rows - used) // self.g)
                if window and part > 0:                   # Q30: the cut item keeps its prefix
                    items.append((e, full, part))
                break
            items.append((e, full, rows))
            used += rows
        return Plan(j, items, ranking)

    def predict_prefetch(self, j, ranking):
        """moepic_predict_prefetch (Q23): plan layer j from ranking R'."""
        self.pending = self._plan(j, np.asarray(ranking))
        tr = StepTrace()
        tr.plan = [(e, f) for (e, f, _) in self.pending.items]
        tr.pcie_prefetch = sum(r for (_, _, r) in self.pending.items) * self.row_bytes
        tr.hbm = tr.pcie_prefetch + self.N * self.d * 2
        return tr

    # ------------------------------------------------------------------ step
    def step(self, i, ids, next_layer=None, ranking_next=None, B=None):
        cfg = self.cfg
        N, I = self.N, self.I
        ids = np.asarray(ids)
        B = ids.shape[0]
        plan = self.pending if (self.pending is not None and self.pending.target == i) else None
        planned = {e: (full, rows) for (e, full, rows) in plan.items} if plan else {}
        # 1. activation set
        Be = {}
        for b in range(B):
            for e in ids[b]:
                Be[int(e)] = Be.get(int(e), 0) + 1
        A = sorted((e for e in Be if self.is_local(e)), key=lambda e: (-Be[e], e))
        Aset = set(A)
        # 2. stats (pre-increment ranks)
        self.stats[i].observe(ids, plan.ranking if plan is not None else None)
        tr = StepTrace()
        # 3. classify
        on = self.cache_on(i)
        cls = {}
        for e in A:
            cached = on and e in self.cache[i]
            p = planned.get(e)
            whole_bottom = p is not None and not p[0] and p[1] == I - self.I_top[i]
            whole_expert = p is not None and p[0] and p[1] == I
            if (cached and (self.I_top[i] == I or whole_bottom)) or whole_expert:
                c = ALPHA
            elif cached:
                c = BETA
            else:
                c = GAMMA
            cls[e] = c
            tr.act.append((e, c))
        # 4. counters
        s = self.step_no[i]
        for e in range(N):
            if e in Aset:
                self.mu[i][e] += Be[e]
                self.nu[i][e] = 0
                self.last[i][e] = s
            else:
                self.nu[i][e] += 1
        self.step_no[i] = s + 1
        # 5. admission
        d2d = 0
        if on:
            for e in A:
                if e in self.cache[i]:
                    continue
                if len(self.cache[i]) < self.C[i]:
                    self.cache[i].add(e)
                    tr.adm.append((e, ADM_FREE))
                    victim = ADM_FREE
                else:
                    cands = sorted(x for x in self.cache[i] if x not in Aset)
                    if not cands:
                        tr.adm.append((e, ADM_NONE))
                        continue
                    if cfg.policy == P.RND:
                        self.rnd[i], z = P.splitmix64_next(self.rnd[i])
                        victim = cands[z % len(cands)]
                    else:
                        keyf = lambda x: P.policy_key(cfg.policy, self.mu[i][x], self.nu[i][x], self.last[i][x], cfg.rho, cfg.omega)
                        victim = min(cands, key=lambda x: (keyf(x), -self.nu[i][x], x))
                    self.cache[i].remove(victim)
                    self.cache[i].add(e)
                    tr.adm.append((e, victim))
                if cls[e] == ALPHA or (e in planned and planned[e][0]):
                    # full expert (or its prefix, Q30) arrived by prefetch: D2D its top rows
                    d2d += 2 * self.I_top[i] * self.row_bytes
        # 6. bytes
        rb = self.row_bytes
        for e in A:
            if cls[e] == BETA:   # minus a prefetched bottom prefix (Q30)
                pre = planned[e][1] if e in planned and not planned[e][0] else 0
                tr.pcie_ondemand += (I - self.I_top[i] - pre) * rb
            elif cls[e] == GAMMA:   # minus a prefetched prefix of the full expert (Q30)
                pre = planned[e][1] if e in planned and planned[e][0] else 0
                tr.pcie_ondemand += (I - pre) * rb
        # 7. plan next layer
        n_router = 1
        if next_layer is not None and ranking_next is not None:
            n_router = 2
            self.pending = self._plan(next_layer, np.asarray(ranking_next))
            tr.plan = [(e, f) for (e, f, _) in self.pending.items]
            tr.pcie_prefetch = sum(r for (_, _, r) in self.pending.items) * rb
        else:
            self.pending = None      # a step always consumes (or discards) the pending plan
        tr.hbm = (len(A) * I * rb + self.n_shared * self.shared_rows() * rb + n_router * N * self.d * 2
                  + B * self.d * 2 + B * self.d * 4 + d2d + tr.pcie_ondemand + tr.pcie_prefetch)
        return tr
