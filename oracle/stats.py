"""Statistics for the cache configurator (TEST INFRASTRUCTURE).

  H_i(C)    cache hit rate with cache size C: hits of the activated experts / (q K)
  P_i(y)    activation frequency of the y-th predicted expert / q
  PH_i(y,C) times the y-th predicted expert hits a size-C cache / q

Reading Q15: the counterfactual size-C cache is "the top-C
experts by running activation frequency" (frequency rank, ties by smaller id), ranks
computed on the counts BEFORE this step's increment.  Per layer-step with B tokens:
ranks are computed once on pre-step counts, then every token contributes (its K
activated experts to H; the batch ranking R' to P and PH), q += B, counts += B_e.
P / PH use q_pred (tokens that had a prediction) as their denominator.
"""
from __future__ import annotations

import numpy as np


class LayerStats:
    def __init__(self, N: int, K: int):
        self.N, self.K = N, K
        self.freq = np.zeros(N, dtype=np.int64)
        self.q = 0
        self.q_pred = 0
        self.rank_hit_hist = np.zeros(N + 1, dtype=np.int64)        # index r = 1..N
        self.pred_hit = np.zeros(N + 1, dtype=np.int64)             # index y = 1..N
        self.pred_rank_hist = np.zeros((N + 1, N + 1), dtype=np.int64)  # [y][r]

    def freq_rank(self) -> np.ndarray:
        """rank[e] in 1..N by (freq desc, id asc) on current counts."""
        order = sorted(range(self.N), key=lambda e: (-self.freq[e], e))
        rank = np.empty(self.N, dtype=np.int64)
        for r, e in enumerate(order):
            rank[e] = r + 1
        return rank

    def observe(self, ids: np.ndarray, ranking):
        """ids [B][K] activated experts; ranking = predicted R' for this layer or None."""
        rank = self.freq_rank()
        B = ids.shape[0]
        for b in range(B):
            act = set(int(x) for x in ids[b])
            for e in ids[b]:
                self.rank_hit_hist[rank[e]] += 1
            if ranking is not None:
                for y, e in enumerate(ranking, start=1):
                    if int(e) in act:
                        self.pred_hit[y] += 1
                    self.pred_rank_hist[y, rank[e]] += 1
        self.q += B
        if ranking is not None:
            self.q_pred += B
        for b in range(B):
            for e in ids[b]:
                self.freq[e] += 1

    # --- derived probabilities ---
    def H(self, C: int) -> float:
        return float(self.rank_hit_hist[1:C + 1].sum()) / float(self.q * self.K)

    def P(self, y: int) -> float:
        return float(self.pred_hit[y]) / float(self.q_pred) if self.q_pred else 0.0

    def PH(self, y: int, C: int) -> float:
        return float(self.pred_rank_hist[y, 1:C + 1].sum()) / float(self.q_pred) if self.q_pred else 0.0
