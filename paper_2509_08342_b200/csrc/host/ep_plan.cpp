// Token-sharded expert-parallel exchange lists (ep_plan.hpp).
#include "ep_plan.hpp"

namespace moepic {

bool ep_plan(const int32_t* ids_all, int N, int K, int G, int me, int Bl, EpLists& o) {
  const int T = G * Bl;
  std::vector<uint32_t> mask(T, 0);   // destination ranks of each token
  for (int t = 0; t < T; ++t)
    for (int k = 0; k < K; ++k) {
      const int e = ids_all[(size_t)t * K + k];
      if (e < 0 || e >= N) return false;
      mask[t] |= 1u << (int)((int64_t)e * G / N);
    }
  // pos[q][t]: row of token t in S_q (or -1); cnt[q][r]: |S_q ∩ tokens(r)|
  std::vector<int32_t> pos((size_t)G * T, -1);
  std::vector<int32_t> cnt((size_t)G * G, 0);
  for (int q = 0; q < G; ++q) {
    int32_t n = 0;
    for (int t = 0; t < T; ++t)
      if (mask[t] >> q & 1u) {
        pos[(size_t)q * T + t] = n++;
        cnt[(size_t)q * G + t / Bl]++;
      }
  }
  // seg[r][q]: first row of the segment "returned by rank q" in rank r's combine buffer
  auto seg = [&](int r, int q) {
    int32_t s = 0;
    for (int q2 = 0; q2 < q; ++q2) s += cnt[(size_t)q2 * G + r];
    return s;
  };
  o = EpLists();
  o.n_send.assign(G, 0);
  o.n_recv.assign(G, 0);
  for (int q = 0; q < G; ++q)
    for (int i = 0; i < Bl; ++i) {
      const int t = me * Bl + i;
      if (!(mask[t] >> q & 1u)) continue;
      o.d_tok.push_back(i);
      o.d_dst.push_back(q);
      o.d_row.push_back(pos[(size_t)q * T + t]);
      o.n_send[q]++;
    }
  std::vector<int32_t> k_in_seg(G, 0);   // running index of tokens of rank r inside S_me
  for (int t = 0; t < T; ++t) {
    if (!(mask[t] >> me & 1u)) continue;
    const int r = t / Bl;
    o.sub.push_back(t);
    o.c_dst.push_back(r);
    o.c_row.push_back(seg(r, me) + k_in_seg[r]++);
    o.n_recv[r]++;
  }
  o.r_off.assign(Bl + 1, 0);
  std::vector<int32_t> seen(G, 0);       // tokens of mine already listed per returning rank
  for (int i = 0; i < Bl; ++i) {
    const int t = me * Bl + i;
    for (int q = 0; q < G; ++q)
      if (mask[t] >> q & 1u) o.r_row.push_back(seg(me, q) + seen[q]++);
    o.r_off[i + 1] = (int32_t)o.r_row.size();
  }
  o.comb_rows = seg(me, G);
  return true;
}

}  // namespace moepic
