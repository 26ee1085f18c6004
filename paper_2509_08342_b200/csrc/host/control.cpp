// Host control plane implementation — see control.hpp.  Compiled with -ffp-contract=off.
#include <cstdlib>
#include "control.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>

namespace moepic {

// ================================================================ RNG
uint64_t splitmix64_next(uint64_t& state) {
  state += 0x9E3779B97F4A7C15ull;
  uint64_t z = state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint64_t layer_stream_seed(uint64_t seed, int layer, uint64_t salt) {
  uint64_t s = seed ^ (0xD1B54A32D192ED03ull * (uint64_t)(layer + 1)) ^ (0x8CB92BA72F3D8DD7ull * salt);
  return splitmix64_next(s);
}

std::vector<int32_t> fisher_yates(int n, uint64_t& state) {
  std::vector<int32_t> p(n);
  std::iota(p.begin(), p.end(), 0);
  for (int i = n - 1; i > 0; --i) {
    uint64_t z = splitmix64_next(state);
    int j = (int)(z % (uint64_t)(i + 1));
    std::swap(p[i], p[j]);
  }
  return p;
}

// ================================================================ statistics
void Stats::init(int n, int k) {
  N = n; K = k; q = q_pred = 0;
  freq.assign(N, 0);
  rank_hit.assign(N + 1, 0);
  pred_hit.assign(N + 1, 0);
  pred_rank.assign((size_t)(N + 1) * (N + 1), 0);
  dirty = true;
}

void Stats::observe(const int32_t* ids, int B, int Kk, const int32_t* ranking) {
  // frequency rank on pre-step counts: (freq desc, id asc), 1-based
  std::vector<int32_t> order(N);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    if (freq[a] != freq[b]) return freq[a] > freq[b];
    return a < b;
  });
  std::vector<int32_t> rank(N);
  for (int r = 0; r < N; ++r) rank[order[r]] = r + 1;
  std::vector<char> act(N);
  for (int b = 0; b < B; ++b) {
    std::fill(act.begin(), act.end(), 0);
    for (int k = 0; k < Kk; ++k) {
      int e = ids[b * Kk + k];
      act[e] = 1;
      rank_hit[rank[e]] += 1;
    }
    if (ranking) {
      for (int y = 1; y <= N; ++y) {
        int e = ranking[y - 1];
        if (act[e]) pred_hit[y] += 1;
        pred_rank[(size_t)y * (N + 1) + rank[e]] += 1;
      }
    }
  }
  q += B;
  if (ranking) q_pred += B;
  for (int b = 0; b < B; ++b)
    for (int k = 0; k < Kk; ++k) freq[ids[b * Kk + k]] += 1;
  dirty = true;
}

void Stats::rebuild() const {
  hit_prefix.assign(N + 1, 0);
  for (int C = 1; C <= N; ++C) hit_prefix[C] = hit_prefix[C - 1] + rank_hit[C];
  pred_prefix.assign((size_t)(N + 1) * (N + 1), 0);
  for (int y = 1; y <= N; ++y)
    for (int C = 1; C <= N; ++C)
      pred_prefix[(size_t)y * (N + 1) + C] =
          pred_prefix[(size_t)y * (N + 1) + C - 1] + pred_rank[(size_t)y * (N + 1) + C];
  dirty = false;
}

double Stats::H(int C) const {
  if (dirty) rebuild();
  return (double)hit_prefix[C] / (double)(q * K);
}
double Stats::P(int y) const {
  if (q_pred == 0) return 0.0;
  return (double)pred_hit[y] / (double)q_pred;
}
double Stats::PH(int y, int C) const {
  if (q_pred == 0) return 0.0;
  if (dirty) rebuild();
  return (double)pred_prefix[(size_t)y * (N + 1) + C] / (double)q_pred;
}

// ================================================================ Alg. 1
SubResult solve_subproblem(const Stats& st, double V, double W, int K, int N, double U_b,
                           double t_load, double t_cexp, double t_moe, double t_att) {
  int C_lo = std::max(1, (int)std::ceil(V - 1e-9));
  if (C_lo > N) C_lo = N;
  bool have = false;
  int best_Y = 0;
  int best_C = 0;
  double best_theta = 0.0, best_m = 0.0;
  const double Kd = (double)K;
  for (int C = C_lo; C <= N; ++C) {
    double theta = V / (double)C;
    if (theta > 1.0) theta = 1.0;
    double m = (Kd * st.H(C)) * theta;
    double cum = 0.0, fcum = 0.0;
    int Y = 0;
    for (int y = 1; y <= N; ++y) {
      double f = 1.0 - st.PH(y, C) * theta;
      double c = f * t_load;
      if (cum + c > W || fcum + f > U_b) break;
      cum = cum + c;
      fcum = fcum + f;
      m = m + f * st.P(y);
      Y = y;
    }
    if (!have || m > best_m) { have = true; best_C = C; best_theta = theta; best_m = m; best_Y = Y; }
  }
  SubResult r;
  r.C = best_C;
  r.theta = best_theta;
  r.m = best_m;
  double x = (Kd - best_m) * t_load - best_m * t_cexp;
  r.T = std::max(0.0, x);
  r.window_next = (t_moe - std::min(best_m * t_cexp, (Kd - best_m) * t_load)) + t_att;
  r.Y = best_Y;
  return r;
}

void expert_split(const std::vector<Stats>& st, const std::vector<double>& V, int K, int N,
                  double U_b, double t_att, double t_moe, double t_head, double t_load,
                  std::vector<double>& T, std::vector<double>& theta, std::vector<int>& C,
                  std::vector<int>* Y) {
  if (Y) Y->assign(V.size(), 0);
  const double t_cexp = t_moe / (double)K;
  double W = t_head + t_att;
  size_t L = V.size();
  T.resize(L); theta.resize(L); C.resize(L);
  for (size_t i = 0; i < L; ++i) {
    SubResult r = solve_subproblem(st[i], V[i], W, K, N, U_b, t_load, t_cexp, t_moe, t_att);
    T[i] = r.T; theta[i] = r.theta; C[i] = r.C;
    if (Y) (*Y)[i] = r.Y;
    W = r.window_next;
  }
}

int vram_allocation(const std::vector<Stats>& st, std::vector<double>& V, double V_e, double zeta,
                    int K, int N, double U_b, double t_att, double t_moe, double t_head,
                    double t_load, std::vector<double>& theta, std::vector<int>& C, bool& converged,
                    std::vector<int>* Y) {
  auto ys = [&](const std::vector<double>& vv) {
    if (!Y) return;
    std::vector<double> t_, th_;
    std::vector<int> c_;
    expert_split(st, vv, K, N, U_b, t_att, t_moe, t_head, t_load, t_, th_, c_, Y);
  };
  const int L = (int)V.size();
  const double delta = zeta * V_e;
  const int cap = 10 * L * (int)std::ceil(1.0 / zeta);
  std::vector<double> T1, T2, T3, T4, th, th_tmp, Vp(L), Vm(L), Vn;
  std::vector<int> C1, c_tmp;
  for (int it = 0; it < cap; ++it) {
    expert_split(st, V, K, N, U_b, t_att, t_moe, t_head, t_load, T1, th, C1);
    for (int i = 0; i < L; ++i) { Vp[i] = V[i] + delta; Vm[i] = std::max(0.0, V[i] - delta); }
    expert_split(st, Vp, K, N, U_b, t_att, t_moe, t_head, t_load, T2, th_tmp, c_tmp);
    expert_split(st, Vm, K, N, U_b, t_att, t_moe, t_head, t_load, T3, th_tmp, c_tmp);
    int i1 = 0;
    for (int i = 1; i < L; ++i)
      if (T1[i] - T2[i] > T1[i1] - T2[i1]) i1 = i;
    int i2 = -1;
    for (int i = 0; i < L; ++i) {
      if (i == i1 || V[i] + 1e-9 < delta) continue;
      if (i2 < 0 || T3[i] - T1[i] < T3[i2] - T1[i2]) i2 = i;
    }
    if (i2 < 0) { theta = th; C = C1; converged = true; ys(V); return it; }
    Vn = V;
    Vn[i1] = Vn[i1] + delta;
    Vn[i2] = Vn[i2] - delta;
    if (Vn[i2] < 0.0) Vn[i2] = 0.0;
    expert_split(st, Vn, K, N, U_b, t_att, t_moe, t_head, t_load, T4, th_tmp, c_tmp);
    double s = 0.0;
    for (int i = 0; i < L; ++i) s = s + (T4[i] - T1[i]);
    if (s >= 0.0) { theta = th; C = C1; converged = true; ys(V); return it; }
    V = Vn;
  }
  expert_split(st, V, K, N, U_b, t_att, t_moe, t_head, t_load, T1, theta, C, Y);
  converged = false;
  return cap;
}

// ================================================================ control plane
ControlPlane::ControlPlane(int L_, int N_, int K_, int d_, int I_, int g_, int U_b_, int n_shared_,
                           int ep_rank_, int ep_size_)
    : L(L_), N(N_), K(K_), d(d_), I(I_), g(g_), U_b(U_b_), n_shared(n_shared_), ep_rank(ep_rank_),
      ep_size(ep_size_) {
  row_bytes = 6ll * d;
  layers.resize(L);
  for (auto& l : layers) {
    l.mu.assign(N, 0);
    l.nu.assign(N, 0);
    l.last.assign(N, -1);
    l.slot_of.assign(N, -1);
    l.st.init(N, K);
  }
}

static double policy_key(int policy, const LayerState& l, int e, double rho, int omega) {
  switch (policy) {
    case kLCP: return (double)l.mu[e] * std::pow(rho, (double)l.nu[e] / (double)omega);  // Eq. 4
    case kLRU: return (double)l.last[e];
    default:   return (double)l.mu[e];   // kLFU
  }
}

std::string ControlPlane::configure(const CacheParams& p, uint64_t slot_pool_rows) {
  // ---- validation (no state change on error)
  if (!(p.v_e >= 0.0)) return "v_e must be >= 0";
  if (p.policy < 0 || p.policy > 3) return "policy out of range";
  if (!(p.rho > 0.0 && p.rho < 1.0)) return "rho must be in (0,1)";
  if (p.omega < 1) return "omega must be >= 1";
  if (!(p.zeta > 0.0 && p.zeta < 1.0)) return "zeta must be in (0,1)";
  if (!p.v_i.empty() && (int)p.v_i.size() != L) return "v_i must have L entries";
  if (!p.theta_i.empty() && (int)p.theta_i.size() != L) return "theta_i must have L entries";
  if (!p.y_cap.empty() && (int)p.y_cap.size() != L) return "y_cap_i must have L entries";
  if (!p.pf_rows.empty() && (int)p.pf_rows.size() != L) return "prefetch_rows_i must have L entries";
  for (int64_t w : p.pf_rows)
    if (w < 0) return "prefetch_rows_i must be >= 0";
  std::vector<double> Vnew;
  std::vector<double> thetas;
  std::vector<int> Cs(L);
  std::vector<int> Ys;   // Eq. 10's Y per layer (solver only): caps the planner (reading Q27)
  if (p.use_solver) {
    for (int i = 0; i < L; ++i)
      if (layers[i].st.q == 0) return "empty accumulator (layer " + std::to_string(i) + ")";
    if (!(p.t_load > 0.0) || !(p.t_moe > 0.0)) return "t_load_exp and t_moe must be > 0 with use_solver";
    if (configured) Vnew = V;
    else if (!p.v_i.empty()) Vnew = p.v_i;
    else Vnew.assign(L, p.v_e / (double)L);
    std::vector<Stats> st(L);
    for (int i = 0; i < L; ++i) st[i] = layers[i].st;
    bool conv = false;
    vram_allocation(st, Vnew, p.v_e, p.zeta, K, N, (double)U_b, p.t_att, p.t_moe, p.t_head, p.t_load,
                    thetas, Cs, conv, &Ys);
  } else {
    Vnew = p.v_i.empty() ? std::vector<double>(L, p.v_e / (double)L) : p.v_i;
    thetas = p.theta_i.empty() ? std::vector<double>(L, 0.5) : p.theta_i;
    double s = 0.0;
    for (double v : Vnew) s = s + v;
    if (s > p.v_e + 1e-9) return "sum v_i exceeds v_e";
    for (int i = 0; i < L; ++i) {
      if (!(thetas[i] > 0.0 && thetas[i] <= 1.0)) return "theta_i[" + std::to_string(i) + "] must be in (0,1]";
      if (!(Vnew[i] >= 0.0)) return "v_i[" + std::to_string(i) + "] must be >= 0";
      int c = (int)std::floor(Vnew[i] / thetas[i] + 1e-9);
      Cs[i] = std::min(N, c);
    }
  }
  std::vector<int> Itop(L);
  uint64_t rows_needed = 0;
  for (int i = 0; i < L; ++i) {
    int it = g * (int)std::floor(thetas[i] * (double)I / (double)g + 1e-9);
    Itop[i] = std::min(I, it);
    if (Cs[i] > 0 && Itop[i] > 0) rows_needed += (uint64_t)Cs[i] * (uint64_t)Itop[i];
  }
  if (rows_needed > slot_pool_rows) return "configuration exceeds the slot pool (v_e_max)";

  // ---- commit
  if (!configured)
    for (int i = 0; i < L; ++i) layers[i].rnd = layer_stream_seed(p.seed, i, 1);
  cfg = p;
  V = Vnew;
  for (int i = 0; i < L; ++i) {
    LayerState& l = layers[i];
    l.C = Cs[i];
    l.I_top = Itop[i];
    l.V = Vnew[i];
    l.Y = Ys.empty() ? -1 : Ys[i];
    std::fill(l.slot_of.begin(), l.slot_of.end(), -1);
    l.slot_expert.assign(std::max(0, l.C), -1);
    l.n_cached = 0;
    if (!l.cache_on()) continue;
    std::vector<int32_t> order;
    if (l.st.q == 0) {                     // cold start: "selected randomly" (Q14)
      if (p.seed == 0) {
        order.resize(N);
        std::iota(order.begin(), order.end(), 0);
      } else {
        uint64_t s = layer_stream_seed(p.seed, i, 2);
        order = fisher_yates(N, s);
      }
    } else if (p.policy == kRND) {
      order = fisher_yates(N, l.rnd);
    } else {                               // rank by cache priority
      order.resize(N);
      std::iota(order.begin(), order.end(), 0);
      std::vector<double> key(N);
      for (int e = 0; e < N; ++e) key[e] = policy_key(p.policy, l, e, p.rho, p.omega);
      std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
        if (key[a] != key[b]) return key[a] > key[b];
        if (l.nu[a] != l.nu[b]) return l.nu[a] < l.nu[b];
        return a < b;
      });
    }
    // EP: only local experts are cached on this rank
    int slot = 0;
    for (int e : order) {
      if (slot >= l.C) break;
      if (!is_local(e)) continue;
      l.slot_of[e] = slot;
      l.slot_expert[slot] = e;
      ++slot;
    }
    l.n_cached = slot;
  }
  configured = true;
  return "";
}

void ControlPlane::step(int layer, const int32_t* ids, int B, const Plan* plan, StepResult& out) {
  classify(layer, ids, B, plan, out);
  commit(layer, ids, B, plan, out);
}

void ControlPlane::classify(int layer, const int32_t* ids, int B, const Plan* plan, StepResult& out) {
  const LayerState& l = layers[layer];
  out = StepResult();
  // 1. activation set (local experts), order (B_e desc, id asc)
  std::vector<int32_t> be(N, 0);
  for (int b = 0; b < B; ++b)
    for (int k = 0; k < K; ++k) be[ids[b * K + k]] += 1;
  for (int e = 0; e < N; ++e)
    if (be[e] > 0 && is_local(e)) out.A.push_back(e);
  std::stable_sort(out.A.begin(), out.A.end(), [&](int a, int b) {
    if (be[a] != be[b]) return be[a] > be[b];
    return a < b;
  });
  // 3. classification against the state before the step
  std::vector<int32_t> pidx(N, -1);
  if (plan)
    for (size_t j = 0; j < plan->items.size(); ++j) pidx[plan->items[j].expert] = (int32_t)j;
  for (int e : out.A) {
    bool cached = l.cached(e);
    int pj = pidx[e];
    // a bottom item counts as loaded only if it holds the whole bottom (Q30: a window-cut item
    // holds a prefix and leaves the rest on demand)
    bool p_bottom = pj >= 0 && !plan->items[pj].full && plan->items[pj].rows == I - l.I_top;
    bool p_full = pj >= 0 && plan->items[pj].full && plan->items[pj].rows == I;
    int8_t c;
    if ((cached && (l.I_top == I || p_bottom)) || p_full) c = kAlpha;
    else if (cached) c = kBeta;
    else c = kGamma;
    out.Be.push_back(be[e]);
    out.cls.push_back(c);
    out.plan_idx.push_back(pj);
    if (c == kAlpha) ++out.alpha; else if (c == kBeta) ++out.beta; else ++out.gamma;
    if (pj >= 0) ++out.pred_hits;
  }
}

void ControlPlane::commit(int layer, const int32_t* ids, int B, const Plan* plan, StepResult& out) {
  LayerState& l = layers[layer];
  // 2. statistics on pre-step counts, prediction = the ranking that planned this layer
  l.st.observe(ids, B, K, plan ? plan->ranking.data() : nullptr);
  std::vector<char> inA(N, 0);
  std::vector<int32_t> be(N, 0);
  for (size_t a = 0; a < out.A.size(); ++a) {
    inA[out.A[a]] = 1;
    be[out.A[a]] = out.Be[a];
  }
  // 4. counters: update first, then choose victims (Q12)
  const int64_t s = l.step_no;
  for (int e = 0; e < N; ++e) {
    if (inA[e]) { l.mu[e] += be[e]; l.nu[e] = 0; l.last[e] = s; }
    else l.nu[e] += 1;
  }
  l.step_no = s + 1;
  // 5. admission in A order (Q11; victims exclude A).  The keys depend only on
  // (mu, nu, last), fixed once the counters are updated, so each candidate's key is computed once
  // per step however many admissions look at it.
  std::vector<double> key;
  if (l.cache_on()) {
    for (size_t a = 0; a < out.A.size(); ++a) {
      int e = out.A[a];
      if (l.slot_of[e] >= 0) continue;
      Admission ad{e, kAdmNone, -1, false};
      if (l.n_cached < l.C) {
        int slot = 0;
        while (l.slot_expert[slot] >= 0) ++slot;
        ad.victim = kAdmFree;
        ad.slot = slot;
        l.slot_expert[slot] = e;
        l.slot_of[e] = slot;
        ++l.n_cached;
      } else {
        std::vector<int32_t> cands;
        for (int x = 0; x < N; ++x)
          if (l.slot_of[x] >= 0 && !inA[x]) cands.push_back(x);
        if (cands.empty()) { out.adm.push_back(ad); continue; }
        int v;
        if (cfg.policy == kRND) {
          uint64_t z = splitmix64_next(l.rnd);
          v = cands[(size_t)(z % (uint64_t)cands.size())];
        } else {
          if (key.empty()) {
            key.assign(N, 0.0);
            for (int x = 0; x < N; ++x)
              if (l.slot_of[x] >= 0 && !inA[x]) key[x] = policy_key(cfg.policy, l, x, cfg.rho, cfg.omega);
          }
          v = cands[0];
          double kv = key[v];
          for (size_t j = 1; j < cands.size(); ++j) {
            int x = cands[j];
            double kx = key[x];
            if (kx < kv || (kx == kv && l.nu[x] > l.nu[v])) { v = x; kv = kx; }
            // equal key and nu: keep the smaller id (cands ascending)
          }
        }
        ad.victim = v;
        ad.slot = l.slot_of[v];
        l.slot_of[v] = -1;
        l.slot_expert[ad.slot] = e;
        l.slot_of[e] = ad.slot;
      }
      // full expert (or its prefix, Q30) arrived by prefetch: its top rows are copied on the device
      ad.d2d_from_plan = out.cls[a] == kAlpha || (out.plan_idx[a] >= 0 && plan->items[out.plan_idx[a]].full);
      if (ad.d2d_from_plan) out.d2d_bytes += 2ull * (uint64_t)l.I_top * (uint64_t)row_bytes;
      out.adm.push_back(ad);
    }
  }
  // 6. on-demand PCIe bytes
  for (size_t a = 0; a < out.A.size(); ++a) {
    if (out.cls[a] == kBeta) {
      const int pj = out.plan_idx[a];
      const int pre = pj >= 0 && !plan->items[pj].full ? plan->items[pj].rows : 0;   // Q30 prefix
      out.pcie_ondemand += (uint64_t)(I - l.I_top - pre) * (uint64_t)row_bytes;
    }
    else if (out.cls[a] == kGamma) {
      const int pj = out.plan_idx[a];
      const int pre = pj >= 0 && plan->items[pj].full ? plan->items[pj].rows : 0;   // Q30 prefix
      out.pcie_ondemand += (uint64_t)(I - pre) * (uint64_t)row_bytes;
    }
  }
}

void ControlPlane::make_plan(int j, const int32_t* ranking, Plan& out) const {
  out.valid = true;
  out.target = j;
  out.items.clear();
  out.ranking.assign(ranking, ranking + N);
  if (!cfg.prefetch) return;
  const LayerState& l = layers[j];
  int64_t cap_rows = (int64_t)U_b * I;
  int ycap = cfg.y_cap.empty() ? N : cfg.y_cap[j];
  const bool window = !cfg.pf_rows.empty();   // Q30: the window replaces Alg. 1's count cap
  if (window) cap_rows = std::min(cap_rows, cfg.pf_rows[j]);
  else if (l.Y >= 0 && solver_y_cap) ycap = std::min(ycap, l.Y);
  int64_t used = 0;
  for (int y = 0; y < N; ++y) {
    int e = ranking[y];
    if ((int)out.items.size() >= ycap) break;
    if (!is_local(e)) continue;
    PlanItem it;
    it.expert = e;
    if (l.cached(e)) {
      it.rows = I - l.I_top;
      if (it.rows == 0) continue;
      it.full = false;
    } else {
      it.rows = I;
      it.full = true;
    }
    if (used + it.rows > cap_rows) {
      const int64_t part = (int64_t)g * ((cap_rows - used) / g);
      if (window && part > 0) {   // Q30: the cut item keeps its prefix
        it.rows = (int32_t)part;
        it.buf_row = used;
        out.items.push_back(it);
      }
      break;
    }
    it.buf_row = used;
    used += it.rows;
    out.items.push_back(it);
  }
}

}  // namespace moepic
