// Host control plane of the MoEpic library: cache manager (LCP Eq. 4 / LRU / LFU / RND),
// activation classification, admission, prefetch planner,
// statistics H/P/PH and the Alg. 1 configurator.
//
// Pure C++17, no CUDA: the same object runs inside the library (moepic_api.cpp) and under the
// host-only test ABI (include/moepic_hostsim.h).  Floating point follows the canonical written
// order of DESIGN.md §Alg1 and is compiled with -ffp-contract=off -fno-fast-math so the results
// are bit-identical to any other IEEE implementation of the same expressions.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace moepic {

enum Policy { kLCP = 0, kLRU = 1, kLFU = 2, kRND = 3 };
enum Cls { kAlpha = 0, kBeta = 1, kGamma = 2 };
constexpr int32_t kAdmFree = -1;
constexpr int32_t kAdmNone = -2;

// ---------------------------------------------------------------- RNG
uint64_t splitmix64_next(uint64_t& state);
uint64_t layer_stream_seed(uint64_t seed, int layer, uint64_t salt);
std::vector<int32_t> fisher_yates(int n, uint64_t& state);

// ---------------------------------------------------------------- statistics
struct Stats {
  int N = 0, K = 0;
  int64_t q = 0, q_pred = 0;
  std::vector<int64_t> freq;            // [N]
  std::vector<int64_t> rank_hit;        // [N+1], index = frequency rank 1..N
  std::vector<int64_t> pred_hit;        // [N+1], index = predicted position y 1..N
  std::vector<int64_t> pred_rank;       // [(N+1)*(N+1)], [y][r]
  // prefix caches (rebuilt lazily after observe)
  mutable bool dirty = true;
  mutable std::vector<int64_t> hit_prefix;    // [N+1]
  mutable std::vector<int64_t> pred_prefix;   // [(N+1)*(N+1)]

  void init(int n, int k);
  void observe(const int32_t* ids, int B, int K, const int32_t* ranking /* may be null */);
  double H(int C) const;
  double P(int y) const;
  double PH(int y, int C) const;

 private:
  void rebuild() const;
};

// ---------------------------------------------------------------- configurator (Alg. 1)
struct SubResult { int C; double theta, m, T, window_next; int Y; };   // Y: prefetches fitting the window
SubResult solve_subproblem(const Stats& st, double V, double W, int K, int N, double U_b,
                           double t_load, double t_cexp, double t_moe, double t_att);
void expert_split(const std::vector<Stats>& st, const std::vector<double>& V, int K, int N,
                  double U_b, double t_att, double t_moe, double t_head, double t_load,
                  std::vector<double>& T, std::vector<double>& theta, std::vector<int>& C,
                  std::vector<int>* Y = nullptr);
// returns iterations; V is updated in place
int vram_allocation(const std::vector<Stats>& st, std::vector<double>& V, double V_e, double zeta,
                    int K, int N, double U_b, double t_att, double t_moe, double t_head,
                    double t_load, std::vector<double>& theta, std::vector<int>& C, bool& converged,
                    std::vector<int>* Y = nullptr);

// ---------------------------------------------------------------- cache + planner state
struct PlanItem {
  int32_t expert;
  bool full;
  int32_t rows;     // rows to copy: I - I_top (bottom) or I (full)
  int64_t buf_row;  // first row inside the plan region of the target buffer
};

struct Plan {
  bool valid = false;
  int target = -1;      // layer the plan serves
  int buf = -1;         // ping-pong half holding it (device side)
  std::vector<PlanItem> items;
  std::vector<int32_t> ranking;   // R' used to build it (feeds P / PH of the target layer)
};

struct LayerState {
  std::vector<int64_t> mu, nu, last;
  int64_t step_no = 0;
  std::vector<int32_t> slot_of;      // expert -> slot or -1
  std::vector<int32_t> slot_expert;  // slot -> expert or -1
  int n_cached = 0;
  int C = 0, I_top = 0;
  double V = 0.0;
  int Y = -1;        // Alg. 1's prefetch count (Eq. 10) when the config came from the solver
  uint64_t rnd = 0;
  Stats st;
  bool cache_on() const { return C > 0 && I_top > 0; }
  bool cached(int e) const { return cache_on() && slot_of[e] >= 0; }
};

struct CacheParams {
  double v_e = 0;
  std::vector<double> v_i, theta_i;   // empty -> defaults
  bool use_solver = false;
  int policy = kLCP;
  double rho = 0.25;
  int omega = 128;
  double zeta = 0.01;
  double t_att = 0, t_moe = 0, t_head = 0, t_load = 0;
  std::vector<int32_t> y_cap;         // empty -> N
  std::vector<int64_t> pf_rows;       // reading Q30: per-layer prefetch window in rows (empty -> none)
  bool prefetch = true;
  uint64_t seed = 0;
};

struct Admission { int32_t expert, victim, slot; bool d2d_from_plan; };

struct StepResult {
  std::vector<int32_t> A;      // distinct activated (local) experts, (B_e desc, id asc)
  std::vector<int32_t> Be;     // tokens per A entry
  std::vector<int8_t> cls;     // per A entry
  std::vector<int32_t> plan_idx;  // per A entry: index into the used plan's items or -1
  std::vector<Admission> adm;
  uint64_t pcie_ondemand = 0, d2d_bytes = 0;
  int alpha = 0, beta = 0, gamma = 0, pred_hits = 0;
};

class ControlPlane {
 public:
  int L, N, K, d, I, g, U_b, n_shared, ep_rank, ep_size;
  int64_t row_bytes;
  std::vector<LayerState> layers;
  CacheParams cfg;
  bool configured = false;
  bool solver_y_cap = true;          // cap the plan at Alg. 1's Y_i (reading Q27); off only in experiments
  std::vector<double> V;             // current allocation (Alg. 1 state)

  ControlPlane(int L, int N, int K, int d, int I, int g, int U_b, int n_shared, int ep_rank,
               int ep_size);
  bool is_local(int e) const { return (int64_t)e * ep_size / N == ep_rank; }

  // Validate + compute the new configuration.  On success layers[i].{C, I_top, V, slots} are
  // updated and the cached set is re-laid out.  Returns "" or an error string.
  std::string configure(const CacheParams& p, uint64_t slot_pool_rows);

  // One layer step (state before the call is what classification sees).  `plan` is the plan
  // made for this layer (or null).  ids: [B][K].  step = classify + commit; the library issues
  // the copies that classification alone decides (beta bottoms) between the two.
  void step(int layer, const int32_t* ids, int B, const Plan* plan, StepResult& out);
  // activation set A (B_e desc, id asc) and classes against the state before the step
  void classify(int layer, const int32_t* ids, int B, const Plan* plan, StepResult& out);
  // statistics, counters, admissions and on-demand bytes of a classified step
  void commit(int layer, const int32_t* ids, int B, const Plan* plan, StepResult& out);

  // Build the prefetch plan for layer j from ranking R'.
  void make_plan(int j, const int32_t* ranking, Plan& out) const;
};

}  // namespace moepic
