// Index lists of the token-sharded expert-parallel exchange (prefill config 5).
// Pure C++: used by the library (moepic_api.cpp) and exported for CPU tests (moepic_ep_plan).
//
// G ranks hold Bl tokens each; global token t = r*Bl + i lives on rank r.  Expert e is owned by
// rank e*G/N.  S_q = the tokens (ascending t) with at least one of their K experts on rank q: the
// sub-batch rank q computes.  Dispatch sends each token row once per destination rank; combine
// returns, per (token, rank), that rank's weighted partial sum; the token's owner adds them in
// rank order.
#pragma once

#include <cstdint>
#include <vector>

namespace moepic {

struct EpLists {
  // dispatch: entries of this rank, grouped by destination rank, tokens ascending
  std::vector<int32_t> d_tok, d_dst, d_row;   // local token, destination rank, row in S_dst
  // the sub-batch S_me: global tokens; for each row j its owner rank and row in the owner's
  // combine buffer
  std::vector<int32_t> sub, c_dst, c_row;
  // reduce: for each local token, rows of this rank's combine buffer (owner rank ascending)
  std::vector<int32_t> r_off, r_row;
  std::vector<int32_t> n_send, n_recv;         // [G]: dispatch rows to / from each rank
  int32_t comb_rows = 0;                       // rows of this rank's combine buffer
};

// ids_all [G*Bl][K]; returns false on an expert id outside [0, N)
bool ep_plan(const int32_t* ids_all, int N, int K, int G, int me, int Bl, EpLists& out);

}  // namespace moepic
