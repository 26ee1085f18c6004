"""MoEpic CPU oracle — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct fp64 implementation of what the split-expert MoE hot
path computes, written from the paper (/root/reference/PAPER.md, cited as P:<line>) with
the readings listed in DESIGN.md §Readings.  It shares no code with the CUDA library
(`paper_2509_08342_b200/`) and neither imports the other.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl
reference` leg may import it.  The product path never calls it; the library fails
loudly when its CUDA extension is missing.

Modules
  numeric       C-N: router logits (canonical fp64 order), top-K, Eq. 2 gate weights,
                SwiGLU experts, the dense MoE layer output, next-layer ranking (Eq. 3).
  policy        LCP priority (Eq. 4) and LRU/LFU/RND keys; splitmix64.
  stats         H_i(C), P_i(y), PH_i(y, C) accumulators.
  configurator  Alg. 1: ExpertSplit / VramAllocation with Eqs. 5-7, 9a/9b, 10.
  replay        C-S state machine: classification, counters, admission, bytes, the
                next-layer prefetch plan, re-layout; one step per layer_forward call.

Parity status: every function is pinned by tests/test_oracle_*.py (see DESIGN.md
§Pins).  Functions without an independent pin say "parity unpinned" in their docstring.
"""
