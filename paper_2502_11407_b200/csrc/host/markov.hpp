// Explicit construction-chain analysis (the reference's markov-verify
// module, markov.hpp:1-70 / markov.cpp:40-364): the paper's §IV-D claims —
// per-level irreducibility thanks to InvTile, aperiodicity, a per-level stationary distribution
// and the product-form value iteration of Eqs. 5-6 — checked on enumerable schedule spaces.
#pragma once

#include <string>
#include <vector>

#include "engine.hpp"

namespace gb {

struct ChainCaps {
  int max_states = 50000;
  int fixed_iteration = 10;  // annealing point the policy is frozen at (multiplier 1.5)
  bool enable_inv_tile = true;
  std::vector<int64_t> vthread_options{1, 2, 4, 8};
  int64_t max_tile_factor = 2;
  Mode mode = Mode::ReferenceCompat;
};

struct ChainEdge {
  int to = -1;
  double prob = 0.0;
  Action action;
  bool artificial = false;  // the absorbing self-loop, not a scheduling move
};

struct Chain {
  std::vector<Sched> states;
  std::vector<std::vector<ChainEdge>> rows;  // row-stochastic
  std::vector<int> level;
  std::vector<char> complete, absorbing;
  std::vector<double> terminal;  // 1/est_seconds at complete states, normalised to max 1

  int size() const { return static_cast<int>(rows.size()); }
  int max_level() const;
};

// Breadth-first closure of the unscheduled state under the engine's candidate policy at
// caps.fixed_iteration. States with no selectable action absorb with an artificial self-loop.
// Throws SpaceTooLarge past caps.max_states.
Chain enumerate_chain(const OpDesc& op, const HwModel& hw, const ChainCaps& caps);

// Per level 0..max_level: every weakly connected piece of the within-level subgraph is a single
// strongly connected component.
std::vector<bool> irreducible_per_level(const Chain& c, std::vector<int>* scc_counts = nullptr);

// Every within-level piece with an edge has cycle-length gcd 1 (BFS-depth gcd argument).
bool aperiodic(const Chain& c);
bool aperiodic_level(const Chain& c, int level);

// Whether power iteration from the uniform start converges on `level` (one SCC; if periodic,
// equal-sized cyclic classes).
bool power_iteration_converges(const Chain& c, int level);

// Stationary vector of the level-restricted, row-renormalised subchain by power iteration
// (L1 residual < 1e-12), indexed by global state id (0 off-level). Throws NotErgodic.
std::vector<double> stationary(const Chain& c, int level, int* sweeps = nullptr);

struct Values {
  std::vector<double> value;
  std::vector<int> policy;  // edge index into rows[i], -1 = none
  int iterations = 0;
};

// Eq. 6 Jacobi sweeps from V0 = terminal at complete states, 1 elsewhere, to a 1e-12 fixed
// point; throws NoConvergence past 10*|states| sweeps.
Values value_iteration(const Chain& c);

// The `analyze` report: counts, per-level SCCs / irreducibility / stationary entropy,
// aperiodicity, V(initial), the greedy policy path; with `detail` every state and edge too.
std::string analysis_json(const OpDesc& op, const HwModel& hw, const ChainCaps& caps, bool detail);

}  // namespace gb
