// Construction engine: the paper's Algorithm 1/2 annealed Markov walk over schedule states.
//
// Reference-compatible mode reproduces src/engine.cpp bit for bit — candidate order, benefit
// normalisation, the mt19937_64 draw sequence (roulette, then record), temperature halving,
// greedy completion (tree_baseline.cpp:13-27) and the final ranking/dedupe (engine.cpp:179-190).
// Differences that do not change results:
//   * restarts run on a thread pool (SPEC.md:334 permits it); each restart owns its rng stream
//     (derive_seed) and the pools are merged in restart order, so the ranked output is identical
//     to the sequential reference;
//   * states are fixed-size PODs and candidate evaluation is allocation-free.
// B200 mode (Mode::B200) keeps the same walk and adds device legality gates on the Cache action
// and a completion step that satisfies them, then ranks by estimate_b200.
#pragma once

#include <cstdint>
#include <functional>
#include <random>
#include <vector>

#include "cost.hpp"
#include "hw.hpp"
#include "op.hpp"
#include "sched.hpp"

namespace gb {

enum class Mode : int { ReferenceCompat = 0, B200 = 1 };

struct EngineCfg {
  double t0 = 1048576.0;  // 2^20: 20 halvings to threshold 1
  double threshold = 1.0;
  int restarts = 8;
  uint64_t seed = 0;
  int top_k = 10;
  std::vector<int64_t> vthread_options{1, 2, 4, 8};
  int64_t max_tile_factor = 2;
  Mode mode = Mode::ReferenceCompat;
  int threads = 0;  // 0 = min(restarts, hardware threads)
  bool enable_inv_tile = true;  // ActionSpace::enable_inv_tile (engine.hpp:31): chain analysis only
  void validate() const;  // throws ConfigError (engine.cpp:11-22)
};

struct Candidate {
  Action action;
  double benefit = 0.0;
  double probability = 0.0;  // 0 iff gated
};

struct Result {
  Sched state;
  Cost cost;
  std::vector<Action> trace;
  uint64_t seed = 0;
  int iterations = 0;
};

using Observer = std::function<void(const Sched&, const std::vector<Candidate>&, double temperature, int iteration)>;

double anneal_cache_multiplier(int iteration);
double record_probability(double temperature);
uint64_t derive_seed(uint64_t seed, int restart);
inline double uniform_unit(std::mt19937_64& rng) { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }

// Fills `out`; returns false (NoLegalAction) when every candidate is gated or none exists.
bool candidates(const OpDesc& op, const HwModel& hw, const Sched& s, const EngineCfg& cfg, int iteration,
                std::vector<Candidate>& out);
int roulette(const std::vector<Candidate>& c, std::mt19937_64& rng);  // throws EmptyCandidates

// One walk with cfg.seed used directly (engine.cpp:105-140): raw snapshots, no cost.
std::vector<Result> construct(const OpDesc& op, const HwModel& hw, const EngineCfg& cfg, const Observer& obs = nullptr);

// Greedy capacity-fitting completion (engine.cpp:149-163); false if some level never fits.
bool complete(const OpDesc& op, const HwModel& hw, Sched& s, std::vector<Action>& trace, Mode mode);
// tc_floor (B200 mode): never halve a tensor-core GEMM's level-1 k tile below two 128 B k-blocks.
bool greedy_fit_step(const OpDesc& op, const Sched& s, Action& out, bool tc_floor = false);

// Multi-restart optimize (engine.cpp:165-192): ranked, deduped, top_k.
std::vector<Result> optimize(const OpDesc& op, const HwModel& hw, const EngineCfg& cfg, const Observer& obs = nullptr);

// Roller-style beam baseline (tree_baseline.cpp:53-108), deterministic.
std::vector<Result> construct_tree(const OpDesc& op, const HwModel& hw, int beam_width, Mode mode);

// B200-mode device legality of a complete (or level-committed) state: threads per CTA,
// per-thread accumulators/registers, shared-memory staging of the level-1 input footprint.
bool b200_feasible(const OpDesc& op, const HwModel& hw, const Sched& s, int upto_level);

Cost cost_of(const OpDesc& op, const HwModel& hw, const Sched& s, Mode mode);

}  // namespace gb
