#include "engine.hpp"

#include <algorithm>
#include <cmath>
#include <thread>

#include "error.hpp"
#include "tcplan.hpp"

namespace gb {

void EngineCfg::validate() const {
  if (!(t0 > threshold && threshold > 0)) throw Error(Code::ConfigError, "need t0 > threshold > 0");
  if (restarts < 1) throw Error(Code::ConfigError, "restarts must be >= 1");
  if (top_k < 1) throw Error(Code::ConfigError, "top_k must be >= 1");
  if (max_tile_factor < 2 || !is_pow2(max_tile_factor))
    throw Error(Code::ConfigError, "max_tile_factor must be a power of two >= 2");
  if (vthread_options.empty()) throw Error(Code::ConfigError, "vthread_options is empty");
  for (int64_t v : vthread_options)
    if (!is_pow2(v)) throw Error(Code::ConfigError, "vthread options must be powers of two >= 1");
}

// The two annealing expressions are written exactly as the reference evaluates them
// (engine.cpp:24-30): same operand order, glibc exp/log, no contraction (-ffp-contract=off).
double anneal_cache_multiplier(int iteration) {
  return 3.0 / (1.0 + std::exp(-(std::log(5.0) / 10.0) * (iteration - 10)));
}

double record_probability(double temperature) {
  return 1.0 - 1.0 / (1.0 + std::exp(-0.5 * (-std::log(temperature) - 10.0)));
}

uint64_t derive_seed(uint64_t seed, int restart) {
  uint64_t z = seed + 0x9E3779B97F4A7C15ULL * static_cast<uint64_t>(restart + 1);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

namespace {

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

std::vector<int64_t> sorted_unique(std::vector<int64_t> v) {
  std::sort(v.begin(), v.end());
  v.erase(std::unique(v.begin(), v.end()), v.end());
  return v;
}

}  // namespace

// B200 legality of the levels committed so far:
//   level 1 committed: the CTA tile must leave at least one full wave of CTAs when the domain
//     is large enough to have one (148 SMs idle otherwise — the reference model has no
//     parallelism term and picks 2-CTA GEMV grids);
//   level L committed: threads/CTA in [32, max_threads_per_block], per-thread accumulators
//     (prod of spatial thread tiles) <= 64 so the thread tile lives in registers.
namespace {

// GEMMs the tensor cores run: their level-1 tile is a gemm_tc program (tcplan.hpp)
bool tc_gemm(const OpDesc& op) { return op.kind == Kind::Gemm && tensor_unit(exec_unit(op)); }

// K-atom floor of the tensor-core ring: the level-1 k tile holds at least two 128-byte k-blocks.
// Halving below it can never be undone by completion (it only halves), so B200-mode completion
// and the tree baseline never take that step.
bool tc_k_floor_broken(const OpDesc& op, const Sched& s, int level) {
  return level == 1 && tc_gemm(op) && s.tile(op, 2, 1) * op.dtype_bytes < 256 && op.ax[2].padded * op.dtype_bytes >= 256;
}

}  // namespace

bool b200_feasible(const OpDesc& op, const HwModel& hw, const Sched& s, int upto_level) {
  if (!hw.is_b200 || s.L < 1) return true;
  const DeviceLimits& d = hw.dev;
  if (upto_level >= 1 && tc_gemm(op)) {
    // tensor-core legality of the level-1 tile: UMMA M = 128 rows (cta_group::1), UMMA N within
    // [16, 256] (fp32 output: <= 128, the epilogue staging shares smem with the ring; TMEM holds
    // two BN-column accumulators), K ring of >= 2 k-blocks of 128 B (K-atom 32 B). Persistent
    // CTAs: no wave gate (the cost prices idle SMs).
    const GemmTcPlan p = gemm_tc_plan(op, s, exec_unit(op) == ExecUnit::TensorBf16, false);
    const bool short_k = op.ax[2].padded * op.dtype_bytes < 256;  // the whole K is one ring
    if (!(p.legal || (short_k && s.tile(op, 0, 1) == std::min<int64_t>(128, op.ax[0].padded) &&
                      s.tile(op, 1, 1) <= gemm_tc_bn_max(exec_unit(op) == ExecUnit::TensorBf16, false))))
      return false;
    if (2 * p.BN > d.tmem_cols) return false;
    // the tile grid fills the SMs when a 64-wide N tile can (the persistent grid is min(tiles, SMs))
    if (gemm_tc_tiles(op, p.BN) < std::min<int64_t>(d.sms, gemm_tc_tiles(op, 64))) return false;
  } else if (upto_level >= 1) {
    int64_t ctas = op.batch, max_ctas = op.batch;
    for (int a = 0; a < op.naxes; ++a) {
      if (op.ax[a].reduce) continue;
      ctas *= cdiv(op.ax[a].extent, s.tile(op, a, 1));
      max_ctas *= cdiv(op.ax[a].extent, 1);
    }
    max_ctas = std::max<int64_t>(1, max_ctas / 128);  // >= 128 outputs per CTA is the useful floor
    if (ctas < std::min<int64_t>(d.sms, max_ctas)) return false;
  }
  if (upto_level >= s.L) {
    int64_t threads = 1, acc = 1;
    for (int a = 0; a < op.naxes; ++a) {
      if (op.ax[a].reduce) continue;
      threads *= s.tile(op, a, 1) / s.tile(op, a, s.L);
      acc *= s.tile(op, a, s.L);
    }
    int64_t outs = 1;
    for (int a = 0; a < op.naxes; ++a)
      if (!op.ax[a].reduce) outs *= std::min(op.ax[a].extent, s.tile(op, a, 1));
    if (threads > d.max_threads_per_block || acc > 64) return false;
    if (s.L >= 2 && threads < std::min<int64_t>(32, outs)) return false;
  }
  return true;
}

bool candidates(const OpDesc& op, const HwModel& hw, const Sched& s, const EngineCfg& cfg, int iteration,
                std::vector<Candidate>& out) {
  out.clear();
  // gate flags ride in a parallel mask; only the Cache candidate is ever gated (engine.cpp:67-73)
  int gated_index = -1;
  if (!s.complete()) {
    const int level = s.edit_level();
    for (ActKind kind : {ActKind::Tile, ActKind::InvTile}) {
      if (kind == ActKind::InvTile && !cfg.enable_inv_tile) continue;
      for (int a = 0; a < op.naxes; ++a) {
        for (int64_t f = 2; f <= cfg.max_tile_factor; f *= 2) {
          const Action act{kind, a, f};
          if (!s.legal(op, act)) continue;
          Sched post = s;
          post.apply_unchecked(op, act);
          out.push_back({act, benefit_tiling(op, s, post, level), 0.0});
        }
      }
    }
  }
  static thread_local std::vector<int64_t> vopts;
  vopts = sorted_unique(cfg.vthread_options);
  for (int a = 0; a < op.naxes; ++a) {
    for (int64_t v : vopts) {
      const Action act{ActKind::SetVThread, a, v};
      if (!s.legal(op, act)) continue;
      out.push_back({act, benefit_vthread(op, hw, s, a, v), 0.0});
    }
  }
  if (!s.complete()) {
    Sched post = s;
    post.cur += 1;
    const double b = benefit_caching(op, hw, s, s.cur, post.cur) * anneal_cache_multiplier(iteration);
    bool gate = !capacity_ok(op, hw, post, post.cur);
    if (!gate && cfg.mode == Mode::B200) gate = !b200_feasible(op, hw, post, post.cur);
    out.push_back({Action{ActKind::Cache, -1, 0}, b, 0.0});
    if (gate) gated_index = static_cast<int>(out.size()) - 1;
  }

  // divide by the max first so huge ratios cannot overflow the sum (engine.cpp:75-87)
  double bmax = 0.0;
  for (size_t i = 0; i < out.size(); ++i)
    if (static_cast<int>(i) != gated_index) bmax = std::max(bmax, out[i].benefit);
  if (bmax <= 0.0) return false;
  double sum = 0.0;
  for (size_t i = 0; i < out.size(); ++i)
    if (static_cast<int>(i) != gated_index) sum += out[i].benefit / bmax;
  for (size_t i = 0; i < out.size(); ++i)
    if (static_cast<int>(i) != gated_index) out[i].probability = (out[i].benefit / bmax) / sum;
  return true;
}

int roulette(const std::vector<Candidate>& c, std::mt19937_64& rng) {
  if (c.empty()) throw Error(Code::EmptyCandidates, "roulette over empty set");
  const double u = uniform_unit(rng);
  double cum = 0.0;
  int last = -1;
  for (size_t i = 0; i < c.size(); ++i) {
    if (c[i].probability <= 0.0) continue;
    last = static_cast<int>(i);
    cum += c[i].probability;
    if (u < cum) return last;
  }
  if (last < 0) throw Error(Code::EmptyCandidates, "all candidates gated");
  return last;  // u landed in the rounding tail
}

std::vector<Result> construct(const OpDesc& op, const HwModel& hw, const EngineCfg& cfg, const Observer& obs) {
  cfg.validate();
  std::mt19937_64 rng(cfg.seed);
  Sched s = Sched::initial(op, hw.schedulable_levels());
  std::vector<Action> trace;
  std::vector<Result> snaps;
  std::vector<Candidate> cands;
  size_t recorded_len = SIZE_MAX;
  double t = cfg.t0;
  int iter = 0;
  while (t > cfg.threshold) {
    if (!candidates(op, hw, s, cfg, iter, cands)) break;  // terminal state: finalize early
    if (obs) obs(s, cands, t, iter);
    const Action pick = cands[static_cast<size_t>(roulette(cands, rng))].action;
    s.apply_unchecked(op, pick);
    trace.push_back(pick);
    if (uniform_unit(rng) < record_probability(t)) {
      snaps.push_back({s, {}, trace, cfg.seed, iter + 1});
      recorded_len = trace.size();
    }
    t /= 2.0;
    ++iter;
  }
  if (recorded_len != trace.size()) snaps.push_back({s, {}, trace, cfg.seed, iter});
  return snaps;
}

// Tile(axis, 2) at the editing level whose child moves the least level traffic; ties keep the
// first axis (strict <), tree_baseline.cpp:13-27.
bool greedy_fit_step(const OpDesc& op, const Sched& s, Action& out, bool tc_floor) {
  if (s.complete()) return false;
  bool found = false;
  int64_t best = 0;
  const int level = s.edit_level();
  for (int a = 0; a < op.naxes; ++a) {
    const Action act{ActKind::Tile, a, 2};
    if (!s.legal(op, act)) continue;
    Sched child = s;
    child.apply_unchecked(op, act);
    if (tc_floor && tc_k_floor_broken(op, child, level)) continue;
    const int64_t q = traffic(op, child, level);
    if (!found || q < best) {
      out = act;
      best = q;
      found = true;
    }
  }
  return found;
}

bool complete(const OpDesc& op, const HwModel& hw, Sched& s, std::vector<Action>& trace, Mode mode) {
  const bool dev = mode == Mode::B200 && hw.is_b200;
  while (!s.complete()) {
    const int target = s.edit_level();
    if (dev && target == 1 && tc_gemm(op)) {
      // shape the level-1 tile into the UMMA range first (M tile 128, N tile <= the epilogue
      // limit): legal Tile actions recorded in the trace, so the schedule replays
      const int64_t bn_max = gemm_tc_bn_max(exec_unit(op) == ExecUnit::TensorBf16, false);
      auto tile_down = [&](int a) {
        const Action act{ActKind::Tile, a, 2};
        if (!s.legal(op, act)) return false;
        s.apply_unchecked(op, act);
        trace.push_back(act);
        return true;
      };
      while (s.tile(op, 0, 1) > 128 && tile_down(0)) {
      }
      while (s.tile(op, 1, 1) > bn_max && tile_down(1)) {
      }
      // narrower N tiles while the grid leaves SMs idle (down to UMMA N = 64)
      const int64_t want = std::min<int64_t>(hw.dev.sms, gemm_tc_tiles(op, 64));
      while (s.tile(op, 1, 1) > 64 && gemm_tc_tiles(op, s.tile(op, 1, 1)) < want && tile_down(1)) {
      }
    }
    while (!capacity_ok(op, hw, s, target) || (dev && !b200_feasible(op, hw, s, target))) {
      Action step;
      if (!greedy_fit_step(op, s, step, dev)) return false;
      s.apply_unchecked(op, step);
      trace.push_back(step);
    }
    s.cur += 1;
    trace.push_back(Action{ActKind::Cache, -1, 0});
  }
  return true;
}

Cost cost_of(const OpDesc& op, const HwModel& hw, const Sched& s, Mode mode) {
  return (mode == Mode::B200 && hw.is_b200) ? estimate_b200(op, hw, s) : estimate(op, hw, s);
}

namespace {

bool better(const Result& a, const Result& b) {
  if (a.cost.est_seconds != b.cost.est_seconds) return a.cost.est_seconds < b.cost.est_seconds;
  if (a.trace.size() != b.trace.size()) return a.trace.size() < b.trace.size();
  return std::lexicographical_compare(a.trace.begin(), a.trace.end(), b.trace.begin(), b.trace.end());
}

std::vector<Result> restart_pool(const OpDesc& op, const HwModel& hw, const EngineCfg& cfg, int r,
                                 const Observer& obs) {
  EngineCfg run = cfg;
  run.seed = derive_seed(cfg.seed, r);
  std::vector<Result> pool;
  for (Result& res : construct(op, hw, run, obs)) {
    if (cfg.mode == Mode::B200) {
      // device gates first; a snapshot they cannot complete keeps the reference completion
      Sched s = res.state;
      std::vector<Action> tr = res.trace;
      if (complete(op, hw, s, tr, Mode::B200)) {
        res.state = s;
        res.trace = std::move(tr);
      } else if (!complete(op, hw, res.state, res.trace, Mode::ReferenceCompat)) {
        continue;
      }
    } else if (!complete(op, hw, res.state, res.trace, cfg.mode)) {
      continue;  // dropped silently (engine.cpp:173)
    }
    res.cost = cost_of(op, hw, res.state, cfg.mode);
    pool.push_back(std::move(res));
  }
  return pool;
}

}  // namespace

std::vector<Result> optimize(const OpDesc& op, const HwModel& hw, const EngineCfg& cfg, const Observer& obs) {
  cfg.validate();
  std::vector<std::vector<Result>> per(static_cast<size_t>(cfg.restarts));
  int workers = cfg.threads > 0 ? cfg.threads : static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  workers = std::min(workers, cfg.restarts);
  if (obs) workers = 1;  // observer calls stay on the caller's thread, in restart order
  if (workers <= 1) {
    for (int r = 0; r < cfg.restarts; ++r) per[static_cast<size_t>(r)] = restart_pool(op, hw, cfg, r, obs);
  } else {
    std::vector<std::thread> pool;
    std::vector<std::exception_ptr> errs(static_cast<size_t>(workers));
    for (int w = 0; w < workers; ++w) {
      pool.emplace_back([&, w] {
        try {
          for (int r = w; r < cfg.restarts; r += workers)
            per[static_cast<size_t>(r)] = restart_pool(op, hw, cfg, r, nullptr);
        } catch (...) {
          errs[static_cast<size_t>(w)] = std::current_exception();
        }
      });
    }
    for (auto& th : pool) th.join();
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
  }
  // merge in restart order: the pool is then element-for-element the sequential reference pool,
  // so std::sort (same comparator, same input order) yields the same permutation
  std::vector<Result> merged;
  for (auto& p : per)
    for (auto& r : p) merged.push_back(std::move(r));
  std::sort(merged.begin(), merged.end(), better);
  merged.erase(std::unique(merged.begin(), merged.end(),
                           [&](const Result& a, const Result& b) {
                             return a.trace == b.trace && a.state.same(b.state, op.naxes);
                           }),
               merged.end());
  if (merged.size() > static_cast<size_t>(cfg.top_k)) merged.resize(static_cast<size_t>(cfg.top_k));
  return merged;
}

namespace {

struct Beam {
  Sched state;
  std::vector<Action> trace;
  int64_t q = 0;
};

void prune(const OpDesc& op, std::vector<Beam>& items, int width) {
  std::sort(items.begin(), items.end(), [](const Beam& a, const Beam& b) {
    if (a.q != b.q) return a.q < b.q;
    return std::lexicographical_compare(a.trace.begin(), a.trace.end(), b.trace.begin(), b.trace.end());
  });
  items.erase(std::unique(items.begin(), items.end(),
                          [&](const Beam& a, const Beam& b) { return a.state.same(b.state, op.naxes); }),
              items.end());
  if (items.size() > static_cast<size_t>(width)) items.resize(static_cast<size_t>(width));
}

}  // namespace

std::vector<Result> construct_tree(const OpDesc& op, const HwModel& hw, int beam_width, Mode mode) {
  if (beam_width < 1) throw Error(Code::ConfigError, "beam_width must be >= 1");
  const bool dev = mode == Mode::B200 && hw.is_b200;
  std::vector<Beam> frontier{{Sched::initial(op, hw.schedulable_levels()), {}, 0}};
  for (int level = 1; level <= hw.schedulable_levels(); ++level) {
    std::vector<Beam> fitting;
    std::vector<Beam> work = std::move(frontier);
    for (Beam& b : work) b.q = traffic(op, b.state, level);
    prune(op, work, beam_width);
    while (!work.empty()) {
      std::vector<Beam> grown;
      for (Beam& b : work) {
        if (capacity_ok(op, hw, b.state, level) && (!dev || b200_feasible(op, hw, b.state, level))) {
          fitting.push_back(std::move(b));
          continue;
        }
        for (int a = 0; a < op.naxes; ++a) {
          const Action act{ActKind::Tile, a, 2};
          if (!b.state.legal(op, act)) continue;
          Beam child{b.state, b.trace, 0};
          child.state.apply_unchecked(op, act);
          if (dev && tc_k_floor_broken(op, child.state, level)) continue;
          child.trace.push_back(act);
          child.q = traffic(op, child.state, level);
          grown.push_back(std::move(child));
        }
      }
      prune(op, grown, beam_width);
      work = std::move(grown);
    }
    prune(op, fitting, beam_width);
    frontier.clear();
    for (Beam& b : fitting) {
      b.state.cur += 1;
      b.trace.push_back(Action{ActKind::Cache, -1, 0});
      frontier.push_back(std::move(b));
    }
  }
  std::vector<Result> out;
  for (Beam& b : frontier) {
    Result r{b.state, {}, std::move(b.trace), 0, 0};
    r.iterations = static_cast<int>(r.trace.size());
    r.cost = cost_of(op, hw, r.state, mode);
    out.push_back(std::move(r));
  }
  std::sort(out.begin(), out.end(), better);
  return out;
}

}  // namespace gb
