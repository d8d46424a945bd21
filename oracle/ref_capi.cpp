// TEST INFRASTRUCTURE ONLY. A C-ABI shim over the reference's own construct library
// (compiled unmodified from /root/reference/proj/src by oracle/Makefile into oracle/_ref/).
// It lets the differential tests, the golden-vector generator (tools/make_golden.py) and
// bench.py's `--impl reference` arm call the reference's public C++ API:
//   TensorOpSpec::parse_text        op_spec.hpp:51
//   HardwareSpec::load_text         hardware.hpp:31
//   optimize / construct            engine.hpp:83-99
//   enumerate_candidates            engine.hpp:54-57
//   memory_traffic / traffic_oracle / estimate_cost   cost_model.hpp:32-71
//   construct_tree / greedy_fit_step                  tree_baseline.hpp:21-26
//   enumerate_space / check_* / stationary / value    markov.hpp:40-67
// Every entry point takes JSON text and returns a malloc'd JSON string (free with ref_free).
// Nothing in the product (paper_2502_11407_b200/) links or loads this file.
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <string>

#include "gensor/cost_model.hpp"
#include "gensor/engine.hpp"
#include "gensor/error.hpp"
#include "gensor/etir.hpp"
#include "gensor/hardware.hpp"
#include "gensor/markov.hpp"
#include "gensor/op_spec.hpp"
#include "gensor/tree_baseline.hpp"

using namespace gensor;

namespace {

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

Json err_json(const std::exception& e) {
  Json j;
  j["error"] = e.what();
  const auto* ge = dynamic_cast<const Error*>(&e);
  j["code"] = ge ? static_cast<int>(ge->code()) : -1;
  return j;
}

EngineConfig cfg_from(const Json& c) {
  EngineConfig cfg;
  if (c.contains("t0")) cfg.t0 = c["t0"].get<double>();
  if (c.contains("threshold")) cfg.threshold = c["threshold"].get<double>();
  if (c.contains("restarts")) cfg.restarts = c["restarts"].get<int>();
  if (c.contains("seed")) cfg.seed = c["seed"].get<uint64_t>();
  if (c.contains("top_k")) cfg.top_k = c["top_k"].get<int>();
  if (c.contains("vthread_options")) cfg.vthread_options = c["vthread_options"].get<std::vector<int64_t>>();
  if (c.contains("max_tile_factor")) cfg.max_tile_factor = c["max_tile_factor"].get<int64_t>();
  return cfg;
}

Json action_json(const Action& a) { return Json::array({static_cast<int>(a.kind), a.axis, a.factor}); }

Action action_from(const Json& j) {
  return Action{static_cast<ActionKind>(j.at(0).get<int>()), j.at(1).get<int>(), j.at(2).get<int64_t>()};
}

Json state_json(const ETIRState& s) {
  Json j;
  j["level"] = s.cur_mem_level();
  Json tiles = Json::array();
  for (int a = 0; a < s.op().num_axes(); ++a) {
    Json per = Json::array();
    for (int l = 1; l <= s.num_levels(); ++l) per.push_back(s.tile_at(a, l));
    tiles.push_back(per);
  }
  j["tiles"] = tiles;
  Json vt = Json::array();
  for (int a = 0; a < s.op().num_axes(); ++a) vt.push_back(s.vthread(a));
  j["vthreads"] = vt;
  j["repr"] = s.repr();
  return j;
}

Json cost_json(const CostEstimate& c) {
  Json j;
  j["est_seconds"] = c.est_seconds;
  j["compute_seconds"] = c.compute_seconds;
  Json mem = Json::array();
  for (const auto& [name, sec] : c.memory_seconds) mem.push_back(Json::array({name, sec}));
  j["memory_seconds"] = mem;
  j["bottleneck"] = c.bottleneck;
  return j;
}

Json result_json(const ScheduleResult& r) {
  Json j;
  j["state"] = state_json(r.state);
  Json tr = Json::array();
  for (const Action& a : r.trace) tr.push_back(action_json(a));
  j["trace"] = tr;
  j["cost"] = cost_json(r.cost);
  j["seed"] = r.seed;
  j["iterations"] = r.iterations;
  return j;
}

ETIRState replay(const TensorOpSpec& op, const HardwareSpec& hw, const Json& trace) {
  ETIRState s = ETIRState::initial(op, hw);
  for (const auto& a : trace) s = s.apply(action_from(a));
  return s;
}

}  // namespace

extern "C" {

void ref_free(char* p) { std::free(p); }

// Multi-restart construction (engine.cpp:165-192) plus its wall time.
char* ref_optimize(const char* op_text, const char* hw_text, const char* cfg_text) {
  try {
    TensorOpSpec op = TensorOpSpec::parse_text(op_text);
    HardwareSpec hw = HardwareSpec::load_text(hw_text);
    EngineConfig cfg = cfg_from(Json::parse(cfg_text));
    auto t0 = std::chrono::steady_clock::now();
    auto results = optimize(op, hw, cfg);
    auto t1 = std::chrono::steady_clock::now();
    Json out;
    out["wall_s"] = std::chrono::duration<double>(t1 - t0).count();
    out["results"] = Json::array();
    for (const auto& r : results) out["results"].push_back(result_json(r));
    return dup(out.dump());
  } catch (const std::exception& e) {
    return dup(err_json(e).dump());
  }
}

// One annealed walk (engine.cpp:105-140) with every visited state's candidate list.
char* ref_construct(const char* op_text, const char* hw_text, const char* cfg_text) {
  try {
    TensorOpSpec op = TensorOpSpec::parse_text(op_text);
    HardwareSpec hw = HardwareSpec::load_text(hw_text);
    EngineConfig cfg = cfg_from(Json::parse(cfg_text));
    Json visits = Json::array();
    StateObserver obs = [&](const ETIRState& s, std::span<const ActionCandidate> cands,
                            const AnnealPoint& at) {
      Json v;
      v["repr"] = s.repr();
      v["temperature"] = at.temperature;
      v["iteration"] = at.iteration;
      Json cj = Json::array();
      for (const auto& c : cands)
        cj.push_back(Json::array({action_json(c.action), c.benefit, c.probability}));
      v["candidates"] = cj;
      visits.push_back(v);
    };
    auto results = construct(op, hw, cfg, obs);
    Json out;
    out["visits"] = visits;
    out["results"] = Json::array();
    for (const auto& r : results) out["results"].push_back(result_json(r));
    return dup(out.dump());
  } catch (const std::exception& e) {
    return dup(err_json(e).dump());
  }
}

// Replays a trace and reports the cost-model quantities of the resulting state.
char* ref_state_eval(const char* op_text, const char* hw_text, const char* trace_text) {
  try {
    TensorOpSpec op = TensorOpSpec::parse_text(op_text);
    HardwareSpec hw = HardwareSpec::load_text(hw_text);
    ETIRState s = replay(op, hw, Json::parse(trace_text));
    Json out;
    out["state"] = state_json(s);
    Json levels = Json::array();
    for (int l = 1; l <= s.num_levels(); ++l) {
      Json lj;
      lj["traffic"] = memory_traffic(s, hw, l);
      lj["footprint"] = tile_footprint_elems(s, l);
      lj["footprint_bytes"] = tile_footprint_bytes(s, l);
      lj["capacity_ok"] = capacity_check(s, hw, l);
      try {
        lj["traffic_oracle"] = traffic_oracle(s, l);
      } catch (const Error&) {
        lj["traffic_oracle"] = nullptr;
      }
      levels.push_back(lj);
    }
    out["levels"] = levels;
    out["utilization"] = utilization(s, hw);
    if (s.complete()) out["cost"] = cost_json(estimate_cost(s, hw));
    Json vb = Json::array();
    for (int a = 0; a < op.num_axes(); ++a) {
      if (op.axis(a).kind != AxisKind::Spatial) continue;
      for (int64_t v : {1, 2, 4, 8}) vb.push_back(Json::array({a, v, benefit_vthread(s, hw, a, v)}));
    }
    out["vthread_benefits"] = vb;
    auto step = greedy_fit_step(s, hw);
    out["greedy_step"] = step ? action_json(*step) : Json(nullptr);
    Json legal = Json::array();
    for (int kind = 0; kind < 4; ++kind)
      for (int a = -1; a < op.num_axes(); ++a)
        for (int64_t f : {0, 1, 2, 4, 8}) {
          Action act{static_cast<ActionKind>(kind), a, f};
          if (s.is_legal(act)) legal.push_back(action_json(act));
        }
    out["legal"] = legal;
    return dup(out.dump());
  } catch (const std::exception& e) {
    return dup(err_json(e).dump());
  }
}

// Candidate list at a replayed state for an explicit anneal point (engine.cpp:32-88).
char* ref_candidates(const char* op_text, const char* hw_text, const char* trace_text,
                     const char* cfg_text, int iteration, double temperature) {
  try {
    TensorOpSpec op = TensorOpSpec::parse_text(op_text);
    HardwareSpec hw = HardwareSpec::load_text(hw_text);
    ETIRState s = replay(op, hw, Json::parse(trace_text));
    EngineConfig cfg = cfg_from(Json::parse(cfg_text));
    ActionSpace space{cfg.vthread_options, cfg.max_tile_factor, true};
    auto cands = enumerate_candidates(s, hw, space, AnnealPoint{temperature, iteration});
    Json out = Json::array();
    for (const auto& c : cands) out.push_back(Json::array({action_json(c.action), c.benefit, c.probability}));
    Json wrap;
    wrap["candidates"] = out;
    return dup(wrap.dump());
  } catch (const std::exception& e) {
    return dup(err_json(e).dump());
  }
}

// Roller-style beam baseline (tree_baseline.cpp:53-108).
char* ref_tree(const char* op_text, const char* hw_text, int beam) {
  try {
    TensorOpSpec op = TensorOpSpec::parse_text(op_text);
    HardwareSpec hw = HardwareSpec::load_text(hw_text);
    TreeConfig tc;
    tc.beam_width = beam;
    auto results = construct_tree(op, hw, tc);
    Json out;
    out["results"] = Json::array();
    for (const auto& r : results) out["results"].push_back(result_json(r));
    return dup(out.dump());
  } catch (const std::exception& e) {
    return dup(err_json(e).dump());
  }
}

// Parsed op: axes (name, extent, padded, reduce), tensors, padded flops, round-trip JSON.
char* ref_op_info(const char* op_text) {
  try {
    TensorOpSpec op = TensorOpSpec::parse_text(op_text);
    Json out;
    Json axes = Json::array();
    for (const Axis& a : op.axes())
      axes.push_back(Json::array({a.name, a.extent, a.padded, a.kind == AxisKind::Reduce}));
    out["axes"] = axes;
    Json tensors = Json::array();
    for (int t = 0; t < op.num_tensors(); ++t) {
      const TensorInfo& ti = op.tensors()[static_cast<size_t>(t)];
      Json dims = Json::array();
      for (const TensorDim& d : ti.dims) dims.push_back(Json::array({d.axis, d.window_axis}));
      Json tj;
      tj["name"] = ti.name;
      tj["is_output"] = ti.is_output;
      tj["dims"] = dims;
      tj["true_dims"] = op.tensor_dims(t, false);
      tensors.push_back(tj);
    }
    out["tensors"] = tensors;
    out["flops_padded"] = op.flops_padded();
    out["stride"] = op.stride();
    out["dtype_bytes"] = op.dtype_bytes();
    out["label"] = op.label();
    out["json"] = op.to_json();
    return dup(out.dump());
  } catch (const std::exception& e) {
    return dup(err_json(e).dump());
  }
}

// The reference's chain model and analyses (markov.cpp:40-364), per state in its own discovery
// order: repr, level, complete, absorbing, terminal, rows; per-level irreducibility; aperiodicity;
// value iteration; the stationary vector of every level listed in caps["stationary_levels"].
char* ref_analyze(const char* op_text, const char* hw_text, const char* caps_text) {
  try {
    TensorOpSpec op = TensorOpSpec::parse_text(op_text);
    HardwareSpec hw = HardwareSpec::load_text(hw_text);
    Json c = Json::parse(caps_text);
    ChainCaps caps;
    if (c.contains("max_states")) caps.max_states = c["max_states"].get<int>();
    if (c.contains("fixed_iteration")) caps.fixed_iteration = c["fixed_iteration"].get<int>();
    if (c.contains("enable_inv_tile")) caps.enable_inv_tile = c["enable_inv_tile"].get<bool>();
    if (c.contains("vthread_options")) caps.vthread_options = c["vthread_options"].get<std::vector<int64_t>>();
    if (c.contains("max_tile_factor")) caps.max_tile_factor = c["max_tile_factor"].get<int64_t>();
    ChainModel m = enumerate_space(op, hw, caps);
    Json out;
    Json states = Json::array(), rows = Json::array();
    for (int i = 0; i < m.num_states(); ++i) {
      states.push_back(m.states[static_cast<size_t>(i)].repr());
      Json row = Json::array();
      for (const ChainEdge& e : m.rows[static_cast<size_t>(i)])
        row.push_back(Json::array({e.to, e.prob, action_json(e.action), e.artificial ? 1 : 0}));
      rows.push_back(row);
    }
    out["states"] = states;
    out["rows"] = rows;
    out["level"] = m.level_of;
    out["complete"] = m.complete;
    out["absorbing"] = m.absorbing;
    out["terminal"] = m.terminal_value;
    out["irreducible"] = check_irreducible_per_level(m);
    out["aperiodic"] = check_aperiodic(m);
    ValueTable vt = value_iteration(m);
    out["value"] = vt.value;
    out["iterations"] = vt.iterations;
    Json pol = Json::array();
    for (const auto& p : vt.policy) pol.push_back(p ? action_json(*p) : Json());
    out["policy"] = pol;
    Json st = Json::object();
    if (c.contains("stationary_levels"))
      for (int l : c["stationary_levels"].get<std::vector<int>>()) st[std::to_string(l)] = stationary_distribution(m, l);
    out["stationary"] = st;
    return dup(out.dump());
  } catch (const std::exception& e) {
    return dup(err_json(e).dump());
  }
}

// Scalar formulas: Eq. 2, Eq. 3, the anneal multiplier and the record sigmoid.
double ref_caching_benefit(double ll, double bl, double lh, double bh, double s) {
  return caching_benefit(ll, bl, lh, bh, s);
}
double ref_vthread_conflict_ratio(int64_t x, int64_t w, int64_t v) { return vthread_conflict_ratio(x, w, v); }
double ref_anneal_cache_multiplier(int it) { return anneal_cache_multiplier(it); }
double ref_record_probability(double t) { return record_probability(t); }
uint64_t ref_derive_seed(uint64_t seed, int r) { return derive_seed(seed, r); }

}  // extern "C"
