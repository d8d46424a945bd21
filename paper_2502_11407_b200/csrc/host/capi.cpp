#include <algorithm>
// C-ABI of the gensor-b200 host library (include/gensor_b200.h). Every entry point catches
// gb::Error / std::exception and turns it into a status code + thread-local message.
#include "gensor_b200.h"

#include <cstring>
#include <memory>
#include <new>
#include <sstream>
#include <string>
#include <vector>

#include "cost.hpp"
#include "device.hpp"
#include "emit.hpp"
#include "markov.hpp"
#include "engine.hpp"
#include "error.hpp"
#include "hw.hpp"
#include "json.hpp"
#include "op.hpp"
#include "sched.hpp"

struct gensor_op {
  gb::OpDesc op;
};
struct gensor_hw {
  gb::HwModel hw;
};
struct gensor_schedule {
  const gb::OpDesc* op = nullptr;
  gb::HwModel hw;  // copied: names for cost reports; small
  gb::Mode mode = gb::Mode::ReferenceCompat;
  std::vector<gb::Result> results;
};
struct gensor_kernel {
  gb::dev::Kernel* k = nullptr;
};

namespace gb {

const char* code_name(Code c) {
  switch (c) {
    case Code::UnknownKind: return "UnknownKind";
    case Code::MissingParam: return "MissingParam";
    case Code::NonPositiveExtent: return "NonPositiveExtent";
    case Code::AxisNotFound: return "AxisNotFound";
    case Code::IllegalAction: return "IllegalAction";
    case Code::LevelOutOfRange: return "LevelOutOfRange";
    case Code::MonotonicityViolation: return "MonotonicityViolation";
    case Code::MissingLevel: return "MissingLevel";
    case Code::IncompleteState: return "IncompleteState";
    case Code::TooLargeToEnumerate: return "TooLargeToEnumerate";
    case Code::NoLegalAction: return "NoLegalAction";
    case Code::EmptyCandidates: return "EmptyCandidates";
    case Code::SpaceTooLarge: return "SpaceTooLarge";
    case Code::NotErgodic: return "NotErgodic";
    case Code::NoConvergence: return "NoConvergence";
    case Code::ShapeMismatch: return "ShapeMismatch";
    case Code::ReplayMismatch: return "ReplayMismatch";
    case Code::ConfigError: return "ConfigError";
    case Code::Cuda: return "Cuda";
    case Code::Unsupported: return "Unsupported";
  }
  return "Error";
}

}  // namespace gb

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

template <class F>
int guarded(F&& f) {
  try {
    g_last_error.clear();
    return f();
  } catch (const gb::Error& e) {
    return fail(static_cast<int>(e.code()) + 1, e.what());
  } catch (const std::bad_alloc&) {
    return fail(GENSOR_EINVALID, "out of memory");
  } catch (const std::exception& e) {
    return fail(GENSOR_ECONFIG, std::string("ConfigError: ") + e.what());
  }
}

// A kernel is instantiated from a schedule of the SAME operator: the schedule's tiles index that
// op's axes and padded extents (an ETIRState belongs to one TensorOpSpec, etir.hpp:75).
void check_schedule_op(const gb::OpDesc& op, const gensor_schedule& s) {
  if (s.op == &op) return;
  if (!s.op || s.op->to_json() != op.to_json())
    throw gb::Error(gb::Code::ShapeMismatch, "schedule was constructed for " + (s.op ? s.op->label() : std::string("?")) +
                                                 ", not for " + op.label());
}

int emit(const std::string& s, char* buf, size_t cap, size_t* need) {
  if (need) *need = s.size() + 1;
  if (!buf || cap < s.size() + 1) return fail(GENSOR_ETRUNCATED, "output buffer too small");
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return GENSOR_OK;
}

gb::EngineCfg cfg_from(const gensor_engine_cfg* c) {
  gb::EngineCfg e;
  if (!c) return e;
  e.t0 = c->t0;
  e.threshold = c->threshold;
  e.restarts = c->restarts;
  e.top_k = c->top_k;
  e.seed = c->seed;
  e.vthread_options.assign(c->vthread_options, c->vthread_options + std::max(0, std::min(8, c->n_vthread_options)));
  e.max_tile_factor = c->max_tile_factor;
  e.mode = c->mode == GENSOR_MODE_B200 ? gb::Mode::B200 : gb::Mode::ReferenceCompat;
  e.threads = c->threads;
  return e;
}

std::vector<gb::Action> trace_from(const std::string& text) {
  gb::json::Value v = gb::json::parse(text);
  if (!v.is_array()) throw gb::Error(gb::Code::ConfigError, "trace must be a JSON array");
  std::vector<gb::Action> out;
  for (const auto& a : v.arr) {
    if (!a.is_array() || a.arr.size() != 3) throw gb::Error(gb::Code::ConfigError, "action must be [kind,axis,factor]");
    int kind = static_cast<int>(a.arr[0].as_int());
    if (kind < 0 || kind > 3) throw gb::Error(gb::Code::ConfigError, "action kind out of range");
    out.push_back({static_cast<gb::ActKind>(kind), static_cast<int>(a.arr[1].as_int()), a.arr[2].as_int()});
  }
  return out;
}

gb::Sched replay(const gb::OpDesc& op, const gb::HwModel& hw, const std::vector<gb::Action>& tr) {
  gb::Sched s = gb::Sched::initial(op, hw.schedulable_levels());
  for (const auto& a : tr) s = s.apply(op, a);
  return s;
}

std::string trace_json(const std::vector<gb::Action>& tr) {
  std::ostringstream os;
  os << "[";
  for (size_t i = 0; i < tr.size(); ++i)
    os << (i ? "," : "") << "[" << static_cast<int>(tr[i].kind) << "," << tr[i].axis << "," << tr[i].factor << "]";
  os << "]";
  return os.str();
}

std::string result_json(const gensor_schedule* s, const gb::Result& r) {
  std::ostringstream os;
  os << "{\"state\":" << r.state.to_json(*s->op) << ",\"trace\":" << trace_json(r.trace);
  if (r.state.complete())
    os << ",\"cost\":" << gb::cost_json(r.cost, s->hw);
  else
    os << ",\"cost\":null";
  os << ",\"seed\":" << r.seed << ",\"iterations\":" << r.iterations << "}";
  return os.str();
}

int make_schedule(const gensor_op* op, const gensor_hw* hw, gb::Mode mode, std::vector<gb::Result>&& res,
                  gensor_schedule** out, int* n_out) {
  auto* s = new gensor_schedule;
  s->op = &op->op;
  s->hw = hw->hw;
  s->mode = mode;
  s->results = std::move(res);
  if (n_out) *n_out = static_cast<int>(s->results.size());
  *out = s;
  return GENSOR_OK;
}

}  // namespace

extern "C" {

const char* gensor_last_error(void) { return g_last_error.c_str(); }
const char* gensor_version(void) { return "gensor-b200 0.1 (sm_100a)"; }

void gensor_engine_cfg_init(gensor_engine_cfg* c) {
  if (!c) return;
  std::memset(c, 0, sizeof *c);
  c->t0 = 1048576.0;
  c->threshold = 1.0;
  c->restarts = 8;
  c->top_k = 10;
  c->seed = 0;
  const int64_t v[4] = {1, 2, 4, 8};
  for (int i = 0; i < 4; ++i) c->vthread_options[i] = v[i];
  c->n_vthread_options = 4;
  c->mode = GENSOR_MODE_REFERENCE_COMPAT;
  c->max_tile_factor = 2;
  c->threads = 0;
}

int gensor_op_parse(const char* json, gensor_op** out) {
  if (!json || !out) return fail(GENSOR_EINVALID, "null argument");
  return guarded([&]() -> int {
    auto* o = new gensor_op{gb::OpDesc::parse_text(json)};
    *out = o;
    return GENSOR_OK;
  });
}

void gensor_op_free(gensor_op* op) { delete op; }

int gensor_op_info(const gensor_op* o, char* buf, size_t cap, size_t* need) {
  if (!o) return fail(GENSOR_EINVALID, "null op");
  return guarded([&]() -> int {
    const gb::OpDesc& op = o->op;
    std::ostringstream os;
    os << "{\"kind\":\"" << gb::kind_name(op.kind) << "\",\"label\":" << gb::json::quote(op.label())
       << ",\"dtype_bytes\":" << op.dtype_bytes << ",\"stride\":" << op.stride << ",\"batch\":" << op.batch
       << ",\"axes\":[";
    for (int a = 0; a < op.naxes; ++a)
      os << (a ? "," : "") << "[\"" << op.ax[a].name << "\"," << op.ax[a].extent << "," << op.ax[a].padded << ","
         << (op.ax[a].reduce ? "true" : "false") << "]";
    os << "],\"tensors\":[";
    for (int t = 0; t < op.ntensors; ++t) {
      int64_t dims[gb::kMaxDims], coef[gb::kMaxAxes];
      int nd = op.tensor_dims(t, false, dims);
      op.affine_coefs(t, coef);
      os << (t ? "," : "") << "{\"name\":\"" << op.t[t].name << "\",\"is_output\":" << (op.t[t].output ? "true" : "false")
         << ",\"dims\":[";
      for (int d = 0; d < op.t[t].ndims; ++d)
        os << (d ? "," : "") << "[" << int(op.t[t].dim[d].axis) << "," << int(op.t[t].dim[d].win) << "]";
      os << "],\"true_dims\":[";
      for (int d = 0; d < nd; ++d) os << (d ? "," : "") << dims[d];
      os << "],\"coef\":[";
      for (int a = 0; a < op.naxes; ++a) os << (a ? "," : "") << coef[a];
      os << "]}";
    }
    os << "],\"flops_padded\":" << op.flops_padded() << ",\"flops\":" << gb::json::num(op.flops_true())
       << ",\"bytes\":" << gb::json::num(op.bytes_true()) << ",\"json\":" << op.to_json() << "}";
    return emit(os.str(), buf, cap, need);
  });
}

int gensor_hw_load(const char* json, gensor_hw** out) {
  if (!json || !out) return fail(GENSOR_EINVALID, "null argument");
  return guarded([&]() -> int {
    *out = new gensor_hw{gb::HwModel::load_text(json)};
    return GENSOR_OK;
  });
}

int gensor_hw_b200(int device, const char* peaks, gensor_hw** out) {
  if (!out) return fail(GENSOR_EINVALID, "null argument");
  return guarded([&]() -> int {
    // device < 0: the nominal B200 limits (hw.hpp defaults) without a device query — construction
    // in B200 mode on a host without a GPU (CPU tests, offline schedule caches)
    gb::DeviceLimits lim = device < 0 ? gb::DeviceLimits{} : gb::dev::query(device);
    if (peaks && *peaks) {
      gb::json::Value p = gb::json::parse(peaks);
      if (const auto* v = p.find("hbm_gbs")) lim.hbm_bytes_per_s = v->as_double() * 1e9;
      if (const auto* v = p.find("bf16_tflops")) lim.bf16_tc_flops = v->as_double() * 1e12;
      if (const auto* v = p.find("tf32_tflops")) lim.tf32_tc_flops = v->as_double() * 1e12;
      if (const auto* v = p.find("fp32_simt_tflops")) lim.fp32_simt_flops = v->as_double() * 1e12;
    }
    *out = new gensor_hw{gb::HwModel::b200(lim)};
    return GENSOR_OK;
  });
}

void gensor_hw_free(gensor_hw* hw) { delete hw; }

int gensor_hw_json(const gensor_hw* hw, char* buf, size_t cap, size_t* need) {
  if (!hw) return fail(GENSOR_EINVALID, "null hw");
  return guarded([&]() -> int { return emit(hw->hw.to_json(), buf, cap, need); });
}

int gensor_optimize(const gensor_op* op, const gensor_hw* hw, const gensor_engine_cfg* cfg, gensor_schedule** out,
                    int* n_out) {
  if (!op || !hw || !out) return fail(GENSOR_EINVALID, "null argument");
  return guarded([&]() -> int {
    gb::EngineCfg c = cfg_from(cfg);
    return make_schedule(op, hw, c.mode, gb::optimize(op->op, hw->hw, c), out, n_out);
  });
}

int gensor_construct(const gensor_op* op, const gensor_hw* hw, const gensor_engine_cfg* cfg, gensor_schedule** out,
                     int* n_out) {
  if (!op || !hw || !out) return fail(GENSOR_EINVALID, "null argument");
  return guarded([&]() -> int {
    gb::EngineCfg c = cfg_from(cfg);
    return make_schedule(op, hw, c.mode, gb::construct(op->op, hw->hw, c), out, n_out);
  });
}

int gensor_construct_tree(const gensor_op* op, const gensor_hw* hw, int beam, int mode, gensor_schedule** out,
                          int* n_out) {
  if (!op || !hw || !out) return fail(GENSOR_EINVALID, "null argument");
  return guarded([&]() -> int {
    gb::Mode m = mode == GENSOR_MODE_B200 ? gb::Mode::B200 : gb::Mode::ReferenceCompat;
    return make_schedule(op, hw, m, gb::construct_tree(op->op, hw->hw, beam, m), out, n_out);
  });
}

int gensor_schedule_from_trace(const gensor_op* op, const gensor_hw* hw, const char* tr, int mode,
                               gensor_schedule** out) {
  if (!op || !hw || !tr || !out) return fail(GENSOR_EINVALID, "null argument");
  return guarded([&]() -> int {
    gb::Mode m = mode == GENSOR_MODE_B200 ? gb::Mode::B200 : gb::Mode::ReferenceCompat;
    gb::Result r;
    r.trace = trace_from(tr);
    r.state = replay(op->op, hw->hw, r.trace);
    r.iterations = static_cast<int>(r.trace.size());
    if (r.state.complete()) r.cost = gb::cost_of(op->op, hw->hw, r.state, m);
    std::vector<gb::Result> v;
    v.push_back(std::move(r));
    return make_schedule(op, hw, m, std::move(v), out, nullptr);
  });
}

int gensor_schedule_json(const gensor_schedule* s, int index, char* buf, size_t cap, size_t* need) {
  if (!s) return fail(GENSOR_EINVALID, "null schedule");
  return guarded([&]() -> int {
    if (index >= static_cast<int>(s->results.size()) || index < -1)
      return fail(GENSOR_EINVALID, "schedule index out of range");
    if (index >= 0) return emit(result_json(s, s->results[static_cast<size_t>(index)]), buf, cap, need);
    std::string all = "[";
    for (size_t i = 0; i < s->results.size(); ++i) all += (i ? "," : "") + result_json(s, s->results[i]);
    return emit(all + "]", buf, cap, need);
  });
}

int gensor_emit_source(const gensor_schedule* s, int index, char* buf, size_t cap, size_t* need) {
  if (!s) return fail(GENSOR_EINVALID, "null schedule");
  return guarded([&]() -> int {
    if (index < 0 || index >= static_cast<int>(s->results.size()))
      return fail(GENSOR_EINVALID, "schedule index out of range");
    const gb::Result& r = s->results[static_cast<size_t>(index)];
    if (!r.state.complete()) throw gb::Error(gb::Code::IncompleteState, "emit_source needs a complete state");
    return emit(gb::emit_source(*s->op, r.state, trace_json(r.trace)), buf, cap, need);
  });
}

int gensor_analyze(const gensor_op* op, const gensor_hw* hw, const char* caps_json, char* buf, size_t cap,
                   size_t* need) {
  if (!op || !hw) return fail(GENSOR_EINVALID, "null argument");
  return guarded([&]() -> int {
    gb::ChainCaps caps;
    bool detail = false;
    if (caps_json && *caps_json) {
      const gb::json::Value c = gb::json::parse(caps_json);
      if (!c.is_object()) throw gb::Error(gb::Code::ConfigError, "caps must be a JSON object");
      if (const auto* v = c.find("max_states")) caps.max_states = static_cast<int>(v->as_int());
      if (const auto* v = c.find("fixed_iteration")) caps.fixed_iteration = static_cast<int>(v->as_int());
      if (const auto* v = c.find("enable_inv_tile")) caps.enable_inv_tile = v->as_int() != 0;
      if (const auto* v = c.find("max_tile_factor")) caps.max_tile_factor = v->as_int();
      if (const auto* v = c.find("vthread_options")) {
        caps.vthread_options.clear();
        for (const auto& x : v->arr) caps.vthread_options.push_back(x.as_int());
      }
      if (const auto* v = c.find("mode")) caps.mode = v->as_string() == "b200" ? gb::Mode::B200 : gb::Mode::ReferenceCompat;
      if (const auto* v = c.find("detail")) detail = v->as_int() != 0;
    }
    if (caps.max_states < 1) throw gb::Error(gb::Code::ConfigError, "max_states must be >= 1");
    return emit(gb::analysis_json(op->op, hw->hw, caps, detail), buf, cap, need);
  });
}

int gensor_schedule_count(const gensor_schedule* s) { return s ? static_cast<int>(s->results.size()) : 0; }
void gensor_schedule_free(gensor_schedule* s) { delete s; }

int gensor_state_eval(const gensor_op* o, const gensor_hw* h, const char* tr, int mode, char* buf, size_t cap,
                      size_t* need) {
  if (!o || !h || !tr) return fail(GENSOR_EINVALID, "null argument");
  return guarded([&]() -> int {
    const gb::OpDesc& op = o->op;
    const gb::HwModel& hw = h->hw;
    gb::Mode m = mode == GENSOR_MODE_B200 ? gb::Mode::B200 : gb::Mode::ReferenceCompat;
    gb::Sched s = replay(op, hw, trace_from(tr));
    std::ostringstream os;
    os << "{\"state\":" << s.to_json(op) << ",\"levels\":[";
    for (int l = 1; l <= s.L; ++l) {
      os << (l > 1 ? "," : "") << "{\"traffic\":" << gb::traffic(op, s, l)
         << ",\"footprint\":" << gb::footprint_elems(op, s, l) << ",\"footprint_bytes\":" << gb::footprint_bytes(op, s, l)
         << ",\"capacity_ok\":" << (gb::capacity_ok(op, hw, s, l) ? "true" : "false") << "}";
    }
    os << "],\"utilization\":" << gb::json::num(gb::utilization(op, hw, s));
    if (s.complete()) os << ",\"cost\":" << gb::cost_json(gb::cost_of(op, hw, s, m), hw);
    os << ",\"vthread_benefits\":[";
    bool first = true;
    for (int a = 0; a < op.naxes; ++a) {
      if (op.ax[a].reduce) continue;
      for (int64_t v : {1, 2, 4, 8}) {
        os << (first ? "" : ",") << "[" << a << "," << v << "," << gb::json::num(gb::benefit_vthread(op, hw, s, a, v))
           << "]";
        first = false;
      }
    }
    gb::Action step;
    os << "],\"greedy_step\":";
    if (gb::greedy_fit_step(op, s, step))
      os << "[" << static_cast<int>(step.kind) << "," << step.axis << "," << step.factor << "]";
    else
      os << "null";
    os << ",\"legal\":[";
    first = true;
    for (int kind = 0; kind < 4; ++kind)
      for (int a = -1; a < op.naxes; ++a)
        for (int64_t f : {0, 1, 2, 4, 8}) {
          gb::Action act{static_cast<gb::ActKind>(kind), a, f};
          if (!s.legal(op, act)) continue;
          os << (first ? "" : ",") << "[" << kind << "," << a << "," << f << "]";
          first = false;
        }
    os << "],\"b200_feasible\":" << (gb::b200_feasible(op, hw, s, s.cur) ? "true" : "false") << "}";
    return emit(os.str(), buf, cap, need);
  });
}

int gensor_candidates(const gensor_op* o, const gensor_hw* h, const char* tr, const gensor_engine_cfg* cfg,
                      int iteration, char* buf, size_t cap, size_t* need) {
  if (!o || !h || !tr) return fail(GENSOR_EINVALID, "null argument");
  return guarded([&]() -> int {
    gb::Sched s = replay(o->op, h->hw, trace_from(tr));
    std::vector<gb::Candidate> c;
    gb::EngineCfg ec = cfg_from(cfg);
    if (!gb::candidates(o->op, h->hw, s, ec, iteration, c))
      throw gb::Error(gb::Code::NoLegalAction, "no selectable action from " + s.repr(o->op));
    std::ostringstream os;
    os << "{\"candidates\":[";
    for (size_t i = 0; i < c.size(); ++i)
      os << (i ? "," : "") << "[[" << static_cast<int>(c[i].action.kind) << "," << c[i].action.axis << ","
         << c[i].action.factor << "]," << gb::json::num(c[i].benefit) << "," << gb::json::num(c[i].probability) << "]";
    os << "]}";
    return emit(os.str(), buf, cap, need);
  });
}

double gensor_caching_benefit(double ll, double bl, double lh, double bh, double s) {
  return gb::caching_benefit(ll, bl, lh, bh, s);
}
double gensor_vthread_conflict_ratio(int64_t x, int64_t w, int64_t v) { return gb::vthread_ratio(x, w, v); }
double gensor_anneal_cache_multiplier(int it) { return gb::anneal_cache_multiplier(it); }
double gensor_record_probability(double t) { return gb::record_probability(t); }
uint64_t gensor_derive_seed(uint64_t seed, int r) { return gb::derive_seed(seed, r); }

int gensor_kernel_prepare(const gensor_op* op, const gensor_schedule* s, int index, int variant, gensor_kernel** out) {
  if (!op || !s || !out) return fail(GENSOR_EINVALID, "null argument");
  return guarded([&]() -> int {
    if (index < 0 || index >= static_cast<int>(s->results.size()))
      return fail(GENSOR_EINVALID, "schedule index out of range");
    check_schedule_op(op->op, *s);
    const gb::Sched& st = s->results[static_cast<size_t>(index)].state;
    if (!st.complete()) throw gb::Error(gb::Code::IncompleteState, "kernel needs a complete schedule");
    auto* k = new gensor_kernel;
    try {
      k->k = gb::dev::prepare(op->op, st, variant);
    } catch (...) {
      delete k;
      throw;
    }
    *out = k;
    return GENSOR_OK;
  });
}

int gensor_kernel_info(const gensor_kernel* k, char* buf, size_t cap, size_t* need) {
  if (!k) return fail(GENSOR_EINVALID, "null kernel");
  return guarded([&]() -> int { return emit(gb::dev::info(k->k), buf, cap, need); });
}

int gensor_execute(const gensor_kernel* k, const void* const* d_in, int n_in, void* d_out, void* stream) {
  if (!k || !d_out || (n_in > 0 && !d_in)) return fail(GENSOR_EINVALID, "null argument");
  return guarded([&]() -> int {
    gb::dev::execute(k->k, d_in, n_in, d_out, nullptr, 0, stream);
    return GENSOR_OK;
  });
}

int gensor_kernel_workspace_size(const gensor_kernel* k, size_t* bytes) {
  if (!k || !bytes) return fail(GENSOR_EINVALID, "null argument");
  *bytes = gb::dev::workspace_bytes(k->k);
  return GENSOR_OK;
}

int gensor_execute_ws(const gensor_kernel* k, const void* const* d_in, int n_in, void* d_out, void* d_workspace,
                      size_t workspace_bytes, void* stream) {
  if (!k || !d_out || (n_in > 0 && !d_in)) return fail(GENSOR_EINVALID, "null argument");
  if (gb::dev::workspace_bytes(k->k) > 0 && !d_workspace) return fail(GENSOR_EINVALID, "null workspace");
  return guarded([&]() -> int {
    gb::dev::execute(k->k, d_in, n_in, d_out, d_workspace, workspace_bytes, stream);
    return GENSOR_OK;
  });
}

int gensor_execute_host(gensor_kernel* k, const void* const* h_in, int n_in, void* h_out, void* stream) {
  if (!k || !h_out || (n_in > 0 && !h_in)) return fail(GENSOR_EINVALID, "null argument");
  return guarded([&]() -> int {
    gb::dev::execute_host(k->k, h_in, n_in, h_out, stream);
    return GENSOR_OK;
  });
}

int gensor_rerank(const gensor_op* op, const gensor_schedule* s, int variant, const void* const* d_in, int n_in,
                  void* d_out, void* stream, int iters, char* buf, size_t cap, size_t* need) {
  if (!op || !s || !d_out || (n_in > 0 && !d_in)) return fail(GENSOR_EINVALID, "null argument");
  return guarded([&]() -> int {
    check_schedule_op(op->op, *s);
    std::vector<std::pair<float, int>> t;
    std::vector<std::string> plans;
    std::ostringstream os;
    os << "{\"ms\":[";
    for (size_t i = 0; i < s->results.size(); ++i) {
      const gb::Sched& st = s->results[i].state;
      float ms = -1.f;
      if (st.complete()) {
        gb::dev::Kernel* k = gb::dev::prepare(op->op, st, variant);
        plans.push_back(gb::dev::plan(k));
        try {
          ms = gb::dev::time_execute(k, d_in, n_in, d_out, stream, iters);
        } catch (...) {
          gb::dev::destroy(k);
          throw;
        }
        gb::dev::destroy(k);
        t.emplace_back(ms, static_cast<int>(i));
      } else {
        plans.push_back("null");
      }
      os << (i ? "," : "") << gb::json::num(ms);
    }
    std::stable_sort(t.begin(), t.end());  // ties keep the analytical order
    os << "],\"order\":[";
    for (size_t i = 0; i < t.size(); ++i) os << (i ? "," : "") << t[i].second;
    os << "],\"best\":" << (t.empty() ? -1 : t[0].second) << ",\"plans\":[";
    for (size_t i = 0; i < plans.size(); ++i) os << (i ? "," : "") << plans[i];
    os << "]}";
    return emit(os.str(), buf, cap, need);
  });
}

void gensor_kernel_free(gensor_kernel* k) {
  if (!k) return;
  gb::dev::destroy(k->k);
  delete k;
}

uint64_t gensor_launch_count(void) { return gb::dev::launch_count(); }

int gensor_kernel_set_timing(gensor_kernel* k, int enable) {
  if (!k) return fail(GENSOR_EINVALID, "null kernel");
  return guarded([&]() -> int {
    gb::dev::set_timing(k->k, enable != 0);
    return GENSOR_OK;
  });
}

int gensor_kernel_timings(gensor_kernel* k, float* ms, int cap, int* n, char* names, size_t names_cap) {
  if (!k || !n) return fail(GENSOR_EINVALID, "null argument");
  return guarded([&]() -> int {
    auto t = gb::dev::timings(k->k);
    *n = static_cast<int>(t.size());
    std::string js = "[";
    for (size_t i = 0; i < t.size(); ++i) {
      if (ms && static_cast<int>(i) < cap) ms[i] = t[i].second;
      js += (i ? "," : "") + gb::json::quote(t[i].first);
    }
    js += "]";
    size_t need = 0;
    if (names) return emit(js, names, names_cap, &need);
    return GENSOR_OK;
  });
}

}  // extern "C"
