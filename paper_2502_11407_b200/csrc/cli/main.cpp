// gensor-b200: the command-line front end (the SPEC's `cli` module, and the
// codegen-interp `verify`/`emit` interfaces; the reference ships none of it —
// its CMake names a missing tools/ directory). Built over the public C-ABI only, so it doubles
// as a complete reference-style caller of libgensor_b200.so.
//
//   schedule      --op F --hw F|b200[:dev] [--engine graph|tree|both] [engine flags] [--out DIR]
//                 -> DIR/results.json (graph) / DIR/results_tree.json (tree) + a summary
//   compare       --suite F --hw F|b200 [--seeds 0,1,..] [--out F.csv]   graph vs tree CSV
//   verify        --results F [--variant V] [--no-exec] [--tol X] [--seed N]
//                 replays every trace to its stored state (ReplayMismatch otherwise), then runs
//                 each schedule's B200 kernel on seeded inputs against reference_compute
//   emit          --results F [--index I] [--out F]       portable C source of the loop nest
//   cost explain  --op F --hw F --trace JSON | --results F [--index I]
//   analyze       --op F --hw F [--max-states N] [--no-inv-tile] [--detail]   chain report JSON
//
// Engine flags: --seed --t0 --threshold --restarts --top-k --mode reference|b200 --beam.
// Exit codes: 0 success, 1 partial failure, 2 usage/config error, 3 resource cap.
// Output files are byte-identical for identical inputs (no clocks or paths inside them).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../host/error.hpp"
#include "../host/json.hpp"
#include "gensor_b200.h"

// The JSON reader (host/json.cpp, linked in directly) reports malformed files as ConfigError;
// the library's own code_name() is not exported, so the CLI names the one code it can see.
const char* gb::code_name(gb::Code c) { return c == gb::Code::ConfigError ? "ConfigError" : "Error"; }

namespace {

namespace J = gb::json;

struct Usage : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct Status : std::runtime_error {  // a C-ABI failure: exit 2 for config errors, 1 otherwise
  int code;
  Status(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void check(int st) {
  if (st != GENSOR_OK) throw Status(st, gensor_last_error());
}

template <class F>
std::string text_out(F&& call) {
  size_t need = 0;
  int st = call(nullptr, 0, &need);
  if (st != GENSOR_OK && st != GENSOR_ETRUNCATED) check(st);
  std::string buf(need, '\0');
  check(call(buf.data(), buf.size(), &need));
  buf.resize(need ? need - 1 : 0);
  return buf;
}

std::string read_file(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw Usage("cannot read '" + path + "'");
  std::ostringstream os;
  os << f.rdbuf();
  return os.str();
}

void write_file(const std::string& path, const std::string& text) {
  std::ofstream f(path, std::ios::binary);
  if (!f) throw Usage("cannot write '" + path + "'");
  f << text;
}

// ---- tiny JSON writer for the parsed documents we re-emit (stable key order = input order) --
void dump(const J::Value& v, std::ostringstream& os) {
  switch (v.type) {
    case J::Type::Null: os << "null"; break;
    case J::Type::Bool: os << (v.b ? "true" : "false"); break;
    case J::Type::Int: os << v.i; break;
    case J::Type::Double: os << J::num(v.d); break;
    case J::Type::String: os << J::quote(v.s); break;
    case J::Type::Array:
      os << "[";
      for (size_t i = 0; i < v.arr.size(); ++i) {
        if (i) os << ",";
        dump(v.arr[i], os);
      }
      os << "]";
      break;
    case J::Type::Object:
      os << "{";
      for (size_t i = 0; i < v.obj.size(); ++i) {
        if (i) os << ",";
        os << J::quote(v.obj[i].first) << ":";
        dump(v.obj[i].second, os);
      }
      os << "}";
      break;
  }
}
std::string dump(const J::Value& v) {
  std::ostringstream os;
  dump(v, os);
  return os.str();
}

// ---- arguments -------------------------------------------------------------------------------
struct Args {
  std::map<std::string, std::string> kv;
  bool has(const std::string& k) const { return kv.count(k) != 0; }
  std::string get(const std::string& k, const std::string& dflt = "") const {
    auto it = kv.find(k);
    return it == kv.end() ? dflt : it->second;
  }
  std::string need(const std::string& k) const {
    if (!has(k)) throw Usage("missing --" + k);
    return get(k);
  }
  double num(const std::string& k, double dflt) const {
    if (!has(k)) return dflt;
    try {
      size_t pos = 0;
      double v = std::stod(get(k), &pos);
      if (pos != get(k).size()) throw std::invalid_argument("trailing");
      return v;
    } catch (const std::exception&) {
      throw Usage("--" + k + ": not a number: '" + get(k) + "'");
    }
  }
};

Args parse_args(int argc, char** argv, int first) {
  static const char* kFlags[] = {"no-exec", "quiet", "no-inv-tile", "detail"};
  Args a;
  for (int i = first; i < argc; ++i) {
    std::string s = argv[i];
    if (s.rfind("--", 0) != 0) throw Usage("unexpected argument '" + s + "'");
    s = s.substr(2);
    bool flag = false;
    for (const char* f : kFlags) flag |= s == f;
    if (flag) {
      a.kv[s] = "1";
    } else {
      if (i + 1 >= argc) throw Usage("--" + s + " needs a value");
      a.kv[s] = argv[++i];
    }
  }
  return a;
}

// ---- handles ---------------------------------------------------------------------------------
struct Op {
  gensor_op* h = nullptr;
  explicit Op(const std::string& json) { check(gensor_op_parse(json.c_str(), &h)); }
  ~Op() { gensor_op_free(h); }
  std::string info() const {
    return text_out([&](char* b, size_t c, size_t* n) { return gensor_op_info(h, b, c, n); });
  }
};
struct Hw {
  gensor_hw* h = nullptr;
  explicit Hw(const std::string& spec, const std::string& peaks_path) {
    if (spec == "b200" || spec.rfind("b200:", 0) == 0) {
      const int dev = spec.size() > 5 ? std::atoi(spec.c_str() + 5) : 0;
      std::string peaks;
      if (!peaks_path.empty()) peaks = read_file(peaks_path);
      check(gensor_hw_b200(dev, peaks.empty() ? nullptr : peaks.c_str(), &h));
    } else {
      const std::string text = spec.size() && spec[0] == '{' ? spec : read_file(spec);
      check(gensor_hw_load(text.c_str(), &h));
    }
  }
  ~Hw() { gensor_hw_free(h); }
  std::string json() const {
    return text_out([&](char* b, size_t c, size_t* n) { return gensor_hw_json(h, b, c, n); });
  }
};
struct Sch {
  gensor_schedule* h = nullptr;
  int n = 0;
  ~Sch() { gensor_schedule_free(h); }
  std::string json(int i) const {
    return text_out([&](char* b, size_t c, size_t* nn) { return gensor_schedule_json(h, i, b, c, nn); });
  }
};
struct Kern {
  gensor_kernel* h = nullptr;
  ~Kern() { gensor_kernel_free(h); }
};

std::string op_text(const Args& a) {
  const std::string s = a.need("op");
  return s.size() && s[0] == '{' ? s : read_file(s);
}

int mode_of(const std::string& m) {
  if (m == "reference" || m == "ref") return GENSOR_MODE_REFERENCE_COMPAT;
  if (m == "b200") return GENSOR_MODE_B200;
  throw Usage("--mode must be reference|b200, got '" + m + "'");
}
const char* mode_name(int m) { return m == GENSOR_MODE_B200 ? "b200" : "reference"; }

gensor_engine_cfg engine_cfg(const Args& a, int mode) {
  gensor_engine_cfg c;
  gensor_engine_cfg_init(&c);
  c.t0 = a.num("t0", c.t0);
  c.threshold = a.num("threshold", c.threshold);
  c.restarts = static_cast<int32_t>(a.num("restarts", c.restarts));
  c.top_k = static_cast<int32_t>(a.num("top-k", c.top_k));
  c.seed = static_cast<uint64_t>(a.num("seed", 0));
  c.mode = mode;
  return c;
}

std::string cfg_json(const gensor_engine_cfg& c, int beam) {
  std::ostringstream os;
  os << "{\"t0\":" << J::num(c.t0) << ",\"threshold\":" << J::num(c.threshold) << ",\"restarts\":" << c.restarts
     << ",\"top_k\":" << c.top_k << ",\"seed\":" << c.seed << ",\"mode\":\"" << mode_name(c.mode)
     << "\",\"beam\":" << beam << "}";
  return os.str();
}

double wall_ms(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

struct EngineRun {
  std::string results_json;  // full results.json text
  double best_cost = INFINITY;
  size_t best_trace = 0;
  int count = 0;
  double ms = 0;
};

EngineRun run_engine(const std::string& engine, const Op& op, const Hw& hw, const gensor_engine_cfg& c, int beam) {
  Sch s;
  const auto t0 = std::chrono::steady_clock::now();
  if (engine == "graph")
    check(gensor_optimize(op.h, hw.h, &c, &s.h, &s.n));
  else
    check(gensor_construct_tree(op.h, hw.h, beam, c.mode, &s.h, &s.n));
  EngineRun r;
  r.ms = wall_ms(t0);
  r.count = s.n;
  const std::string all = s.json(-1);
  const J::Value doc = J::parse(all);
  for (const auto& res : doc.arr) {
    const double cost = res.find("cost")->find("est_seconds")->as_double();
    if (cost < r.best_cost) {
      r.best_cost = cost;
      r.best_trace = res.find("trace")->arr.size();
    }
  }
  const J::Value opdoc = J::parse(op.info());
  std::ostringstream os;
  os << "{\"format\":\"gensor-b200/results/1\",\"engine\":\"" << engine << "\",\"op\":" << dump(*opdoc.find("json"))
     << ",\"hw\":" << hw.json() << ",\"config\":" << cfg_json(c, beam) << ",\"results\":" << all << "}\n";
  r.results_json = os.str();
  return r;
}

// ---- schedule --------------------------------------------------------------------------------
int cmd_schedule(const Args& a) {
  const std::string engine = a.get("engine", "graph");
  if (engine != "graph" && engine != "tree" && engine != "both") throw Usage("--engine must be graph|tree|both");
  Op op(op_text(a));
  Hw hw(a.need("hw"), a.get("peaks"));
  const gensor_engine_cfg c = engine_cfg(a, mode_of(a.get("mode", "reference")));
  const int beam = static_cast<int>(a.num("beam", 4));
  const std::string out = a.get("out", ".");
  const J::Value info = J::parse(op.info());
  std::printf("op %s\n", info.find("label")->as_string().c_str());
  double best[2] = {INFINITY, INFINITY};
  int k = 0;
  for (const char* e : {"graph", "tree"}) {
    ++k;
    if (engine != "both" && engine != e) continue;
    EngineRun r = run_engine(e, op, hw, c, beam);
    const std::string path = out + (std::string(e) == "graph" ? "/results.json" : "/results_tree.json");
    write_file(path, r.results_json);
    best[k - 1] = r.best_cost;
    std::printf("%-5s results=%d best_cost=%.6g s trace_len=%zu wall=%.2f ms -> %s\n", e, r.count, r.best_cost,
                r.best_trace, r.ms, path.c_str());
  }
  if (engine == "both") std::printf("graph/tree = %.6g\n", best[0] / best[1]);
  return 0;
}

// ---- compare ---------------------------------------------------------------------------------
std::vector<uint64_t> parse_seeds(const std::string& s) {
  std::vector<uint64_t> out;
  std::stringstream ss(s);
  std::string tok;
  while (std::getline(ss, tok, ','))
    if (!tok.empty()) out.push_back(std::stoull(tok));
  if (out.empty()) throw Usage("--seeds is empty");
  return out;
}

int cmd_compare(const Args& a) {
  const J::Value suite = J::parse(read_file(a.need("suite")));
  const J::Value* ops = suite.is_object() ? suite.find("ops") : &suite;
  if (!ops || !ops->is_array()) throw Usage("suite must be a JSON array (or {\"ops\": [...]})");
  if (ops->arr.empty()) throw Usage("empty suite");
  Hw hw(a.need("hw"), a.get("peaks"));
  const int mode = mode_of(a.get("mode", "reference"));
  const std::vector<uint64_t> seeds = parse_seeds(a.get("seeds", "0"));
  const int beam = static_cast<int>(a.num("beam", 4));
  std::ostringstream csv;
  csv << "op_label,tree_cost,graph_cost,ratio,graph_wall_ms,tree_wall_ms,status\n";
  double log_sum = 0;
  int ok_rows = 0, failed = 0;
  for (const J::Value& item : ops->arr) {
    const J::Value* opdoc = item.is_object() && item.has("op") ? item.find("op") : &item;
    std::string label = item.is_object() && item.has("label") ? item.find("label")->as_string() : "";
    try {
      Op op(dump(*opdoc));
      if (label.empty()) label = J::parse(op.info()).find("label")->as_string();
      double g = INFINITY, gms = 0;
      for (uint64_t seed : seeds) {
        Args sa = a;
        sa.kv["seed"] = std::to_string(seed);
        EngineRun r = run_engine("graph", op, hw, engine_cfg(sa, mode), beam);
        g = std::min(g, r.best_cost);
        gms += r.ms;
      }
      EngineRun t = run_engine("tree", op, hw, engine_cfg(a, mode), beam);
      char row[512];
      std::snprintf(row, sizeof row, "\"%s\",%.9g,%.9g,%.9g,%.3f,%.3f,ok\n", label.c_str(), t.best_cost, g,
                    g / t.best_cost, gms / static_cast<double>(seeds.size()), t.ms);
      csv << row;
      log_sum += std::log(g / t.best_cost);
      ++ok_rows;
    } catch (const std::exception& e) {
      std::string msg = e.what();
      std::replace(msg.begin(), msg.end(), '"', '\'');
      csv << "\"" << label << "\",,,,,,\"error: " << msg << "\"\n";
      ++failed;
    }
  }
  char geo[128];
  std::snprintf(geo, sizeof geo, "geomean,,,%.9g,,,%s\n", ok_rows ? std::exp(log_sum / ok_rows) : NAN,
                failed ? "partial" : "ok");
  csv << geo;
  if (a.has("out"))
    write_file(a.get("out"), csv.str());
  else
    std::fputs(csv.str().c_str(), stdout);
  return failed ? 1 : 0;
}

// ---- reference_compute (verify's checker: the Table III formulas) ----------
struct OpInfo {
  std::string kind;
  int dtype_bytes = 4;
  int64_t batch = 1;
  std::vector<int64_t> ext;
  std::vector<bool> reduce;
  struct T {
    std::vector<int64_t> coef;
    int64_t elems = 1;
  };
  std::vector<T> t;  // inputs..., output last
};

OpInfo op_info(const Op& op) {
  const J::Value v = J::parse(op.info());
  OpInfo o;
  o.kind = v.find("kind")->as_string();
  o.dtype_bytes = static_cast<int>(v.find("dtype_bytes")->as_int());
  o.batch = v.find("batch")->as_int();
  for (const auto& ax : v.find("axes")->arr) {
    o.ext.push_back(ax.arr[1].as_int());
    o.reduce.push_back(ax.arr[3].b);
  }
  for (const auto& t : v.find("tensors")->arr) {
    OpInfo::T tt;
    for (const auto& c : t.find("coef")->arr) tt.coef.push_back(c.as_int());
    for (const auto& d : t.find("true_dims")->arr) tt.elems *= d.as_int();
    o.t.push_back(tt);
  }
  return o;
}

std::vector<double> reference_compute(const OpInfo& o, const std::vector<std::vector<float>>& in) {
  const size_t nout = static_cast<size_t>(o.t.back().elems * o.batch);
  std::vector<double> y(nout, 0.0);
  if (o.kind == "softmax") {
    const int64_t M = o.ext[0], N = o.ext[1];
    for (int64_t m = 0; m < M; ++m) {
      const float* x = in[0].data() + m * N;
      double mx = -INFINITY, sum = 0;
      for (int64_t n = 0; n < N; ++n) mx = std::max(mx, static_cast<double>(x[n]));
      for (int64_t n = 0; n < N; ++n) sum += std::exp(static_cast<double>(x[n]) - mx);
      for (int64_t n = 0; n < N; ++n) y[static_cast<size_t>(m * N + n)] = std::exp(static_cast<double>(x[n]) - mx) / sum;
    }
    return y;
  }
  const size_t na = o.ext.size();
  const size_t nin = in.size();
  int64_t divisor = 1;
  for (size_t a = 0; a < na; ++a)
    if (o.reduce[a]) divisor *= o.ext[a];
  for (int64_t b = 0; b < o.batch; ++b) {
    std::vector<int64_t> idx(na, 0);
    for (;;) {
      int64_t off[4] = {0, 0, 0, 0};
      for (size_t a = 0; a < na; ++a)
        for (size_t ti = 0; ti <= nin; ++ti) off[ti] += idx[a] * o.t[ti].coef[a];
      double v = in[0][static_cast<size_t>(b * o.t[0].elems + off[0])];
      if (nin > 1) v *= in[1][static_cast<size_t>(b * o.t[1].elems + off[1])];
      y[static_cast<size_t>(b * o.t[nin].elems + off[nin])] += v;
      int a = static_cast<int>(na) - 1;
      for (; a >= 0; --a) {
        if (++idx[static_cast<size_t>(a)] < o.ext[static_cast<size_t>(a)]) break;
        idx[static_cast<size_t>(a)] = 0;
      }
      if (a < 0) break;
    }
  }
  if (o.kind == "avgpool2d")
    for (double& v : y) v /= static_cast<double>(divisor);
  return y;
}

uint16_t to_bf16(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7fffu + ((u >> 16) & 1u);  // round to nearest even (finite inputs)
  return static_cast<uint16_t>(u >> 16);
}
float from_bf16(uint16_t h) {
  uint32_t u = static_cast<uint32_t>(h) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

double variant_tol(const std::string& name) {
  if (name == "tc_tf32") return 2e-3;
  if (name == "tc_bf16") return 1e-2;
  if (name == "simt_parity") return 1e-6;  // SPEC.md:497 single-precision mode
  return 1e-5;                             // fp32 FFMA families (simt_f32, stream)
}

int variant_of(const std::string& v) {
  static const std::pair<const char*, int> kV[] = {{"auto", GENSOR_VARIANT_AUTO},       {"simt_parity", 0},
                                                   {"simt_f32", 1},                   {"tc_tf32", 2},
                                                   {"tc_bf16", 3},                    {"stream", 4}};
  for (const auto& p : kV)
    if (v == p.first) return p.second;
  throw Usage("unknown --variant '" + v + "'");
}

struct ExecCheck {
  std::string variant;
  bool exact_ok = true;
  double err = 0, tol = 0;
};

ExecCheck exec_check(const Op& op, const OpInfo& o, const Sch& s, int index, int variant, uint64_t seed, double tol_override) {
  Kern k;
  check(gensor_kernel_prepare(op.h, s.h, index, variant, &k.h));
  ExecCheck ec;
  const J::Value kinfo = J::parse(text_out([&](char* b, size_t c, size_t* n) { return gensor_kernel_info(k.h, b, c, n); }));
  ec.variant = kinfo.find("variant_name")->as_string();
  const bool bf16 = o.dtype_bytes == 2;
  // bf16 outputs carry 8 mantissa bits whatever the accumulation: the bf16 bar applies.
  ec.tol = tol_override > 0 ? tol_override : std::max(variant_tol(ec.variant), bf16 ? 1e-2 : 0.0);
  const size_t nin = o.t.size() - 1;
  const size_t nout = static_cast<size_t>(o.t.back().elems * o.batch);
  std::mt19937_64 rng(seed);
  const bool integer_exact = o.kind == "gemm" || o.kind == "gemv" || o.kind == "conv2d" || o.kind == "dwconv2d";
  for (int pass = integer_exact ? 0 : 1; pass < 2; ++pass) {
    std::vector<std::vector<float>> xs(nin);
    std::vector<std::vector<uint16_t>> xh(nin);
    std::vector<const void*> ptrs;
    for (size_t ti = 0; ti < nin; ++ti) {
      const size_t n = static_cast<size_t>(o.t[ti].elems * o.batch);
      xs[ti].resize(n);
      for (float& v : xs[ti]) {
        const double u = static_cast<double>(rng() >> 11) * 0x1.0p-53;
        v = pass == 0 ? static_cast<float>(static_cast<int>(u * 5.0) - 2) : static_cast<float>(2.0 * u - 1.0);
      }
      if (bf16) {
        xh[ti].resize(n);
        for (size_t i = 0; i < n; ++i) {
          xh[ti][i] = to_bf16(xs[ti][i]);
          xs[ti][i] = from_bf16(xh[ti][i]);
        }
        ptrs.push_back(xh[ti].data());
      } else {
        ptrs.push_back(xs[ti].data());
      }
    }
    const std::vector<double> ref = reference_compute(o, xs);
    std::vector<float> got(nout);
    std::vector<uint16_t> goth(bf16 ? nout : 0);
    check(gensor_execute_host(k.h, ptrs.data(), static_cast<int>(nin), bf16 ? static_cast<void*>(goth.data()) : got.data(),
                              nullptr));
    if (bf16)
      for (size_t i = 0; i < nout; ++i) got[i] = from_bf16(goth[i]);
    if (pass == 0) {
      for (size_t i = 0; i < nout; ++i) {
        const float want = bf16 ? from_bf16(to_bf16(static_cast<float>(ref[i]))) : static_cast<float>(ref[i]);
        if (!(got[i] == want)) ec.exact_ok = false;
      }
    } else {
      double num = 0, den = 0;
      for (size_t i = 0; i < nout; ++i) {
        const double d = std::fabs(static_cast<double>(got[i]) - ref[i]);
        num = std::isnan(d) ? INFINITY : std::max(num, d);
        den = std::max(den, std::fabs(ref[i]));
      }
      ec.err = den > 0 ? num / den : num;
    }
  }
  return ec;
}

// ---- verify ----------------------------------------------------------------------------------
int cmd_verify(const Args& a) {
  const J::Value doc = J::parse(read_file(a.need("results")));
  const J::Value* opdoc = doc.find("op");
  const J::Value* hwdoc = doc.find("hw");
  const J::Value* results = doc.find("results");
  const J::Value* cfg = doc.find("config");
  if (!opdoc || !hwdoc || !results || !results->is_array()) throw Usage("not a gensor-b200 results file");
  Op op(dump(*opdoc));
  Hw hw(dump(*hwdoc), "");
  const int mode = mode_of(cfg && cfg->has("mode") ? cfg->find("mode")->as_string() : "reference");
  const int variant = variant_of(a.get("variant", "auto"));
  const bool exec = !a.has("no-exec");
  const uint64_t seed = static_cast<uint64_t>(a.num("seed", 0));
  const double tol_override = a.num("tol", 0);
  const OpInfo o = op_info(op);
  int failed = 0;
  bool device = exec;
  for (size_t i = 0; i < results->arr.size(); ++i) {
    const J::Value& r = results->arr[i];
    const std::string trace = dump(*r.find("trace"));
    const std::string want = r.find("state")->find("repr")->as_string();
    Sch s;
    int st = gensor_schedule_from_trace(op.h, hw.h, trace.c_str(), mode, &s.h);
    std::string got;
    if (st == GENSOR_OK) {
      s.n = gensor_schedule_count(s.h);
      got = J::parse(s.json(0)).find("state")->find("repr")->as_string();
    }
    if (st != GENSOR_OK || got != want) {
      std::printf("result %zu: ReplayMismatch: %s\n", i,
                  st != GENSOR_OK ? gensor_last_error() : ("replayed '" + got + "' != stored '" + want + "'").c_str());
      ++failed;
      continue;
    }
    if (!device) {
      std::printf("result %zu: replay ok  %s\n", i, want.c_str());
      continue;
    }
    try {
      const ExecCheck ec = exec_check(op, o, s, 0, variant, seed, tol_override);
      const bool pass = ec.exact_ok && ec.err <= ec.tol;
      std::printf("result %zu: replay ok  %-11s integer-exact=%s max_rel_err=%.3g tol=%.1g %s  %s\n", i,
                  ec.variant.c_str(), ec.exact_ok ? "yes" : "NO", ec.err, ec.tol, pass ? "PASS" : "FAIL", want.c_str());
      failed += pass ? 0 : 1;
    } catch (const Status& e) {
      if (e.code == GENSOR_ECUDA) {  // no usable device: replay-only from here on
        std::printf("result %zu: replay ok  (execute skipped: %s)\n", i, e.what());
        device = false;
      } else if (e.code == GENSOR_EUNSUPPORTED) {
        std::printf("result %zu: replay ok  (variant unsupported: %s)\n", i, e.what());
      } else {
        std::printf("result %zu: FAIL %s\n", i, e.what());
        ++failed;
      }
    }
  }
  std::printf("%s: %zu result(s), %d failed\n", failed ? "FAIL" : "PASS", results->arr.size(), failed);
  return failed ? 1 : 0;
}

// ---- emit / cost explain -----------------------------------------------------------------------
struct Loaded {
  std::unique_ptr<Op> op;
  std::unique_ptr<Hw> hw;
  Sch s;
};

void load_result(const Args& a, Loaded& L, int index) {
  const J::Value doc = J::parse(read_file(a.need("results")));
  const J::Value* results = doc.find("results");
  if (!doc.find("op") || !doc.find("hw") || !results) throw Usage("not a gensor-b200 results file");
  if (index < 0 || static_cast<size_t>(index) >= results->arr.size()) throw Usage("--index out of range");
  const J::Value* cfg = doc.find("config");
  L.op = std::make_unique<Op>(dump(*doc.find("op")));
  L.hw = std::make_unique<Hw>(dump(*doc.find("hw")), "");
  const int mode = mode_of(cfg && cfg->has("mode") ? cfg->find("mode")->as_string() : "reference");
  const std::string trace = dump(*results->arr[static_cast<size_t>(index)].find("trace"));
  check(gensor_schedule_from_trace(L.op->h, L.hw->h, trace.c_str(), mode, &L.s.h));
  L.s.n = gensor_schedule_count(L.s.h);
}

int cmd_emit(const Args& a) {
  Loaded L;
  load_result(a, L, static_cast<int>(a.num("index", 0)));
  const std::string src =
      text_out([&](char* b, size_t c, size_t* n) { return gensor_emit_source(L.s.h, 0, b, c, n); });
  if (a.has("out"))
    write_file(a.get("out"), src);
  else
    std::fputs(src.c_str(), stdout);
  return 0;
}

int cmd_cost_explain(const Args& a) {
  std::string out;
  if (a.has("results")) {
    const J::Value doc = J::parse(read_file(a.need("results")));
    const int index = static_cast<int>(a.num("index", 0));
    const J::Value* results = doc.find("results");
    if (!results || index < 0 || static_cast<size_t>(index) >= results->arr.size()) throw Usage("--index out of range");
    const J::Value* cfg = doc.find("config");
    Op op(dump(*doc.find("op")));
    Hw hw(dump(*doc.find("hw")), "");
    const int mode = mode_of(cfg && cfg->has("mode") ? cfg->find("mode")->as_string() : "reference");
    const std::string trace = dump(*results->arr[static_cast<size_t>(index)].find("trace"));
    out = text_out([&](char* b, size_t c, size_t* n) { return gensor_state_eval(op.h, hw.h, trace.c_str(), mode, b, c, n); });
  } else {
    Op op(op_text(a));
    Hw hw(a.need("hw"), a.get("peaks"));
    const std::string trace = a.need("trace");
    const int mode = mode_of(a.get("mode", "reference"));
    out = text_out([&](char* b, size_t c, size_t* n) { return gensor_state_eval(op.h, hw.h, trace.c_str(), mode, b, c, n); });
  }
  std::printf("%s\n", out.c_str());
  return 0;
}

// ---- analyze (markov-verify SPEC.md:380-457) ----------------------------------
int cmd_analyze(const Args& a) {
  Op op(op_text(a));
  Hw hw(a.need("hw"), a.get("peaks"));
  std::ostringstream caps;
  caps << "{\"max_states\":" << static_cast<int64_t>(a.num("max-states", 50000))
       << ",\"fixed_iteration\":" << static_cast<int64_t>(a.num("fixed-iteration", 10))
       << ",\"enable_inv_tile\":" << (a.has("no-inv-tile") ? 0 : 1) << ",\"max_tile_factor\":"
       << static_cast<int64_t>(a.num("max-tile-factor", 2)) << ",\"mode\":\"" << mode_name(mode_of(a.get("mode", "reference")))
       << "\",\"detail\":" << (a.has("detail") ? 1 : 0) << "}";
  const std::string c = caps.str();
  const std::string out =
      text_out([&](char* b, size_t cap, size_t* n) { return gensor_analyze(op.h, hw.h, c.c_str(), b, cap, n); }) + "\n";
  if (a.has("out"))
    write_file(a.get("out"), out);
  else
    std::fputs(out.c_str(), stdout);
  return 0;
}

void usage() {
  std::fputs(
      "usage: gensor-b200 <command> [flags]\n"
      "  schedule     --op F --hw F|b200[:dev] [--engine graph|tree|both] [--seed N] [--t0 X]\n"
      "               [--threshold X] [--restarts N] [--top-k N] [--mode reference|b200] [--beam N]\n"
      "               [--peaks MEASURED_PEAKS.json] [--out DIR]\n"
      "  compare      --suite F --hw F|b200 [--seeds 0,1,..] [--mode ..] [--out F.csv]\n"
      "  verify       --results F [--variant auto|simt_parity|simt_f32|tc_tf32|tc_bf16|stream]\n"
      "               [--no-exec] [--tol X] [--seed N]\n"
      "  emit         --results F [--index I] [--out F]\n"
      "  cost explain --op F --hw F --trace JSON [--mode ..] | --results F [--index I]\n"
      "  analyze      --op F --hw F [--max-states N] [--fixed-iteration N] [--no-inv-tile]\n"
      "               [--max-tile-factor N] [--mode ..] [--detail] [--out F]\n"
      "exit codes: 0 ok, 1 partial failure, 2 usage/config error, 3 resource cap\n",
      stderr);
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    usage();
    return 2;
  }
  const std::string cmd = argv[1];
  try {
    if (cmd == "schedule") return cmd_schedule(parse_args(argc, argv, 2));
    if (cmd == "compare") return cmd_compare(parse_args(argc, argv, 2));
    if (cmd == "verify") return cmd_verify(parse_args(argc, argv, 2));
    if (cmd == "emit") return cmd_emit(parse_args(argc, argv, 2));
    if (cmd == "analyze") return cmd_analyze(parse_args(argc, argv, 2));
    if (cmd == "cost" && argc >= 3 && std::string(argv[2]) == "explain") return cmd_cost_explain(parse_args(argc, argv, 3));
    if (cmd == "-h" || cmd == "--help" || cmd == "help") {
      usage();
      return 0;
    }
    usage();
    return 2;
  } catch (const Usage& e) {
    std::fprintf(stderr, "gensor-b200 %s: %s\n", cmd.c_str(), e.what());
    return 2;
  } catch (const Status& e) {
    std::fprintf(stderr, "gensor-b200 %s: %s\n", cmd.c_str(), e.what());
    return e.code == GENSOR_ESPACE_TOO_LARGE || e.code == GENSOR_ETOO_LARGE_TO_ENUMERATE ? 3 : 2;
  } catch (const std::exception& e) {  // JSON parse errors from the files we read
    std::fprintf(stderr, "gensor-b200 %s: %s\n", cmd.c_str(), e.what());
    return 2;
  }
}
