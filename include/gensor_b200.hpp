// gensor-b200 C++ facade: the reference's C++ surface (namespace gensor, include/gensor/*.hpp)
// re-exposed over the C-ABI in gensor_b200.h, header-only, so a reference-style caller swaps
//   #include "gensor/engine.hpp"        ->  #include "gensor_b200.hpp"
//   gensor::optimize(op, hw, cfg)       ->  gensor_b200::optimize(op, hw, cfg)
// and gains the execute half the reference only specifies.
//
//   reference                                   facade
//   TensorOpSpec::parse_text  op_spec.hpp:51    TensorOpSpec::parse_text
//   HardwareSpec::load_text   hardware.hpp:31   HardwareSpec::load_text / HardwareSpec::b200
//   EngineConfig              engine.hpp:14-24  EngineConfig (+ mode, threads)
//   optimize / construct      engine.hpp:83-99  optimize / construct -> Schedules
//   construct_tree            tree_baseline.hpp:26   construct_tree
//   gensor::Error{code()}     error.hpp:29-40   gensor_b200::Error{code()} (same ordinals, same what())
//   (SPEC) lower + interpret  SPEC.md:470-487   Kernel(op, schedules, i, variant).execute(...)
//
// Lifetimes follow the reference: an op outlives its schedules and kernels (etir.hpp:75).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "gensor_b200.h"

namespace gensor_b200 {

class Error : public std::runtime_error {
 public:
  Error(int status, const std::string& what) : std::runtime_error(what), status_(status) {}
  int status() const { return status_; }
  // The reference's ErrorCode ordinal (error.hpp:8-27), or -1 for the B200-only codes.
  int code() const { return status_ >= 1 && status_ <= 18 ? status_ - 1 : -1; }

 private:
  int status_;
};

inline void check(int status) {
  if (status != GENSOR_OK) throw Error(status, gensor_last_error());
}

template <typename F>
std::string json_out(F&& call) {
  size_t need = 0;
  int st = call(nullptr, 0, &need);
  if (st != GENSOR_OK && st != GENSOR_ETRUNCATED) check(st);
  std::string buf(need, '\0');
  check(call(buf.data(), buf.size(), &need));
  buf.resize(need ? need - 1 : 0);
  return buf;
}

class TensorOpSpec {
 public:
  static TensorOpSpec parse_text(const std::string& json) {
    gensor_op* h = nullptr;
    check(gensor_op_parse(json.c_str(), &h));
    return TensorOpSpec(h);
  }
  TensorOpSpec(TensorOpSpec&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
  TensorOpSpec& operator=(TensorOpSpec&& o) noexcept {
    std::swap(h_, o.h_);
    return *this;
  }
  TensorOpSpec(const TensorOpSpec&) = delete;
  ~TensorOpSpec() { gensor_op_free(h_); }
  std::string info_json() const {
    return json_out([&](char* b, size_t c, size_t* n) { return gensor_op_info(h_, b, c, n); });
  }
  const gensor_op* handle() const { return h_; }

 private:
  explicit TensorOpSpec(gensor_op* h) : h_(h) {}
  gensor_op* h_;
};

class HardwareSpec {
 public:
  static HardwareSpec load_text(const std::string& json) {
    gensor_hw* h = nullptr;
    check(gensor_hw_load(json.c_str(), &h));
    return HardwareSpec(h);
  }
  // B200 device model: live device query + measured peaks (MEASURED_PEAKS.json text or empty).
  static HardwareSpec b200(int device, const std::string& measured_peaks_json = "") {
    gensor_hw* h = nullptr;
    check(gensor_hw_b200(device, measured_peaks_json.empty() ? nullptr : measured_peaks_json.c_str(), &h));
    return HardwareSpec(h);
  }
  HardwareSpec(HardwareSpec&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
  HardwareSpec(const HardwareSpec&) = delete;
  ~HardwareSpec() { gensor_hw_free(h_); }
  std::string to_json() const {
    return json_out([&](char* b, size_t c, size_t* n) { return gensor_hw_json(h_, b, c, n); });
  }
  const gensor_hw* handle() const { return h_; }

 private:
  explicit HardwareSpec(gensor_hw* h) : h_(h) {}
  gensor_hw* h_;
};

struct EngineConfig {
  double t0 = 1048576.0;
  double threshold = 1.0;
  int restarts = 8;
  uint64_t seed = 0;
  int top_k = 10;
  std::vector<int64_t> vthread_options{1, 2, 4, 8};
  int64_t max_tile_factor = 2;
  int mode = GENSOR_MODE_REFERENCE_COMPAT;
  int threads = 0;

  gensor_engine_cfg to_c() const {
    gensor_engine_cfg c;
    gensor_engine_cfg_init(&c);
    c.t0 = t0;
    c.threshold = threshold;
    c.restarts = restarts;
    c.seed = seed;
    c.top_k = top_k;
    c.n_vthread_options = static_cast<int32_t>(vthread_options.size() < 8 ? vthread_options.size() : 8);
    for (int i = 0; i < c.n_vthread_options; ++i) c.vthread_options[i] = vthread_options[static_cast<size_t>(i)];
    c.max_tile_factor = max_tile_factor;
    c.mode = mode;
    c.threads = threads;
    return c;
  }
};

// Ranked ScheduleResults (engine.hpp:67-73), as JSON per result: state, trace, cost, seed.
class Schedules {
 public:
  Schedules(Schedules&& o) noexcept : h_(std::exchange(o.h_, nullptr)), n_(o.n_) {}
  Schedules(const Schedules&) = delete;
  ~Schedules() { gensor_schedule_free(h_); }
  int size() const { return n_; }
  std::string json(int index) const {
    return json_out([&](char* b, size_t c, size_t* n) { return gensor_schedule_json(h_, index, b, c, n); });
  }
  // Portable C source of result `index`'s loop nest (SPEC.md:488-496 emit_source).
  std::string emit_source(int index) const {
    return json_out([&](char* b, size_t c, size_t* n) { return gensor_emit_source(h_, index, b, c, n); });
  }
  const gensor_schedule* handle() const { return h_; }

 private:
  friend Schedules optimize(const TensorOpSpec&, const HardwareSpec&, const EngineConfig&);
  friend Schedules construct(const TensorOpSpec&, const HardwareSpec&, const EngineConfig&);
  friend Schedules construct_tree(const TensorOpSpec&, const HardwareSpec&, int, int);
  Schedules(gensor_schedule* h, int n) : h_(h), n_(n) {}
  gensor_schedule* h_;
  int n_;
};

inline Schedules optimize(const TensorOpSpec& op, const HardwareSpec& hw, const EngineConfig& cfg = {}) {
  gensor_schedule* h = nullptr;
  int n = 0;
  const gensor_engine_cfg c = cfg.to_c();
  check(gensor_optimize(op.handle(), hw.handle(), &c, &h, &n));
  return Schedules(h, n);
}

inline Schedules construct(const TensorOpSpec& op, const HardwareSpec& hw, const EngineConfig& cfg = {}) {
  gensor_schedule* h = nullptr;
  int n = 0;
  const gensor_engine_cfg c = cfg.to_c();
  check(gensor_construct(op.handle(), hw.handle(), &c, &h, &n));
  return Schedules(h, n);
}

inline Schedules construct_tree(const TensorOpSpec& op, const HardwareSpec& hw, int beam_width = 4,
                                int mode = GENSOR_MODE_REFERENCE_COMPAT) {
  gensor_schedule* h = nullptr;
  int n = 0;
  check(gensor_construct_tree(op.handle(), hw.handle(), beam_width, mode, &h, &n));
  return Schedules(h, n);
}

// The execute step: a kernel instantiated from schedule result `index` (lower(state)), run on
// device buffers (execute) or host buffers (execute_host, the interpreter's convention).
class Kernel {
 public:
  Kernel(const TensorOpSpec& op, const Schedules& s, int index = 0, int variant = GENSOR_VARIANT_AUTO) {
    check(gensor_kernel_prepare(op.handle(), s.handle(), index, variant, &h_));
  }
  Kernel(Kernel&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
  Kernel(const Kernel&) = delete;
  ~Kernel() { gensor_kernel_free(h_); }
  void execute(const std::vector<const void*>& d_inputs, void* d_output, void* stream = nullptr) const {
    check(gensor_execute(h_, d_inputs.data(), static_cast<int>(d_inputs.size()), d_output, stream));
  }
  void execute_host(const std::vector<const void*>& h_inputs, void* h_output, void* stream = nullptr) {
    check(gensor_execute_host(h_, h_inputs.data(), static_cast<int>(h_inputs.size()), h_output, stream));
  }
  std::string info_json() const {
    return json_out([&](char* b, size_t c, size_t* n) { return gensor_kernel_info(h_, b, c, n); });
  }

 private:
  gensor_kernel* h_ = nullptr;
};

}  // namespace gensor_b200
