#include "hw.hpp"

#include <sstream>

#include "error.hpp"
#include "op.hpp"

namespace gb {

namespace {

double num_or(const json::Value& o, const char* key, double dflt) {
  const json::Value* v = o.find(key);
  return v ? v->as_double() : dflt;
}

int64_t int_or(const json::Value& o, const char* key, int64_t dflt) {
  const json::Value* v = o.find(key);
  return v ? v->as_int() : dflt;
}

}  // namespace

HwModel HwModel::load_text(const std::string& text) { return load(json::parse(text)); }

HwModel HwModel::load(const json::Value& doc) {
  HwModel hw;
  if (const json::Value* n = doc.find("name")) hw.name = n->as_string();
  const json::Value* lv = doc.find("levels");
  if (!lv || !lv->is_array() || lv->arr.empty())
    throw Error(Code::MissingLevel, "hardware spec needs a nonempty 'levels' array");

  for (const json::Value& lj : lv->arr) {
    MemLevel m;
    if (const json::Value* n = lj.find("name"))
      m.name = n->as_string();
    else
      m.name = "level" + std::to_string(hw.levels.size());
    const json::Value* cap = lj.find("capacity_bytes");
    if (cap && cap->is_string()) {
      if (cap->s != "unlimited") throw Error(Code::ConfigError, "capacity_bytes must be a number or \"unlimited\"");
      m.unlimited = true;
    } else {
      if (!cap) throw Error(Code::ConfigError, "level '" + m.name + "' missing capacity_bytes");
      m.capacity_bytes = cap->as_int();
      if (m.capacity_bytes <= 0) throw Error(Code::ConfigError, "level '" + m.name + "' capacity must be positive");
    }
    m.bandwidth = num_or(lj, "bandwidth_bytes_per_cycle", 0.0);
    m.latency = num_or(lj, "latency_cycles", 0.0);
    m.bank_width = int_or(lj, "bank_width_elems", 0);
    if (m.bandwidth <= 0.0) throw Error(Code::ConfigError, "level '" + m.name + "' bandwidth must be positive");
    if (m.latency < 0.0) throw Error(Code::ConfigError, "level '" + m.name + "' latency must be nonnegative");
    hw.levels.push_back(m);
  }

  for (size_t i = 1; i < hw.levels.size(); ++i) {
    const MemLevel& outer = hw.levels[i - 1];
    const MemLevel& inner = hw.levels[i];
    if (inner.unlimited) throw Error(Code::MonotonicityViolation, "only level 0 may be unlimited");
    if (!outer.unlimited && inner.capacity_bytes >= outer.capacity_bytes)
      throw Error(Code::MonotonicityViolation, "capacity of '" + inner.name + "' must be below '" + outer.name + "'");
    if (inner.bandwidth <= outer.bandwidth)
      throw Error(Code::MonotonicityViolation, "bandwidth of '" + inner.name + "' must exceed '" + outer.name + "'");
  }

  hw.peak_flops = num_or(doc, "peak_flops", 1.0e12);
  hw.clock_hz = num_or(doc, "clock_hz", 1.0e9);
  hw.max_threads_per_block = int_or(doc, "max_threads_per_block", 1024);
  if (hw.peak_flops <= 0 || hw.clock_hz <= 0 || hw.max_threads_per_block <= 0)
    throw Error(Code::ConfigError, "peak_flops, clock_hz and max_threads_per_block must be positive");
  if (const json::Value* vo = doc.find("vthread_options")) {
    hw.vthread_options.clear();
    for (const json::Value& v : vo->arr) {
      int64_t opt = v.as_int();
      if (opt < 1 || !is_pow2(opt)) throw Error(Code::ConfigError, "vthread options must be powers of two >= 1");
      hw.vthread_options.push_back(opt);
    }
    if (hw.vthread_options.empty()) throw Error(Code::ConfigError, "vthread_options must not be empty");
  }

  // Optional device block: a document written by to_json() for a B200 model round-trips.
  if (const json::Value* d = doc.find("b200")) {
    hw.is_b200 = true;
    DeviceLimits& L = hw.dev;
    L.sms = static_cast<int>(int_or(*d, "sms", L.sms));
    L.smem_per_block = int_or(*d, "smem_per_block", L.smem_per_block);
    L.smem_per_sm = int_or(*d, "smem_per_sm", L.smem_per_sm);
    L.regs_per_sm = int_or(*d, "regs_per_sm", L.regs_per_sm);
    L.max_regs_per_thread = static_cast<int>(int_or(*d, "max_regs_per_thread", L.max_regs_per_thread));
    L.max_threads_per_block = static_cast<int>(int_or(*d, "max_threads_per_block", L.max_threads_per_block));
    L.max_threads_per_sm = static_cast<int>(int_or(*d, "max_threads_per_sm", L.max_threads_per_sm));
    L.max_blocks_per_sm = static_cast<int>(int_or(*d, "max_blocks_per_sm", L.max_blocks_per_sm));
    L.l2_bytes = int_or(*d, "l2_bytes", L.l2_bytes);
    L.tmem_cols = int_or(*d, "tmem_cols", L.tmem_cols);
    L.sm_clock_hz = num_or(*d, "sm_clock_hz", L.sm_clock_hz);
    L.hbm_bytes_per_s = num_or(*d, "hbm_bytes_per_s", L.hbm_bytes_per_s);
    L.fp32_simt_flops = num_or(*d, "fp32_simt_flops", L.fp32_simt_flops);
    L.tf32_tc_flops = num_or(*d, "tf32_tc_flops", L.tf32_tc_flops);
    L.bf16_tc_flops = num_or(*d, "bf16_tc_flops", L.bf16_tc_flops);
  }
  return hw;
}

// B200 model. Level bandwidths are chip-aggregate bytes per SM-clock cycle so the cost model's
// Q·dtype / (B·clock) is a chip-level transfer time:
//   hbm3e : measured copy bandwidth / clock;
//   smem  : 128 B/clk/SM crossbar x SMs; capacity = max dynamic smem per block;
//   regs  : 4 B x 128 lanes x 4 operands... per SM x SMs; capacity = per-thread register budget
//           (the thread tile's footprint lives in registers).
// Latencies are SM cycles (HBM ~800, smem ~30, regs 1). Banked level = smem, 32 banks x 4 B.
HwModel HwModel::b200(const DeviceLimits& lim) {
  HwModel hw;
  hw.name = "b200";
  hw.is_b200 = true;
  hw.dev = lim;
  hw.clock_hz = lim.sm_clock_hz;
  hw.peak_flops = lim.fp32_simt_flops;
  hw.max_threads_per_block = lim.max_threads_per_block;
  MemLevel hbm{"hbm3e", true, 0, lim.hbm_bytes_per_s / lim.sm_clock_hz, 800.0, 0};
  MemLevel smem{"smem", false, lim.smem_per_block, 128.0 * lim.sms, 30.0, 32};
  MemLevel regs{"regs", false, 4LL * lim.max_regs_per_thread, 4.0 * 32 * 3 * 4 * lim.sms, 1.0, 0};
  hw.levels = {hbm, smem, regs};
  return hw;
}

int HwModel::banked_level() const {
  for (int i = num_levels() - 1; i >= 0; --i)
    if (levels[static_cast<size_t>(i)].bank_width > 0) return i;
  return -1;
}

std::string HwModel::to_json() const {
  std::ostringstream os;
  os << "{\"name\":" << json::quote(name) << ",\"peak_flops\":" << json::num(peak_flops)
     << ",\"clock_hz\":" << json::num(clock_hz) << ",\"max_threads_per_block\":" << max_threads_per_block
     << ",\"vthread_options\":[";
  for (size_t i = 0; i < vthread_options.size(); ++i) os << (i ? "," : "") << vthread_options[i];
  os << "],\"levels\":[";
  for (size_t i = 0; i < levels.size(); ++i) {
    const MemLevel& m = levels[i];
    os << (i ? "," : "") << "{\"name\":" << json::quote(m.name) << ",\"capacity_bytes\":";
    if (m.unlimited)
      os << "\"unlimited\"";
    else
      os << m.capacity_bytes;
    os << ",\"bandwidth_bytes_per_cycle\":" << json::num(m.bandwidth) << ",\"latency_cycles\":"
       << json::num(m.latency) << ",\"bank_width_elems\":" << m.bank_width << "}";
  }
  os << "]";
  if (is_b200) {
    const DeviceLimits& L = dev;
    os << ",\"b200\":{\"sms\":" << L.sms << ",\"smem_per_block\":" << L.smem_per_block
       << ",\"smem_per_sm\":" << L.smem_per_sm << ",\"regs_per_sm\":" << L.regs_per_sm
       << ",\"max_regs_per_thread\":" << L.max_regs_per_thread
       << ",\"max_threads_per_block\":" << L.max_threads_per_block
       << ",\"max_threads_per_sm\":" << L.max_threads_per_sm << ",\"max_blocks_per_sm\":" << L.max_blocks_per_sm
       << ",\"l2_bytes\":" << L.l2_bytes << ",\"tmem_cols\":" << L.tmem_cols
       << ",\"sm_clock_hz\":" << json::num(L.sm_clock_hz) << ",\"hbm_bytes_per_s\":" << json::num(L.hbm_bytes_per_s)
       << ",\"fp32_simt_flops\":" << json::num(L.fp32_simt_flops)
       << ",\"tf32_tc_flops\":" << json::num(L.tf32_tc_flops) << ",\"bf16_tc_flops\":" << json::num(L.bf16_tc_flops)
       << "}";
  }
  os << "}";
  return os.str();
}

}  // namespace gb
