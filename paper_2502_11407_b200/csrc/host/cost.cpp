#include "cost.hpp"

#include <algorithm>
#include <cmath>
#include <sstream>

#include "error.hpp"
#include "json.hpp"
#include "tcplan.hpp"

namespace gb {

namespace {

inline void check_level(const Sched& s, int level) {
  if (level < 1 || level > s.L) throw Error(Code::LevelOutOfRange, "level " + std::to_string(level));
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

inline int64_t sum_tile_elems(const OpDesc& op, const Sched& s, int level) {
  int64_t tile[kMaxAxes];
  int64_t counts[kMaxTensors];
  s.tiles_at(op, level, tile);
  op.tile_elems(tile, counts);
  int64_t total = 0;
  for (int t = 0; t < op.ntensors; ++t) total += counts[t];
  return total;
}

}  // namespace

int64_t footprint_elems(const OpDesc& op, const Sched& s, int level) {
  check_level(s, level);
  return sum_tile_elems(op, s, level);
}

int64_t footprint_bytes(const OpDesc& op, const Sched& s, int level) {
  return sum_tile_elems(op, s, level) * op.dtype_bytes;
}

bool capacity_ok(const OpDesc& op, const HwModel& hw, const Sched& s, int level) {
  if (level < 0 || level >= hw.num_levels()) throw Error(Code::LevelOutOfRange, "level " + std::to_string(level));
  const MemLevel& m = hw.levels[static_cast<size_t>(level)];
  if (m.unlimited || level == 0) return true;
  return footprint_bytes(op, s, level) <= m.capacity_bytes;
}

int64_t traffic(const OpDesc& op, const Sched& s, int level) {
  check_level(s, level);
  int64_t tile[kMaxAxes];
  int64_t regions[kMaxTensors];
  s.tiles_at(op, level, tile);
  int64_t instances = 1;
  for (int a = 0; a < op.naxes; ++a) instances *= op.ax[a].padded / tile[a];
  op.tile_elems(tile, regions);
  int64_t q = 0;
  for (int t = 0; t < op.ntensors; ++t)
    q += op.t[t].output ? op.tensor_elems(t, /*padded=*/true) : instances * regions[t];
  return q;
}

// Eq. 1: Q(T) F(T') / (Q(T') F(T)).
double benefit_tiling(const OpDesc& op, const Sched& before, const Sched& after, int level) {
  const double qb = static_cast<double>(traffic(op, before, level));
  const double qa = static_cast<double>(traffic(op, after, level));
  const double fb = static_cast<double>(footprint_elems(op, before, level));
  const double fa = static_cast<double>(footprint_elems(op, after, level));
  return (qb * fa) / (qa * fb);
}

// Eq. 2: (L_low + S/B_low) / (L_high + S/B_high).
double caching_benefit(double lat_low, double bw_low, double lat_high, double bw_high, double s_bytes) {
  return (lat_low + s_bytes / bw_low) / (lat_high + s_bytes / bw_high);
}

double benefit_caching(const OpDesc& op, const HwModel& hw, const Sched& s, int from_level, int to_level) {
  if (to_level != from_level + 1 || from_level < 0 || to_level >= hw.num_levels())
    throw Error(Code::LevelOutOfRange, "cache step " + std::to_string(from_level) + "->" + std::to_string(to_level));
  const MemLevel& lo = hw.levels[static_cast<size_t>(from_level)];
  const MemLevel& hi = hw.levels[static_cast<size_t>(to_level)];
  const double bytes = static_cast<double>(footprint_bytes(op, s, to_level));
  return caching_benefit(lo.latency, lo.bandwidth, hi.latency, hi.bandwidth, bytes);
}

// Eq. 3: ceil(x/W) / ceil(x/(V W)).
double vthread_ratio(int64_t x, int64_t bank_width, int64_t v) {
  if (bank_width <= 0) return 1.0;
  return static_cast<double>(ceil_div(x, bank_width)) / static_cast<double>(ceil_div(x, v * bank_width));
}

double benefit_vthread(const OpDesc& op, const HwModel& hw, const Sched& s, int axis, int64_t v) {
  if (op.ax[axis].reduce) throw Error(Code::IllegalAction, "vthread benefit on reduce axis");
  const int banked = hw.banked_level();
  if (banked < 0) return 1.0;
  return vthread_ratio(s.tile(op, axis, banked), hw.levels[static_cast<size_t>(banked)].bank_width, v);
}

double utilization(const OpDesc& op, const HwModel& hw, const Sched& s) {
  const int banked = hw.banked_level();
  if (banked < 0) return 1.0;
  const int64_t w = hw.levels[static_cast<size_t>(banked)].bank_width;
  int64_t worst = 1;
  for (int a = 0; a < op.naxes; ++a) {
    if (op.ax[a].reduce) continue;
    worst = std::max(worst, ceil_div(s.tile(op, a, banked), s.vt(a) * w));
  }
  return std::clamp(1.0 / static_cast<double>(worst), 0.1, 1.0);
}

Cost estimate(const OpDesc& op, const HwModel& hw, const Sched& s) {
  if (!s.complete())
    throw Error(Code::IncompleteState, "cost needs a complete schedule, cur_mem_level=" + std::to_string(s.cur));
  Cost c;
  c.compute_seconds = static_cast<double>(op.flops_padded()) / hw.peak_flops / utilization(op, hw, s);
  c.est_seconds = c.compute_seconds;
  c.bottleneck = -1;
  auto channel = [&](int src, int64_t elems) {
    const double bytes = static_cast<double>(elems) * op.dtype_bytes;
    const double sec = bytes / (hw.levels[static_cast<size_t>(src)].bandwidth * hw.clock_hz);
    c.memory_seconds.push_back(sec);
    if (sec > c.est_seconds) {
      c.est_seconds = sec;
      c.bottleneck = src;
    }
  };
  if (s.L == 0) {
    int64_t total = 0;
    for (int t = 0; t < op.ntensors; ++t) total += op.tensor_elems(t, true);
    channel(0, total);
  } else {
    for (int l = 1; l <= s.L; ++l) channel(l - 1, traffic(op, s, l));
  }
  return c;
}

// B200 cost. The reference channels are kept; the compute channel changes:
//   * CTAs = prod over spatial axes of ceil(true extent / level-1 tile) (guarded tails skipped);
//   * threads/CTA = prod over spatial axes of level-1 / level-L tile;
//   * resident CTAs/SM from threads, registers (thread tile accumulators + operands) and smem
//     (level-1 footprint), each against the device limits;
//   * waves = ceil(CTAs / (SMs x resident)); the compute time is the ideal time divided by the
//     fraction of SM-slots the waves actually fill, and by the bank-conflict utilisation.
// The peak is the op's execution peak (fp32 SIMT for fp32 ops, bf16 TC for 2-byte ops).
Cost estimate_b200(const OpDesc& op, const HwModel& hw, const Sched& s) {
  Cost c = estimate(op, hw, s);
  const DeviceLimits& d = hw.dev;
  const ExecUnit unit = exec_unit(op);
  const double hbm_floor = op.bytes_true() / d.hbm_bytes_per_s;
  if (op.kind == Kind::Gemm && tensor_unit(unit)) {
    // the tensor-core program this state instantiates (UMMA tile, ring depth from the level-1 tile)
    const bool bf16 = unit == ExecUnit::TensorBf16;
    const GemmTcPlan p = gemm_tc_plan(op, s, bf16, false);
    const int64_t M = op.param("M"), N = op.param("N"), K = op.param("K");
    const double t = gemm_tc_seconds(d, M, N, K, op.batch, op.dtype_bytes, op.dtype_bytes, p,
                                     bf16 ? d.bf16_tc_flops : d.tf32_tc_flops);
    const double tiles = static_cast<double>(((M + p.BM - 1) / p.BM) * ((N + p.BN - 1) / p.BN) * op.batch);
    c.waves = std::ceil(tiles / (d.sms / p.cs * p.cs));
    c.occupancy = tiles / (c.waves * d.sms);
    c.compute_seconds = t;
    c.est_seconds = std::max(t, hbm_floor + kLaunchSeconds);
    c.bottleneck = t >= hbm_floor + kLaunchSeconds ? -1 : 0;
    c.exec_seconds = c.est_seconds;
    return c;
  }
  if (op.kind == Kind::Conv2d && tensor_unit(unit)) {
    const ConvFlatPlan p = conv_flat_plan_of(op, s);
    if (p.shape_ok) {  // the conv_flat program this state instantiates (filter groups, CTA pairs)
      const double t = conv_flat_seconds(op, d, p);
      const int64_t pos_tiles = op.param("N") * ((op.param("OH") * op.param("W") + 123) / 124);
      const double ctas = static_cast<double>(p.FG * std::min<int64_t>(pos_tiles, d.sms / p.FG));
      c.waves = std::ceil(static_cast<double>(p.FG * pos_tiles) / ctas);
      c.occupancy = ctas / d.sms;
      c.compute_seconds = t;
      c.est_seconds = std::max(t, hbm_floor + kLaunchSeconds);
      c.bottleneck = t >= hbm_floor + kLaunchSeconds ? -1 : 0;
      c.exec_seconds = c.est_seconds;
      return c;
    }
  }
  const int L = std::max(1, s.L);
  double ctas = static_cast<double>(op.batch);
  int64_t threads = 1, acc = 1;
  for (int a = 0; a < op.naxes; ++a) {
    if (op.ax[a].reduce) continue;
    const int64_t t1 = s.L ? s.tile(op, a, 1) : op.ax[a].padded;
    const int64_t tl = s.L ? s.tile(op, a, L) : 1;
    ctas *= static_cast<double>(ceil_div(op.ax[a].extent, t1));
    threads *= t1 / tl;
    acc *= tl;
  }
  const int64_t warps = ceil_div(threads, 32);
  int64_t by_threads = std::max<int64_t>(1, d.max_threads_per_sm / std::max<int64_t>(32, warps * 32));
  const int64_t regs_per_thread = std::min<int64_t>(d.max_regs_per_thread, 32 + 2 * acc);
  int64_t by_regs = std::max<int64_t>(1, d.regs_per_sm / std::max<int64_t>(1, regs_per_thread * warps * 32));
  int64_t smem = s.L ? footprint_bytes(op, s, 1) : 0;
  int64_t by_smem = smem > 0 ? std::max<int64_t>(1, d.smem_per_sm / smem) : d.max_blocks_per_sm;
  const int64_t resident = std::min<int64_t>({by_threads, by_regs, by_smem, d.max_blocks_per_sm});
  const double slots = static_cast<double>(d.sms) * static_cast<double>(resident);
  c.waves = std::ceil(ctas / slots);
  c.occupancy = ctas / (c.waves * slots);
  // warps actually issuing per SM vs the 4 schedulers x 4 warps needed to hide FMA latency
  const double warps_per_sm = std::min<double>(64.0, static_cast<double>(warps * resident) * c.occupancy);
  const double issue = std::min(1.0, warps_per_sm / 16.0);
  const double peak = op.dtype_bytes == 2 ? d.bf16_tc_flops : d.fp32_simt_flops;
  c.compute_seconds = op.flops_true() / peak / utilization(op, hw, s) / c.occupancy / issue;
  c.est_seconds = c.compute_seconds;
  c.bottleneck = -1;
  for (size_t i = 0; i < c.memory_seconds.size(); ++i)
    if (c.memory_seconds[i] > c.est_seconds) {
      c.est_seconds = c.memory_seconds[i];
      c.bottleneck = static_cast<int>(i);
    }
  // HBM floor on true bytes (every byte once), independent of tiling
  if (hbm_floor > c.est_seconds) {
    c.est_seconds = hbm_floor;
    c.bottleneck = 0;
  }
  // the family `auto` runs: tensor-core conv outside conv_flat's shapes (fixed-shape plans), the
  // HBM-streaming family (bandwidth-bound), or this SIMT estimate
  if (op.kind == Kind::Conv2d && tensor_unit(unit))
    c.exec_seconds = conv_tc_seconds(op, d);
  else if (unit == ExecUnit::Hbm) {
    // the HBM-streaming family (row / window ops): every byte once at the family's measured
    // fraction of the copy bandwidth, whatever the work-unit size the state picks
    // (est_seconds keeps the state's SIMT-style estimate: it ranks the states, which only pick
    // the work-unit size here, and is the program `simt_f32` would run)
    c.exec_seconds = hbm_floor / kStreamHbmEff + kLaunchSeconds;
  }
  else
    c.exec_seconds = c.est_seconds + kLaunchSeconds;
  return c;
}

std::string cost_json(const Cost& c, const HwModel& hw) {
  std::ostringstream os;
  os << "{\"est_seconds\":" << json::num(c.est_seconds) << ",\"compute_seconds\":" << json::num(c.compute_seconds)
     << ",\"memory_seconds\":[";
  for (size_t i = 0; i < c.memory_seconds.size(); ++i)
    os << (i ? "," : "") << "[" << json::quote(hw.levels[i].name) << "," << json::num(c.memory_seconds[i]) << "]";
  os << "],\"bottleneck\":"
     << json::quote(c.bottleneck < 0 ? std::string("compute") : hw.levels[static_cast<size_t>(c.bottleneck)].name);
  if (hw.is_b200)
    os << ",\"waves\":" << json::num(c.waves) << ",\"occupancy\":" << json::num(c.occupancy)
       << ",\"exec_seconds\":" << json::num(c.exec_seconds);
  os << "}";
  return os.str();
}

}  // namespace gb
