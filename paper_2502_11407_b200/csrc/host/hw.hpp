// Hardware model: the memory hierarchy and compute peaks that drive transition benefits and
// analytical cost.
//
// Reference-format documents load exactly as HardwareSpec::load does (hardware.cpp:10-70):
// level 0 is the farthest level and the only one allowed to be "unlimited", capacities strictly
// decrease inward, bandwidths strictly increase inward. Those documents drive the
// reference-compatible construction mode.
//
// The B200 model (HwModel::b200) is new: it is built from the live device query (SM count,
// shared memory per block, register file, L2 size, clocks) plus the driver-measured peaks, and
// carries the device limits that the B200 construction mode turns into legality gates and a
// wave/occupancy cost term.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "json.hpp"

namespace gb {

struct MemLevel {
  std::string name;
  bool unlimited = false;
  int64_t capacity_bytes = 0;
  double bandwidth = 0.0;     // bytes / cycle
  double latency = 0.0;       // cycles
  int64_t bank_width = 0;     // elements; 0 = unbanked
};

// Device limits consumed by the B200 construction mode and by kernel legalization.
struct DeviceLimits {
  int sms = 148;
  int64_t smem_per_block = 232448;   // 227 KB opt-in
  int64_t smem_per_sm = 233472;      // 228 KB
  int64_t regs_per_sm = 65536;
  int max_regs_per_thread = 255;
  int max_threads_per_block = 1024;
  int max_threads_per_sm = 2048;
  int max_blocks_per_sm = 32;
  int64_t l2_bytes = 126LL << 20;
  int64_t tmem_cols = 512;
  double sm_clock_hz = 1.965e9;
  double hbm_bytes_per_s = 6537e9;          // measured copy bandwidth
  double fp32_simt_flops = 74.4e12;         // 148 SM * 128 lanes * 2 * clock
  double tf32_tc_flops = 1.1e15;            // nominal dense; replaced by measurement when known
  double bf16_tc_flops = 1632.4e12;         // measured burst (MEASURED_PEAKS.json)
};

class HwModel {
 public:
  static HwModel load(const json::Value& doc);
  static HwModel load_text(const std::string& text);
  // B200 model from limits (device query + measured peaks); 3 levels: hbm3e, smem, regs.
  static HwModel b200(const DeviceLimits& lim);

  std::string name = "unnamed";
  std::vector<MemLevel> levels;
  double peak_flops = 1.0e12;
  double clock_hz = 1.0e9;
  int64_t max_threads_per_block = 1024;
  std::vector<int64_t> vthread_options{1, 2, 4, 8};

  bool is_b200 = false;  // set for the device model; enables the B200 construction gates
  DeviceLimits dev;

  int num_levels() const { return static_cast<int>(levels.size()); }
  int schedulable_levels() const { return static_cast<int>(levels.size()) - 1; }
  int banked_level() const;  // innermost level with bank_width > 0, or -1 (hardware.cpp:105-109)

  std::string to_json() const;
};

}  // namespace gb
