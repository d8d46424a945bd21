// Analytical cost model: per-level traffic Q and footprint F, the paper's three transition
// benefits (Eqs. 1-3), and the end-state cost estimate.
//
// In reference-compatible mode every function reproduces the reference's double arithmetic
// operation for operation (src/cost_model.cpp:21-211, hardware.cpp:117-130), which is what makes
// the construction walk bit-identical. The B200 mode adds, on top of the same terms, a
// wave-quantisation / occupancy factor and per-variant peaks (estimate_b200 below).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "hw.hpp"
#include "op.hpp"
#include "sched.hpp"

namespace gb {

struct Cost {
  double est_seconds = 0.0;
  double compute_seconds = 0.0;
  std::vector<double> memory_seconds;  // one per source level 0..L-1 (names from the hw model)
  int bottleneck = -1;                 // -1 = compute, else the source level index
  double waves = 0.0;                  // B200 mode only: CTA waves over the SMs
  double occupancy = 0.0;              // B200 mode only: fraction of the last wave's SM slots used
  double exec_seconds = 0.0;           // B200 mode only: predicted time of the `auto` kernel family
};

int64_t footprint_elems(const OpDesc& op, const Sched& s, int level);
int64_t footprint_bytes(const OpDesc& op, const Sched& s, int level);
bool capacity_ok(const OpDesc& op, const HwModel& hw, const Sched& s, int level);

// Q at `level`: inputs re-loaded once per level tile instance, output written once
// (cost_model.cpp:30-48). Padded scheduling domain.
int64_t traffic(const OpDesc& op, const Sched& s, int level);

double benefit_tiling(const OpDesc& op, const Sched& before, const Sched& after, int level);
double caching_benefit(double lat_low, double bw_low, double lat_high, double bw_high, double s_bytes);
double benefit_caching(const OpDesc& op, const HwModel& hw, const Sched& s, int from_level, int to_level);
double vthread_ratio(int64_t x, int64_t bank_width, int64_t v);
double benefit_vthread(const OpDesc& op, const HwModel& hw, const Sched& s, int axis, int64_t v);
double utilization(const OpDesc& op, const HwModel& hw, const Sched& s);

// Reference-compatible estimate (cost_model.cpp:179-211). Throws IncompleteState.
Cost estimate(const OpDesc& op, const HwModel& hw, const Sched& s);

// B200 estimate. GEMMs that run on the tensor cores are priced as the
// gemm_tc program the state instantiates (tcplan.hpp); other ops keep the reference terms with the
// compute channel scaled by wave quantisation, SM occupancy and the execution unit's peak.
// exec_seconds = the predicted time of the kernel family `auto` runs (the LPT weight).
Cost estimate_b200(const OpDesc& op, const HwModel& hw, const Sched& s);

std::string cost_json(const Cost& c, const HwModel& hw);

}  // namespace gb
