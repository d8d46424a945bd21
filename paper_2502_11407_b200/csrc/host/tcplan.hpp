// Tensor-core side of the B200 model: which execution unit `auto` lowers an op to, the gemm_tc
// plan a complete schedule instantiates, and the analytical time of that plan.
//
// The reference's cost model knows one peak and no parallelism (cost_model.cpp:179-211); on B200
// the dense contractions run on tcgen05 tensor cores, so the B200 construction mode prices a
// GEMM state as the tensor-core program it becomes:
//   level-1 m tile -> UMMA M (128 rows per CTA tile, cta_group::1),
//   level-1 n tile -> UMMA N = the CTA tile's width BN (TMEM: two accumulators of BN columns),
//   level-1 k tile -> the shared-memory ring depth in 128-byte k-blocks (the level-1 A and B
//                     boxes are what the ring holds; K-atom = 32 B, at least two k-blocks);
//   vthreads on n  -> CTAs of a thread-block cluster that work on adjacent n tiles and share
//                     one A tile by TMA multicast (Gensor's vThreads are cooperating units that
//                     split one tile; on B200 the units that share a tile are cluster CTAs);
// and gates the states no kernel can run (b200_feasible). Header-only: used by the host engine
// (g++) and by the kernel instantiation in exec.cu (nvcc), so both read the state the same way.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>

#include "../kernels/flat_table.h"
#include "hw.hpp"
#include "op.hpp"
#include "sched.hpp"

namespace gb {

enum class ExecUnit { TensorTf32, TensorBf16, Hbm, Simt };

// The unit `auto` runs an op on (gb::dev::resolve_variant without the device): fp32 GEMM / conv
// -> tf32 tensor cores, bf16 GEMM -> bf16 tensor cores, row / window ops -> the HBM-streaming
// family, everything else -> the SIMT family.
inline ExecUnit exec_unit(const OpDesc& op) {
  if (op.dtype_bytes != 2 && op.dtype_bytes != 4) return ExecUnit::Simt;
  switch (op.kind) {
    case Kind::Gemm:
      if ((op.param("K") * op.dtype_bytes) % 16 == 0 && (op.param("N") * op.dtype_bytes) % 16 == 0)
        return op.dtype_bytes == 2 ? ExecUnit::TensorBf16 : ExecUnit::TensorTf32;
      return ExecUnit::Simt;
    case Kind::Conv2d:
      return op.dtype_bytes == 4 ? ExecUnit::TensorTf32 : ExecUnit::Simt;
    case Kind::Gemv:
    case Kind::Softmax:
      return op.dtype_bytes == 4 && op.batch == 1 ? ExecUnit::Hbm : ExecUnit::Simt;
    case Kind::AvgPool2d:
    case Kind::DwConv2d:
      return op.dtype_bytes == 4 && op.batch == 1 && op.ax[4].extent <= 8 && op.ax[5].extent <= 8 ? ExecUnit::Hbm
                                                                                                   : ExecUnit::Simt;
  }
  return ExecUnit::Simt;
}

inline bool tensor_unit(ExecUnit u) { return u == ExecUnit::TensorTf32 || u == ExecUnit::TensorBf16; }

// Measured / structural constants of the tensor-core model:
constexpr double kTcL2BytesPerClkPerSm = 128.0;  // L2 -> SM TMA feed per SM
constexpr double kTcKBlockFloorClk = 256.0;      // measured per-k-block floor of gemm_tc at BN = 64 (~260 clk,
                                                 // round-1 trace), unchanged by A multicast (G: 14.3 us at
                                                 // cluster 1 and 4): barrier / TMA issue bound
constexpr double kTcStoreBytesPerClkPerSm = 64.0;
constexpr double kTcTmaLatencyClk = 1000.0;      // TMA box round trip + commit -> mbarrier
constexpr double kLaunchSeconds = 5.0e-6;        // fixed cost of one execute: an empty 148-CTA kernel timed by
                                                 // events after the bench's L2-flush write costs 5.1-5.9 us
                                                 // (tools/launch_cost.cu; 3.8 us back to back)
constexpr double kStreamHbmEff = 0.8;            // HBM-streaming family: measured 0.74-0.87 of the copy bandwidth
constexpr int kTcRingBytes = 227 * 1024 - 2048;  // opt-in smem minus barriers / alignment

struct GemmTcPlan {
  int BM = 128;
  int BN = 64;
  int stages = 4;
  int cs = 1;         // cluster size along N (A multicast)
  bool legal = true;  // the state is UMMA-shaped (b200_feasible's tensor-core gate)
};

inline int gemm_tc_bn_max(bool bf16, bool x3) { return x3 ? 64 : (bf16 ? 256 : 128); }

// Ring depth that fits next to the epilogue staging (4 warps x 32 rows x BN outputs).
inline int gemm_tc_ring_max(int BN, int es, bool x3) {
  const int stage = (128 * 128 + BN * 128) * (x3 ? 2 : 1);
  const int staging = 4 * 32 * BN * es;
  return std::min(8, (kTcRingBytes - staging) / stage);
}

// gemm_tc plan of a complete state (GEMM ops; batch is a grid dimension).
inline GemmTcPlan gemm_tc_plan(const OpDesc& op, const Sched& s, bool bf16, bool x3) {
  GemmTcPlan p;
  const int es = bf16 ? 2 : 4;
  const int64_t pm = op.ax[0].padded, pn = op.ax[1].padded;
  const int64_t tm = s.L ? s.tile(op, 0, 1) : pm, tn = s.L ? s.tile(op, 1, 1) : pn, tk = s.L ? s.tile(op, 2, 1) : 1;
  const int bn_max = gemm_tc_bn_max(bf16, x3);
  p.legal = tm == std::min<int64_t>(128, pm) && tn <= bn_max && tk * es >= 256;
  int bn = 64;
  while (bn < tn && bn < bn_max) bn *= 2;
  p.BN = x3 ? 64 : bn;
  const int ring = gemm_tc_ring_max(p.BN, es, x3);
  p.stages = static_cast<int>(std::clamp<int64_t>(tk * es / 128, 2, ring));
  const int64_t tiles_n = (op.param("N") + p.BN - 1) / p.BN;
  int cs = static_cast<int>(std::min<int64_t>(x3 ? 1 : 4, s.L ? s.vt(1) : 1));
  while (cs > 1 && tiles_n % cs) cs /= 2;
  p.cs = cs;
  (void)pn;
  return p;
}

// Tiles of a GEMM at N tile width bn (persistent grid of min(tiles, SMs) CTAs).
inline int64_t gemm_tc_tiles(const OpDesc& op, int64_t bn) {
  return ((op.param("M") + 127) / 128) * ((op.param("N") + bn - 1) / bn) * op.batch;
}

// Analytical time (s) of a gemm_tc plan: persistent CTAs over ceil(M/128) x ceil(N/BN) x batch
// tiles; a k-block costs the slowest of its MMAs (tensor peak per SM), its L2 -> smem feed and
// the TMA round trip spread over the ring's stages; the TMEM double buffer overlaps each tile's
// epilogue with the next tile's k-loop.
inline double gemm_tc_seconds(const DeviceLimits& d, int64_t M, int64_t N, int64_t K, int64_t batch, int es,
                              int es_out, const GemmTcPlan& p, double peak, int mmas_per_step = 1) {
  const double clk = d.sm_clock_hz;
  const int64_t tiles = ((M + p.BM - 1) / p.BM) * ((N + p.BN - 1) / p.BN) * batch;
  const double rounds = std::ceil(static_cast<double>(tiles) / d.sms);
  const int64_t nk = (K * es + 127) / 128;
  const double peak_sm = peak / d.sms;
  const double kb_elems = 128.0 / es;
  const double t_mma = mmas_per_step * 2.0 * p.BM * p.BN * kb_elems / peak_sm;
  const double t_feed = (static_cast<double>(p.BM) / p.cs + p.BN) * 128.0 / (kTcL2BytesPerClkPerSm * clk);
  const double t_lat = kTcTmaLatencyClk / p.stages / clk;
  const double t_kb = std::max({t_mma, t_feed, t_lat, kTcKBlockFloorClk / clk});
  const double t_tile = static_cast<double>(nk) * t_kb + kTcTmaLatencyClk / clk;
  const double t_epi = static_cast<double>(p.BM) * p.BN * es_out / (kTcStoreBytesPerClkPerSm * clk);
  return rounds * std::max(t_tile, t_epi) + std::min(t_tile, t_epi) + kLaunchSeconds;
}

// Time of the tensor-core conv families (implicit GEMM: M = output positions, N = F,
// K = C*R*S; the plans are fixed-shape, 128 positions x all filters per tile) plus the pre-pass
// that converts the filter bank and, for windows, the NCHW input.
inline double conv_tc_seconds(const OpDesc& op, const DeviceLimits& d) {
  const int64_t n = op.param("N"), f = op.param("F"), c = op.param("C");
  const int64_t r = op.param("R"), s = op.param("S"), oh = op.param("OH"), ow = op.param("OW");
  GemmTcPlan p;
  p.BN = 64;
  while (p.BN < f && p.BN < 256) p.BN *= 2;
  p.stages = 4;
  const double t = gemm_tc_seconds(d, n * oh * ow, f, c * r * s, 1, 4, 4, p, d.tf32_tc_flops);
  const double in_bytes = static_cast<double>(n * c * op.param("H") * op.param("W")) * 4;
  const double prepass = (r > 1 || s > 1) ? 2.0 * in_bytes / d.hbm_bytes_per_s + kLaunchSeconds : kLaunchSeconds;
  return t + prepass;
}

// ---- conv_flat (kernels/conv_flat.cu): the stride-1 conv over flattened NCHW planes ----------
// A complete state instantiates it as follows:
//   level-1 f tile      -> the filter group width FN (16 / 32 / 64 filters, at most F rounded to
//                          16): F splits into FG = ceil(F / FN) groups; each group is a set of
//                          CTAs with its own resident filter bank, UMMA N = taps x FN per offset
//                          group, and re-reads the input (from L2) once per group;
//   level-1 h x w tile  -> UMMA M: a tile of >= 256 output positions pairs two 128-position
//                          tiles on a CTA pair (cta_group::2, each CTA holds half of the bank)
//                          when the filters are one 64-wide group of a 3x3 window; smaller tiles
//                          run one 128-position tile per CTA.
struct ConvFlatPlan {
  bool shape_ok = false;  // stride 1, C % 32 == 0, F <= 64, 16 B plane pitch, not 1x1
  int FN = 64, FG = 1;
  bool pair = false;
};

inline bool conv_flat_shape(const OpDesc& op) {
  if (op.kind != Kind::Conv2d || op.dtype_bytes != 4 || op.batch != 1 || op.stride != 1) return false;
  const int64_t C = op.param("C"), F = op.param("F"), R = op.param("R"), S = op.param("S");
  const int64_t H = op.param("H"), W = op.param("W");
  return C % 32 == 0 && F >= 1 && F <= 64 && (H * W) % 4 == 0 && R * S <= dev::kFlatMaxTaps && R <= H && S <= W &&
         (R > 1 || S > 1);
}

inline ConvFlatPlan conv_flat_plan_of(const OpDesc& op, const Sched& s) {
  ConvFlatPlan p;
  p.shape_ok = conv_flat_shape(op);
  if (!p.shape_ok) return p;
  const int64_t F = op.param("F"), F16 = (F + 15) / 16 * 16;
  const int64_t tf = s.L ? std::min(s.tile(op, 1, 1), F) : F;
  const int64_t th = s.L ? std::min(s.tile(op, 2, 1), op.ax[2].extent) : op.ax[2].extent;
  const int64_t tw = s.L ? std::min(s.tile(op, 3, 1), op.ax[3].extent) : op.ax[3].extent;
  p.FN = static_cast<int>(std::min<int64_t>(F16, std::clamp<int64_t>((tf + 15) / 16 * 16, 16, 64)));
  p.FG = static_cast<int>((F + p.FN - 1) / p.FN);
  p.pair = p.FG == 1 && p.FN == 64 && op.param("R") == 3 && op.param("S") == 3 && op.param("W") >= 6 &&
           th * tw >= 256;
  // the resident bank (half of it per CTA of a pair) next to the input ring (4 stages single, 6
  // on pairs) and the epilogue records must fit the 227 KB of shared memory (conv_flat_plan)
  const int64_t bank = op.param("C") / 32 * op.param("R") * op.param("S") * p.FN * 128;
  auto fits = [&](bool pair) { return bank / (pair ? 2 : 1) + (pair ? 6 : 4) * 16384 + 12288 + 2048 <= 227 * 1024; };
  if (p.pair && !fits(true)) p.pair = false;
  p.shape_ok = fits(p.pair) && dev::flat_table(static_cast<int>(op.param("R")), static_cast<int>(op.param("S")),
                                               static_cast<int>(op.param("W")), p.FN, p.pair).ok;
  return p;
}

// Analytical time (s) of a conv_flat program. Per 128-position tile an SM's shared-memory
// datapath carries the A stages (TMA writes), the A operand reads of every UMMA k-step, the
// filter bank reads (halved on a CTA pair) and the epilogue's shuffles / records / stores; the
// tile costs the slower of that at 128 B / clk and the tensor work (measured 4.7 k
// vs 4.3 k modelled single-CTA, 3.5 k vs 3.7 k on pairs). Persistent CTAs: FG groups of
// min(tiles, SMs / FG) CTAs; the first UMMA starts ~5 k cycles after launch (bank image, TMEM,
// ring fill) and the last tile's epilogue trails the loop.
inline double conv_flat_seconds(const OpDesc& op, const DeviceLimits& d, const ConvFlatPlan& p) {
  const int R = static_cast<int>(op.param("R")), S = static_cast<int>(op.param("S"));
  const int W = static_cast<int>(op.param("W")), C = static_cast<int>(op.param("C"));
  const int64_t N = op.param("N"), OH = op.param("OH");
  const dev::FlatTable tb = dev::flat_table(R, S, W, p.FN, p.pair);
  const int nck = C / 32, T = R * S;
  int ops0 = 0, ops1 = 0;
  for (int g = 0; g < tb.ngroups; ++g) ops0 += tb.grp_nop[0][g], ops1 += tb.grp_nop[1][g];
  const double a_tma = static_cast<double>(tb.ngroups) * nck * 16384.0;
  const double a_rd = static_cast<double>(ops0 + (nck - 1) * ops1) * 4 * 4096.0;
  const double b_rd = static_cast<double>(nck) * T * p.FN * 128.0 / (p.pair ? 2 : 1);
  const double epi = 128.0 * p.FN * 4 * 4;
  const double smem_clk = (a_tma + a_rd + b_rd + epi) / kTcL2BytesPerClkPerSm;
  const double tensor_clk = 2.0 * 128 * T * p.FN * C / (d.tf32_tc_flops / d.sms / d.sm_clock_hz);
  const double t_tile = std::max(smem_clk, tensor_clk) / d.sm_clock_hz;
  const int64_t pos_tiles = N * ((OH * W + 123) / 124);
  const int64_t ctas_g = std::max<int64_t>(1, std::min<int64_t>(pos_tiles, d.sms / p.FG));
  const double rounds = std::ceil(static_cast<double>(pos_tiles) / static_cast<double>(ctas_g));
  return 5000.0 / d.sm_clock_hz + (rounds + 1) * t_tile + kLaunchSeconds;
}

}  // namespace gb
