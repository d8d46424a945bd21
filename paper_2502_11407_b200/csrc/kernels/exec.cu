// Execute step: instantiate a kernel family from a complete schedule and launch it.
// This is the device replacement of the SPEC's lower()+interpret().
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <sstream>
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <unordered_map>
#include <string>
#include <vector>

#include "../host/device.hpp"
#include "../host/error.hpp"
#include "../host/json.hpp"
#include "../host/lower.hpp"
#include "../host/tcplan.hpp"
#include "common.cuh"
#include "launch.h"

namespace gb::dev {

namespace {
std::atomic<uint64_t> g_launches{0};

const char* kVariantNames[] = {"simt_parity", "simt_f32", "tc_tf32", "tc_bf16", "stream", "tc_3xtf32"};
}  // namespace

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(Code::Cuda, std::string(what) + ": " + cudaGetErrorString(e));
}

void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

void set_smem_attr(const void* kern, size_t bytes, const char* what) {
  static std::mutex mu;
  static std::unordered_map<const void*, size_t> done;
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = done[kern];
  if (have >= bytes) return;
  check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)), what);
  have = bytes;
}
uint64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }


enum class Family { Generic, GemmTc, ConvTc, ConvGemm, ConvFlat, Stream };

// Tensor maps of one (inputs, output, workspace) pointer tuple. Encoding is pure host work, but
// at a few microseconds per execute it would show on the microsecond-scale ops, so the handle
// keeps the last few tuples (results never depend on the cache).
struct CallMaps {
  const void* key[4] = {nullptr, nullptr, nullptr, nullptr};
  bool valid = false;
  uint64_t used = 0;
  GemmTcMaps g;
  ConvTcMaps c;
  CUtensorMap w;
  CUtensorMap x;  // conv_flat: the caller's NCHW input as {H*W, N*C}; simt gemv (fast 3): A as {N, M}
};
constexpr int kMapCache = 4;

// Per-stream device workspace (pre-pass outputs of the conv families): two executes of one
// handle on different streams never share one.
struct WsSlot {
  cudaStream_t stream = nullptr;
  void* ptr = nullptr;
};

// An instantiated kernel. The plan fields are immutable after prepare(); execute() only touches
// the mutex-guarded caches (workspace slots, tensor maps), so one handle may be executed from
// several threads / streams at once (include/gensor_b200.h).
struct Kernel {
  OpDesc op;
  Sched state;
  int variant = 0;
  Family family = Family::Generic;
  GenericPlan gplan{};
  bool f64 = false;
  GemmTcArgs gemm;
  ConvTcArgs conv;
  ConvGemmArgs cgemm;
  ConvFlatArgs flat;
  StreamArgs stream;
  int launches = 1;
  std::vector<std::string> launch_names{"generic_simt"};
  std::string plan_info;
  size_t ws_bytes = 0;  // device workspace one execute needs (0: none)
  mutable std::mutex mu;
  mutable std::vector<WsSlot> ws_slots;
  mutable CallMaps maps[kMapCache];
  mutable uint64_t map_clock = 0;
  // per-launch timing instrumentation (gensor_kernel_set_timing): events recorded around each
  // internal launch of the executes issued while it is on; meant for one stream at a time
  mutable bool timing = false;
  mutable cudaEvent_t ev[8] = {};
  mutable int marks_used = 0;
  // host-buffer execute staging (gensor_execute_host takes a non-const handle: one call at a time)
  void* d_in[3] = {nullptr, nullptr, nullptr};
  void* d_out = nullptr;
  struct HostPipe* pipe = nullptr;  // chunked copy/compute overlap for execute_host (lazy)
};

// execute_host pipelining: the op is cut along an outer independent axis (conv/pool images,
// GEMM batch or rows, GEMV/softmax rows) into chunks; chunk c's H2D copy, chunk c-1's kernels and
// chunk c-2's D2H copy run concurrently on three streams (two copy engines + the SMs).
struct HostPipe {
  bool usable = false;
  int64_t extent = 0, q = 0;  // split extent, chunk size (the last chunk may be smaller)
  bool split[3] = {false, false, false};
  size_t unit_bytes[4] = {0, 0, 0, 0};  // bytes per split unit: inputs 0..2, output (index 3)
  Kernel* sub[2] = {nullptr, nullptr};  // kernels for chunk sizes q and the remainder
  cudaStream_t s_in = nullptr, s_out = nullptr;
  std::vector<cudaEvent_t> ev_in, ev_k;
  cudaEvent_t ev_shared = nullptr, ev_begin = nullptr;
};

namespace {

size_t tensor_bytes(const OpDesc& op, int t) {
  return static_cast<size_t>(op.tensor_elems(t, false)) * op.dtype_bytes * static_cast<size_t>(op.batch);
}

int64_t pow2_clamp(int64_t v, int64_t lo, int64_t hi) {
  int64_t p = lo;
  while (p < v && p < hi) p <<= 1;
  return p;
}

bool stream_ok(const OpDesc& op) {
  if (op.dtype_bytes != 4 || op.batch != 1) return false;
  switch (op.kind) {
    case Kind::Gemv:
    case Kind::Softmax:
      return true;
    case Kind::AvgPool2d:
    case Kind::DwConv2d:
      return op.ax[4].extent <= 8 && op.ax[5].extent <= 8;  // window axes (i,j / r,s)
    default:
      return false;
  }
}

// Reduce-iteration order of one output under the interpreter's loop nest (SPEC.md:470-478 /
// oracle_interpret): per level the reduce axes in axis order (radix T_{l-1}/T_l, step T_l), then
// the scalar reduce loops (radix T_L, step 1); guarded (padded) iterations are skipped.
void window_order(const OpDesc& op, const Sched& s, StreamWinArgs& w) {
  int ra = -1, sa = -1;
  for (int a = 0; a < op.naxes; ++a)
    if (op.ax[a].reduce) (ra < 0 ? ra : sa) = a;
  struct Loop {
    int axis;
    int64_t radix, step;
  };
  std::vector<Loop> loops;
  const int L = s.L;
  for (int l = 1; l <= L; ++l)
    for (int a : {ra, sa}) loops.push_back({a, s.tile(op, a, l - 1) / s.tile(op, a, l), s.tile(op, a, l)});
  for (int a : {ra, sa}) loops.push_back({a, L ? s.tile(op, a, L) : op.ax[a].padded, 1});
  std::vector<int64_t> dig(loops.size(), 0);
  w.n_order = 0;
  for (;;) {
    int64_t r = 0, c = 0;
    for (size_t q = 0; q < loops.size(); ++q) (loops[q].axis == ra ? r : c) += dig[q] * loops[q].step;
    if (r < w.R && c < w.S) w.order[w.n_order++] = static_cast<uint8_t>((r << 4) | c);
    int q = static_cast<int>(loops.size()) - 1;
    for (; q >= 0; --q) {
      if (++dig[static_cast<size_t>(q)] < loops[static_cast<size_t>(q)].radix) break;
      dig[static_cast<size_t>(q)] = 0;
    }
    if (q < 0) break;
  }
  bool rmajor = true, smajor = true;
  for (int q = 0; q < w.n_order; ++q) {
    const int r = w.order[q] >> 4, c = w.order[q] & 15;
    rmajor &= (r * w.S + c) == q;
    smajor &= (c * w.R + r) == q;
  }
  w.order_kind = rmajor ? 1 : (smajor ? 2 : 0);
}

// Stream plan from a complete schedule: the level-1 spatial tile is the CTA work unit.
StreamArgs lower_stream(const OpDesc& op, const Sched& s, int sms) {
  StreamArgs a;
  a.sms = sms;
  auto t1 = [&](int axis) { return s.L ? s.tile(op, axis, 1) : op.ax[axis].padded; };
  if (op.kind == Kind::Gemv || op.kind == Kind::Softmax) {
    a.kind = op.kind == Kind::Gemv ? StreamKind::Gemv : StreamKind::Softmax;
    a.M = op.ax[0].extent;
    a.N = op.ax[1].extent;
    // gemv: a row is split over wpr warps so each warp keeps 8 x 128-bit loads in flight per lane
    if (op.kind == Kind::Gemv) {
      a.wpr = 1;
      while (a.wpr < 8 && a.N / 4 >= static_cast<int64_t>(a.wpr) * 2 * 32 * 8) a.wpr *= 2;
    }
    // rows a CTA covers per step: gemv 8/wpr, short-row softmax (warp per row, N <= 1024) 8
    const int64_t step = op.kind == Kind::Gemv ? 8 / a.wpr : (a.N % 4 == 0 && a.N <= 1024 ? 8 : 1);
    // rows per unit: the level-1 m tile, halved while the grid would see fewer than 4 units per
    // resident CTA slot (8 x 256-thread CTAs per SM), so the persistent CTAs finish together
    int64_t rpu = std::max<int64_t>(step, t1(0));
    const int64_t slots = static_cast<int64_t>(sms) * 8;
    while (rpu > step && (a.M + rpu - 1) / rpu < 4 * slots) rpu = std::max<int64_t>(step, rpu / 2);
    a.rows_per_unit = std::min<int64_t>(std::max<int64_t>(1, a.M), rpu);
    return a;
  }
  a.kind = op.kind == Kind::AvgPool2d ? StreamKind::AvgPool : StreamKind::DwConv;
  StreamWinArgs& w = a.win;
  w.sms = sms;
  // axes n c h w + window axes (pool i j / dw r s), op_spec.cpp:184-193
  w.C = op.ax[1].extent;
  w.planes = op.ax[0].extent * w.C;
  w.H = op.param("H");
  w.W = op.param("W");
  w.OH = op.ax[2].extent;
  w.OW = op.ax[3].extent;
  w.R = static_cast<int32_t>(op.ax[4].extent);
  w.S = static_cast<int32_t>(op.ax[5].extent);
  w.stride = static_cast<int32_t>(op.stride);
  w.divisor = op.kind == Kind::AvgPool2d ? w.R * w.S : 0;
  window_order(op, s, w);
  // band: the level-1 h tile (output rows), cut so one staging buffer stays <= 24 KB (3 CTAs of
  // three buffers per SM) and rounded to the 4-row thread tile; among the legal band heights the
  // one that keeps the CTA's warps fullest is taken.
  const int h_axis = 2;
  const int64_t want = std::min<int64_t>(t1(h_axis), w.OH);
  const int64_t tiles_x = (w.OW + kWinTW - 1) / kWinTW;
  int64_t best = 1;
  double best_eff = -1.0;
  for (int64_t b = 1; b <= std::max<int64_t>(1, want); b = b < kWinTH ? b + 1 : b + kWinTH) {
    const int64_t rows = ((b + kWinTH - 1) / kWinTH * kWinTH - 1) * w.stride + w.R + 1;
    if ((rows * w.W + 8) * 4 > 24 * 1024 && b > 1) break;
    const int64_t tiles = tiles_x * ((b + kWinTH - 1) / kWinTH);
    const int64_t thr = std::min<int64_t>(256, (tiles + 31) / 32 * 32);
    const double rounds = std::ceil(static_cast<double>(tiles) / thr);
    const double eff = static_cast<double>(tiles) / (rounds * thr) + 1e-3 * static_cast<double>(b) / want;
    if (eff >= best_eff) {
      best_eff = eff;
      best = b;
    }
  }
  w.band_rows = static_cast<int32_t>(best);
  w.in_rows = static_cast<int32_t>((best - 1) * w.stride + w.R);
  w.bands = (w.OH + best - 1) / best;
  w.units = w.planes * w.bands;
  // staging buffer: the band's input rows plus slack so that partial edge tiles (rows rounded
  // up to the thread tile, columns past OW) read inside the buffer; those reads only feed
  // outputs that are never stored
  const int64_t rows_rd = ((best + kWinTH - 1) / kWinTH * kWinTH - 1) * w.stride + w.R + 1;
  w.buf_floats = (std::max<int64_t>(rows_rd, w.in_rows) * w.W + 4 + kWinTW * w.stride + 3) / 4 * 4;
  const int64_t tiles = tiles_x * ((best + kWinTH - 1) / kWinTH);
  w.threads = static_cast<int32_t>(std::min<int64_t>(256, (tiles + 31) / 32 * 32));
  return a;
}

bool gemm_tc_ok(const OpDesc& op, bool bf16) {
  if (op.kind != Kind::Gemm) return false;
  if (bf16 != (op.dtype_bytes == 2)) return false;  // operands are read in their stored dtype
  return gemm_tc_supported(static_cast<int>(op.param("M")), static_cast<int>(op.param("N")),
                           static_cast<int>(op.param("K")), op.dtype_bytes);
}

// conv_ns (tf32, stride 1, S <= 3, S*F <= 256): NCHW in place, filter columns folded into N
bool conv_ns_ok(const OpDesc& op, bool bf16) {
  if (op.kind != Kind::Conv2d || op.dtype_bytes != 4 || bf16) return false;
  if (dev_env("GENSOR_CONV_NS") && dev_env("GENSOR_CONV_NS")[0] == '0') return false;  // A/B
  return conv_ns_supported(static_cast<int>(op.param("C")), static_cast<int>(op.param("F")),
                           static_cast<int>(op.param("R")), static_cast<int>(op.param("S")),
                           static_cast<int>(op.stride), bf16) &&
         conv_tc_prepass_fits(static_cast<int>(op.param("C")), static_cast<int>(op.param("W")));
}

// stride-2 convs with few channels (ResNet stem): conv_ns over the space-to-depth form
bool conv_s2d_ok(const OpDesc& op, bool bf16) {
  if (op.kind != Kind::Conv2d || op.dtype_bytes != 4 || bf16) return false;
  if (dev_env("GENSOR_CONV_S2D") && dev_env("GENSOR_CONV_S2D")[0] == '0') return false;  // A/B
  return conv_s2d_supported(static_cast<int>(op.param("C")), static_cast<int>(op.param("F")),
                            static_cast<int>(op.param("R")), static_cast<int>(op.param("S")),
                            static_cast<int>(op.stride), bf16);
}

bool conv_tc_ok(const OpDesc& op, bool bf16) {
  if (op.kind != Kind::Conv2d || op.dtype_bytes != 4) return false;
  if (conv_s2d_ok(op, bf16)) return true;
  // conv_tc pays an NHWC pre-pass and wins through filter-row reuse: only for windows (R >= 2)
  if (op.param("R") < 2 && !bf16) return false;  // (bf16: conv_gemm has no bf16 path)
  if (conv_ns_ok(op, bf16)) return true;
  return conv_tc_supported(static_cast<int>(op.param("C")), static_cast<int>(op.param("F")),
                           static_cast<int>(op.param("R")), static_cast<int>(op.param("S")),
                           static_cast<int>(op.stride), bf16) &&
         conv_tc_prepass_fits(static_cast<int>(op.param("C")), static_cast<int>(op.param("W")));
}

// 1x1 stride-1 conv (tf32) as a batched GEMM with the filter bank shared by the batch:
// O[n] (F x P) = K (F x C) . I[n] (C x P) — the NCHW input is already the MN-major B operand and
// the NCHW output the row-major C, so no pre-pass and no im2col (TMA strides: C, P multiples of 4).
bool conv1x1_gemm_ok(const OpDesc& op, bool bf16) {
  if (op.kind != Kind::Conv2d || op.dtype_bytes != 4 || bf16 || op.stride != 1) return false;
  if (op.param("R") != 1 || op.param("S") != 1) return false;
  if (dev_env("GENSOR_CONV1X1_GEMM") && dev_env("GENSOR_CONV1X1_GEMM")[0] == '0') return false;  // A/B
  const int64_t P = op.param("H") * op.param("W");
  // per-image N tiles of 128 positions: small planes (14x14 -> 77 % of the tile used) stay with
  // conv_gemm, which flattens the positions of all images into M (measured on ResNet-50)
  if (P < 512 && P % 128 != 0) return false;
  return op.param("C") % 4 == 0 && P % 4 == 0 && gemm_tc_supported(static_cast<int>(op.param("F")), static_cast<int>(P),
                                                                     static_cast<int>(op.param("C")), 4);
}

// conv_flat (tf32, stride 1, C % 32 == 0, F <= 64, H*W % 4 == 0): flattened NCHW planes read in
// place by TMA (no NHWC copy); the bank conversion is a PDL-chained launch. With a state, its
// level-1 tiles choose the program (tcplan.hpp conv_flat_plan_of: filter groups, CTA pairs).
bool conv_flat_ok(const OpDesc& op, bool bf16, int sms, ConvFlatArgs* out, const Sched* s) {
  if (op.kind != Kind::Conv2d || op.dtype_bytes != 4 || bf16 || op.batch != 1) return false;
  if (dev_env("GENSOR_CONV_FLAT") && dev_env("GENSOR_CONV_FLAT")[0] == '0') return false;  // A/B
  int fn = 0;
  bool pair = true;
  if (s) {
    const ConvFlatPlan p = conv_flat_plan_of(op, *s);
    fn = p.FN;
    pair = p.pair;
  }
  ConvFlatArgs a;
  if (!conv_flat_plan(static_cast<int>(op.param("N")), static_cast<int>(op.param("C")),
                      static_cast<int>(op.param("H")), static_cast<int>(op.param("W")),
                      static_cast<int>(op.param("F")), static_cast<int>(op.param("R")),
                      static_cast<int>(op.param("S")), static_cast<int>(op.stride), sms, a, fn, pair))
    return false;
  if (a.R < 2 && a.S < 2) return false;  // 1x1: gemm_tc / conv_gemm
  if (out) *out = a;
  return true;
}

// General implicit-GEMM conv (tf32): any stride / window / channel count.
bool conv_gemm_ok(const OpDesc& op, bool bf16) { return op.kind == Kind::Conv2d && op.dtype_bytes == 4 && !bf16; }

int resolve_variant(const OpDesc& op, int variant) {
  if (variant != -1) return variant;
  if (op.kind == Kind::Gemm && op.dtype_bytes == 2 && gemm_tc_ok(op, true)) return 3;
  if (op.kind == Kind::Gemm && gemm_tc_ok(op, false)) return 2;
  if (op.kind == Kind::Conv2d && (conv_tc_ok(op, false) || conv_gemm_ok(op, false))) return 2;
  if (stream_ok(op)) return 4;
  return 1;
}

// simt_f32 fast paths (kernels/generic.cu k_simt_gemm / k_simt_gemv): the same plan — tiles,
// vthreads, ascending single-axis reduce — executed by register-tiled kernels when its shape fits
// their envelope (one round of thread slots, power-of-two thread tiles up to 8, shared memory).
void simt_fast_path(const OpDesc& op, GenericPlan& p, int64_t optin) {
  if (dev_env("GENSOR_SIMT_FAST") && dev_env("GENSOR_SIMT_FAST")[0] == '0') return;  // A/B
  auto tile_ok = [](int t) { return t == 1 || t == 2 || t == 4 || t == 8; };
  if (p.rounds != 1 || p.nred != 1) return;
  if (op.kind == Kind::Gemm && p.nsp == 2 && tile_ok(p.T[0]) && tile_ok(p.T[1])) {
    const int64_t bm = p.B[0], bn = p.B[1], bk = p.chunk_tile[0], pad = 0;  // A rows swizzled, no pad
    const int64_t smem = (bm * bk + bk * bn) * 4;
    if (smem > optin) return;
    p.fast = 1;
    p.fast_pad = static_cast<int32_t>(pad);
    p.smem_bytes = static_cast<int32_t>(smem);
  } else if (op.kind == Kind::Gemv && p.nsp == 1 && tile_ok(p.T[0]) && op.dtype_bytes == 4) {
    const int64_t n = p.ext[p.red[0]];
    // TMA path: every thread owns one row per row group (vthreads == thread tile), unit-stride
    // 16 B-aligned rows, at most 256 threads, x resident in shared memory
    const int64_t tma_smem = 1024 + 3LL * p.slots * 128 * 8 + n * 4;
    if (p.V[0] == p.T[0] && p.coef[0][p.red[0]] == 1 && (p.coef[0][p.sp[0]] & 3) == 0 && p.slots <= 256 &&
        p.slots % 8 == 0 && op.batch == 1 && tma_smem <= optin) {
      p.fast = 3;
      p.smem_bytes = static_cast<int32_t>(tma_smem);
      return;
    }
    p.fast = 2;
    p.fast_pad = n * 4 <= std::min<int64_t>(optin, 96 * 1024) ? 1 : 0;  // x staged in shared memory
    p.smem_bytes = p.fast_pad ? static_cast<int32_t>(n * 4) : 0;
  }
}

int current_device_sms(int* optin_smem) {
  int dev = 0, sms = 0, optin = 0;
  check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
  check_cuda(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "sm count");
  check_cuda(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev), "smem optin");
  if (optin_smem) *optin_smem = optin;
  return sms;
}

}  // namespace

DeviceLimits query(int device) {
  DeviceLimits lim;
  cudaDeviceProp prop;
  check_cuda(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
  lim.sms = prop.multiProcessorCount;
  lim.smem_per_block = static_cast<int64_t>(prop.sharedMemPerBlockOptin);
  lim.smem_per_sm = static_cast<int64_t>(prop.sharedMemPerMultiprocessor);
  lim.regs_per_sm = prop.regsPerMultiprocessor;
  lim.max_threads_per_block = prop.maxThreadsPerBlock;
  lim.max_threads_per_sm = prop.maxThreadsPerMultiProcessor;
  lim.max_blocks_per_sm = prop.maxBlocksPerMultiProcessor;
  lim.l2_bytes = prop.l2CacheSize;
  int clock_khz = 0;
  if (cudaDeviceGetAttribute(&clock_khz, cudaDevAttrClockRate, device) == cudaSuccess && clock_khz > 0)
    lim.sm_clock_hz = clock_khz * 1e3;
  lim.fp32_simt_flops = static_cast<double>(lim.sms) * 128.0 * 2.0 * lim.sm_clock_hz;
  return lim;
}

Kernel* prepare(const OpDesc& op, const Sched& s, int variant) {
  if (!s.complete()) throw Error(Code::IncompleteState, "kernel needs a complete schedule");
  // the kernels read fp32 (dtype_bytes 4) or bf16 (dtype_bytes 2) storage only
  if (op.dtype_bytes != 2 && op.dtype_bytes != 4)
    throw Error(Code::Unsupported, "dtype_bytes " + std::to_string(op.dtype_bytes) +
                                       " has no kernel: execute supports 4 (fp32) and 2 (bf16)");
  auto* k = new Kernel;
  k->op = op;
  k->state = s;
  k->variant = resolve_variant(op, variant);
  std::ostringstream pi;
  try {
    int optin = 0;
    const int sms = current_device_sms(&optin);
    switch (k->variant) {
      case 0:
      case 1: {
        k->f64 = k->variant == 0;
        k->family = Family::Generic;
        k->gplan = lower_generic(op, s, generic_max_width(k->f64), op.dtype_bytes, optin);
        if (!k->f64) simt_fast_path(op, k->gplan, optin);
        pi << plan_json(k->gplan);
        break;
      }
      case 2:
      case 3: {
        const bool bf16 = k->variant == 3;
        const bool conv1x1 = conv1x1_gemm_ok(op, bf16);
        if ((op.kind == Kind::Gemm && gemm_tc_ok(op, bf16)) || conv1x1) {
          k->family = Family::GemmTc;
          k->launch_names = {"gemm_tc"};
          GemmTcArgs& g = k->gemm;
          if (conv1x1) {  // O[n] = K . I[n]: M = F, N = H*W, K = C, batch = images, A shared
            g.M = static_cast<int>(op.param("F"));
            g.N = static_cast<int>(op.param("H") * op.param("W"));
            g.K = static_cast<int>(op.param("C"));
            g.batch = static_cast<int>(op.param("N"));
            g.a_shared = true;
          } else {
            g.M = static_cast<int>(op.param("M"));
            g.N = static_cast<int>(op.param("N"));
            g.K = static_cast<int>(op.param("K"));
            g.batch = static_cast<int>(op.batch);
          }
          g.bf16 = bf16;
          auto tiles = [&](int b) { return static_cast<int64_t>((g.M + 127) / 128) * ((g.N + b - 1) / b) * g.batch; };
          if (conv1x1) {
            // the filter bank is A (M = F): full-width 128-position N tiles, halved while SMs idle
            int bn = 128;
            while (bn > 64 && tiles(bn) < sms) bn /= 2;
            g.BN = bn;
            const int nkb = (g.K * op.dtype_bytes + 127) / 128;
            g.stages = std::min(gemm_tc_max_stages(bn, bf16), nkb > 8 ? 8 : nkb > 4 ? 6 : 4);
          } else {
            // the constructed state is the program (tcplan.hpp): UMMA N = the level-1 n tile,
            // ring depth = the level-1 k tile in 128-byte k-blocks
            const GemmTcPlan tp = gemm_tc_plan(op, s, bf16, false);
            g.BN = tp.BN;
            g.stages = tp.stages;
            g.cs = tp.cs;
          }
          if (const char* e = dev_env("GENSOR_GEMM_BN")) g.BN = std::atoi(e);
          if (const char* e = dev_env("GENSOR_GEMM_STAGES")) g.stages = std::atoi(e);
          const int bn = g.BN;
          g.sms = sms;
          // A multicast across a cluster of n-tiles: the state's n-axis vthreads (tcplan.hpp)
          if (const char* e = dev_env("GENSOR_GEMM_CLUSTER")) g.cs = std::atoi(e);
          const int tn = (g.N + bn - 1) / bn;
          while (g.cs > 1 && tn % g.cs) g.cs /= 2;
          // CTA pairs (cta_group::2, UMMA M = 256): when the tile has two 128-row halves and the B
          // tile splits into whole 128 B column chunks; a state asking for A multicast keeps it
          // (measured: GPT-2's GEMMs 4.23 -> 3.35 ms per step; at fewer pair tiles than SM pairs,
          // e.g. the 1024^3 GEMM, the single-CTA tiles fill more SMs and stay ahead)
          const char* pe = dev_env("GENSOR_GEMM_PAIR");  // developer A/B: '0' never, '1' whenever legal
          g.pair = g.cs == 1 && g.M >= 256 && (g.BN / 2) * op.dtype_bytes >= 128 &&
                   (static_cast<int64_t>((g.M + 255) / 256) * ((g.N + g.BN - 1) / g.BN) * g.batch >= sms / 2 ||
                    (pe && pe[0] == '1')) &&
                   !(pe && pe[0] == '0');
          pi << "{\"family\":\"gemm_tc\"" << (conv1x1 ? ",\"conv1x1\":\"O[n] = K . I[n], filter bank shared\"" : "")
             << ",\"BM\":" << (g.pair ? 256 : 128) << ",\"BN\":" << g.BN << ",\"BK_bytes\":128,\"stages\":"
             << gemm_tc_stages(g) << ",\"tiles\":" << (g.pair ? tiles(g.BN) / 2 : tiles(g.BN))
             << ",\"grid\":" << std::min<int64_t>(g.pair ? 2 * (tiles(g.BN) / 2) : tiles(g.BN), sms)
             << ",\"block\":192,\"persistent\":true,\"cluster_n\":" << g.cs
             << ",\"cta_pair\":" << (g.pair ? "true" : "false") << "}";
        } else if (op.kind == Kind::Conv2d && conv_flat_ok(op, bf16, sms, &k->flat, &s)) {
          k->family = Family::ConvFlat;
          k->launch_names = {"conv_flat"};
          const ConvFlatArgs& c = k->flat;
          k->launches = 2;  // bank conversion + conv (programmatic dependent launch), timed as one span
          k->ws_bytes = c.ws_bytes;
          pi << "{\"family\":\"conv_flat\",\"M_tile\":\"128 wide positions of one image (124 outputs)\",\"FN\":"
             << c.FN << ",\"filter_groups\":" << c.FG << ",\"tap_groups\":[";
          for (int g = 0; g < c.tb.ngroups; ++g) {
            pi << (g ? "," : "") << "{\"a\":" << (c.tb.group_o[g] & ~3) << ",\"umma\":[";
            for (int o = c.tb.grp_op0[1][g]; o < c.tb.grp_op0[1][g] + c.tb.grp_nop[1][g]; ++o)
              pi << (o > c.tb.grp_op0[1][g] ? "," : "") << "{\"b0\":" << c.tb.op_dcol[o] / c.FN << ",\"N\":" << c.tb.op_n[o]
                 << "}";
            pi << "]}";
          }
          pi << "],\"tiles\":" << c.FG * c.total << ",\"grid\":"
             << (c.pair ? 2 * std::min((c.total + 1) / 2, sms / 2) : c.FG * std::min(c.total, sms / c.FG))
             << ",\"stages\":" << c.stages
             << ",\"mma_issue\":\"" << (c.spec >= 0 ? "specialised (3x3, W mod 4)" : "table-driven")
             << "\",\"cta_pair\":" << (c.pair ? "true" : "false") << ",\"prezero\":" << c.tb.prezero
             << ",\"grid_note\":\"" << (c.pair ? "clusters of 2 CTAs, UMMA M = 256 (cta_group::2), half the bank per CTA" : "one CTA per tile stream")
             << "\",\"block\":576,\"launches\":2,\"A\":\"MN-major TMA boxes straight from the NCHW input\",\"B\":\"bank image converted by a PDL-chained launch, bulk-copied, resident\"}";
        } else if (op.kind == Kind::Conv2d && conv_tc_ok(op, bf16) &&
                   !(dev_env("GENSOR_CONV_FAMILY") && std::string(dev_env("GENSOR_CONV_FAMILY")) == "gemm" &&
                     !bf16)) {  // developer switch: A/B the two conv families on one shape
          k->family = Family::ConvTc;
          k->launches = 1;
          k->launch_names = {"conv_tc"};
          ConvTcArgs& c = k->conv;
          c.N = static_cast<int>(op.param("N"));
          c.C = static_cast<int>(op.param("C"));
          c.H = static_cast<int>(op.param("H"));
          c.W = static_cast<int>(op.param("W"));
          c.F = static_cast<int>(op.param("F"));
          c.R = static_cast<int>(op.param("R"));
          c.S = static_cast<int>(op.param("S"));
          c.OH = static_cast<int>(op.param("OH"));
          c.OW = static_cast<int>(op.param("OW"));
          c.bf16 = bf16;
          c.sms = sms;
          const size_t es = bf16 ? 2 : 4;
          size_t wb = static_cast<size_t>(c.R) * c.S * c.F * c.C * es;
          c.s2d = conv_s2d_ok(op, bf16);
          c.ns = c.s2d || conv_ns_ok(op, bf16);
          size_t xb = static_cast<size_t>(c.N) * c.H * c.W * c.C * es;
          if (c.s2d) {  // X2 [N][H/2][W/2][4C] and W2 [R/2][S/2][F][4C]
            xb = static_cast<size_t>(c.N) * ((c.H + 1) / 2) * ((c.W + 1) / 2) * 4 * c.C * es;
            wb = static_cast<size_t>((c.R + 1) / 2) * ((c.S + 1) / 2) * c.F * 4 * c.C * es;
          }
          c.w_off = 0;
          c.x_off = (wb + 255) & ~size_t(255);
          c.ws_bytes = c.x_off + xb;
          k->ws_bytes = c.ws_bytes;
          k->launches = 2;  // filter conversion + conv (programmatic dependent launch), timed as one span
          k->launch_names = {c.ns ? "conv_ns" : "conv_tc"};
          if (c.ns) {
            const int gs = c.s2d ? (c.S + 1) / 2 : c.S;
            const int tw = (c.OW + 32 - gs) / (33 - gs);
            const int vw = (c.OW + tw - 1) / tw;
            const int tiles = c.N * ((c.OH + 3) / 4) * tw;
            int fn = 32;
            while (fn < c.F) fn *= 2;
            pi << "{\"family\":\"conv_ns\"" << (c.s2d ? ",\"space_to_depth\":\"stride 2 -> stride 1 over 4C channels\"" : "")
               << ",\"M_tile\":\"4 rows x 32 input columns (" << vw
               << " outputs)\",\"UMMA_N\":" << gs * fn << ",\"tiles\":" << tiles << ",\"grid\":" << std::min(tiles, sms)
               << ",\"block\":320,\"launches\":2,\"A\":\"K-major TMA boxes from the NHWC pre-pass copy\",\"prepass\":\"NCHW->NHWC + K-major filters, PDL\"}";
          } else {
            const int tiles = ((c.N + 1) / 2) * ((c.OH + 7) / 8) * ((c.OW + 7) / 8);
            pi << "{\"family\":\"conv_tc\",\"M_tile\":\"8 rows x 2 images x 8 columns\",\"FN\":" << c.F
               << ",\"tiles\":" << tiles << ",\"grid\":" << std::min(tiles, sms)
               << ",\"block\":192,\"launches\":2,\"A\":\"K-major TMA boxes from the NHWC pre-pass copy\",\"prepass\":\"NCHW->NHWC + K-major filters, PDL\"}";
          }
        } else if (conv_gemm_ok(op, bf16)) {
          k->family = Family::ConvGemm;
          k->launches = 2;  // filter conversion + conv (programmatic dependent launch), one span
          k->launch_names = {"conv_gemm"};
          ConvGemmArgs& c = k->cgemm;
          c.N = static_cast<int>(op.param("N"));
          c.C = static_cast<int>(op.param("C"));
          c.H = static_cast<int>(op.param("H"));
          c.W = static_cast<int>(op.param("W"));
          c.F = static_cast<int>(op.param("F"));
          c.R = static_cast<int>(op.ax[5].extent);
          c.S = static_cast<int>(op.ax[6].extent);
          c.stride = static_cast<int>(op.stride);
          c.OH = static_cast<int>(op.ax[2].extent);
          c.OW = static_cast<int>(op.ax[3].extent);
          c.sms = sms;
          // N tile: the schedule's level-1 f tile widened to the UMMA N covering F (<= 256): the
          // A tile is produced once per N tile, so a wide N tile is what keeps the MMA fed
          int bn = static_cast<int>(pow2_clamp(std::max<int64_t>(s.L ? s.tile(op, 1, 1) : 128, c.F), 64, 256));
          while (bn > 64 && bn / 2 >= c.F) bn /= 2;
          c.BN = bn;
          c.packed = c.C * c.S <= 64 && c.C < 32;
          const int Cp = c.packed ? (c.S * c.C + 3) / 4 * 4 : (c.C + 3) / 4 * 4;
          const size_t planes = c.packed ? c.R : static_cast<size_t>(c.R) * c.S;
          c.ws_bytes = planes * c.F * Cp * 4;
          k->ws_bytes = c.ws_bytes;
          const int64_t P = static_cast<int64_t>(c.N) * c.OH * c.OW;
          const int64_t tiles = ((P + 127) / 128) * ((c.F + bn - 1) / bn);
          pi << "{\"family\":\"conv_gemm\",\"BM\":128,\"BN\":" << bn << ",\"tiles\":" << tiles
             << ",\"grid\":" << std::min<int64_t>(tiles, sms)
             << ",\"block\":416,\"launches\":2,\"packed_sc\":" << c.packed
             << ",\"A\":\"MN-major im2col from NCHW in place\"}";
        } else {
          throw Error(Code::Unsupported, std::string(kVariantNames[k->variant]) + " not available for " + op.label());
        }
        break;
      }
      case 5: {  // fp32-grade tensor-core GEMM: 3xTF32 operand split inside gemm_tc
        if (!(op.kind == Kind::Gemm && gemm_tc_ok(op, false)))
          throw Error(Code::Unsupported, std::string("tc_3xtf32 not available for ") + op.label());
        k->family = Family::GemmTc;
        k->launch_names = {"gemm_tc_3xtf32"};
        GemmTcArgs& g = k->gemm;
        g.M = static_cast<int>(op.param("M"));
        g.N = static_cast<int>(op.param("N"));
        g.K = static_cast<int>(op.param("K"));
        g.batch = static_cast<int>(op.batch);
        g.x3 = true;
        g.BN = 64;  // two operand copies per stage: the 64-wide N tile keeps 4 stages in smem
        g.sms = sms;
        g.stages = gemm_tc_max_stages(64, false, true);
        const int64_t tiles = static_cast<int64_t>((g.M + 127) / 128) * ((g.N + 63) / 64) * g.batch;
        pi << "{\"family\":\"gemm_tc\",\"split\":\"3xTF32: A_lo.B_hi + A_hi.B_lo + A_hi.B_hi\",\"BM\":128,\"BN\":64"
           << ",\"BK_bytes\":128,\"stages\":" << std::min(4, g.stages) << ",\"tiles\":" << tiles
           << ",\"grid\":" << std::min<int64_t>(tiles, sms) << ",\"block\":320,\"persistent\":true}";
        break;
      }
      case 4: {
        if (!stream_ok(op))
          throw Error(Code::Unsupported, std::string("stream not available for ") + op.label());
        k->family = Family::Stream;
        k->stream = lower_stream(op, s, sms);
        const StreamArgs& a = k->stream;
        static const char* names[] = {"gemv_stream", "softmax_stream", "avgpool_stream", "dwconv_stream"};
        k->launch_names = {names[static_cast<int>(a.kind)]};
        pi << "{\"family\":\"" << names[static_cast<int>(a.kind)] << "\"";
        if (a.kind == StreamKind::Gemv || a.kind == StreamKind::Softmax)
          pi << ",\"rows_per_unit\":" << a.rows_per_unit << ",\"warps_per_row\":" << a.wpr << ",\"units\":"
             << (a.M + a.rows_per_unit - 1) / a.rows_per_unit << ",\"block\":256,\"grid\":\"persistent\"";
        else
          pi << ",\"band_rows\":" << a.win.band_rows << ",\"in_rows\":" << a.win.in_rows << ",\"units\":"
             << a.win.units << ",\"block\":" << a.win.threads << ",\"thread_tile\":[" << kWinTH << "," << kWinTW << "],\"order_kind\":"
             << a.win.order_kind << ",\"smem_per_cta\":" << 3 * a.win.buf_floats * 4 << ",\"grid\":\"persistent\"";
        pi << "}";
        break;
      }
      default:
        throw Error(Code::Unsupported, "variant " + std::to_string(variant) + " not available for " + op.label());
    }
  } catch (...) {
    delete k;
    throw;
  }
  k->plan_info = pi.str();
  return k;
}

void destroy(Kernel* k) {
  if (!k) return;
  if (HostPipe* hp = k->pipe) {
    for (Kernel* sk : hp->sub) destroy(sk);
    for (cudaEvent_t e : hp->ev_in) cudaEventDestroy(e);
    for (cudaEvent_t e : hp->ev_k) cudaEventDestroy(e);
    if (hp->ev_shared) cudaEventDestroy(hp->ev_shared);
    if (hp->ev_begin) cudaEventDestroy(hp->ev_begin);
    if (hp->s_in) cudaStreamDestroy(hp->s_in);
    if (hp->s_out) cudaStreamDestroy(hp->s_out);
    delete hp;
  }
  for (void* p : k->d_in)
    if (p) cudaFree(p);
  if (k->d_out) cudaFree(k->d_out);
  for (const WsSlot& w : k->ws_slots)
    if (w.ptr) cudaFree(w.ptr);
  for (auto& e : k->ev)
    if (e) cudaEventDestroy(e);
  delete k;
}

std::string plan(const Kernel* k) { return k->plan_info; }

std::string info(const Kernel* k) {
  std::ostringstream os;
  os << "{\"variant\":" << k->variant << ",\"variant_name\":\"" << kVariantNames[k->variant]
     << "\",\"op\":" << k->op.to_json() << ",\"state\":" << k->state.to_json(k->op)
     << ",\"flops\":" << json::num(k->op.flops_true()) << ",\"bytes\":" << json::num(k->op.bytes_true())
     << ",\"launches\":" << k->launches << ",\"plan\":" << k->plan_info;
  if (k->pipe && k->pipe->usable)  // execute_host pipeline (set up by the first host-buffer execute)
    os << ",\"host_pipe\":{\"split_extent\":" << k->pipe->extent << ",\"chunk\":" << k->pipe->q
       << ",\"chunks\":" << k->pipe->ev_in.size() << "}";
  os << "}";
  return os.str();
}

size_t workspace_bytes(const Kernel* k) { return k->ws_bytes; }

namespace {

// The calling stream's workspace slot, allocated on the stream's first execute. A first execute
// inside a stream capture allocates in relaxed capture mode (the allocation is not captured).
void* stream_workspace(const Kernel* k, cudaStream_t st) {
  std::lock_guard<std::mutex> lock(k->mu);
  for (const WsSlot& w : k->ws_slots)
    if (w.stream == st) return w.ptr;
  cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
  check_cuda(cudaThreadExchangeStreamCaptureMode(&mode), "capture mode");
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, k->ws_bytes);
  if (e == cudaSuccess) e = cudaMemset(p, 0, k->ws_bytes);  // families keep completion counters in it
  cudaThreadExchangeStreamCaptureMode(&mode);
  check_cuda(e, "kernel workspace");
  k->ws_slots.push_back({st, p});
  return p;
}

// Tensor maps of this call's pointers (cached per pointer tuple).
void call_maps(const Kernel* k, const void* const* d_in, int n_in, void* d_out, void* ws, CallMaps& out) {
  const void* key[4] = {d_in[0], n_in > 1 ? d_in[1] : nullptr, d_out, ws};
  std::lock_guard<std::mutex> lock(k->mu);
  CallMaps* slot = &k->maps[0];
  for (CallMaps& m : k->maps) {
    if (m.valid && std::memcmp(m.key, key, sizeof key) == 0) {
      m.used = ++k->map_clock;
      out = m;
      return;
    }
    if (!m.valid || m.used < slot->used) slot = &m;
  }
  CallMaps fresh;
  std::memcpy(fresh.key, key, sizeof key);
  switch (k->family) {
    case Family::GemmTc:  // 1x1 conv: inputs are (I, K) but the GEMM is K . I
      if (k->gemm.a_shared)
        gemm_tc_maps(k->gemm, d_in[1], d_in[0], d_out, fresh.g);
      else
        gemm_tc_maps(k->gemm, d_in[0], d_in[1], d_out, fresh.g);
      break;
    case Family::ConvTc:
      conv_tc_maps(k->conv, ws, d_out, fresh.c);
      break;
    case Family::ConvGemm:
      conv_gemm_map(k->cgemm, ws, fresh.w);
      break;
    case Family::ConvFlat:
      conv_flat_map(k->flat, d_in[0], fresh.x);
      break;
    case Family::Generic:
      if (k->gplan.fast == 3) {  // simt gemv through TMA: A[M][N] row-major, box {32 columns, slots rows}
        const GenericPlan& p = k->gplan;
        const uint64_t dims[2] = {static_cast<uint64_t>(p.ext[p.red[0]]), static_cast<uint64_t>(p.ext[p.sp[0]])};
        const uint64_t strides[1] = {static_cast<uint64_t>(p.coef[0][p.sp[0]]) * 4};
        const uint32_t box[2] = {32, static_cast<uint32_t>(p.slots)};
        encode_map(&fresh.x, false, false, d_in[0], 2, dims, strides, box);
      }
      break;
    default:
      break;
  }
  fresh.valid = true;
  fresh.used = ++k->map_clock;
  *slot = fresh;
  out = fresh;
}

}  // namespace

void execute(const Kernel* k, const void* const* d_in, int n_in, void* d_out, void* ws, size_t ws_size,
             void* stream) {
  const OpDesc& op = k->op;
  if (n_in != op.input_count())
    throw Error(Code::ShapeMismatch,
                "expected " + std::to_string(op.input_count()) + " inputs, got " + std::to_string(n_in));
  for (int i = 0; i < n_in; ++i)
    if (!d_in[i]) throw Error(Code::ShapeMismatch, "null input pointer");
  auto st = static_cast<cudaStream_t>(stream);
  const bool own_ws = !ws;
  if (k->ws_bytes) {
    if (!ws)
      ws = stream_workspace(k, st);
    else if (ws_size < k->ws_bytes)
      throw Error(Code::ShapeMismatch, "workspace of " + std::to_string(ws_size) + " bytes, the kernel needs " +
                                     std::to_string(k->ws_bytes));
  }
  Marks mk;
  if (k->timing) mk.ev = k->ev;
  switch (k->family) {
    case Family::Generic: {
      const CUtensorMap* gm = nullptr;
      CallMaps m;
      if (k->gplan.fast == 3) {
        call_maps(k, d_in, n_in, d_out, ws, m);
        gm = &m.x;
      }
      mk.mark(st);
      launch_generic(k->gplan, k->f64, op.dtype_bytes == 2, d_in[0], n_in > 1 ? d_in[1] : nullptr, d_out,
                     static_cast<int>(op.batch), st, gm);
      mk.mark(st);
      break;
    }
    case Family::GemmTc: {
      CallMaps m;
      call_maps(k, d_in, n_in, d_out, ws, m);
      mk.mark(st);
      launch_gemm_tc(k->gemm, m.g, st);
      mk.mark(st);
      break;
    }
    case Family::ConvTc: {
      CallMaps m;
      call_maps(k, d_in, n_in, d_out, ws, m);
      launch_conv_tc(k->conv, m.c, d_in[0], d_in[1], d_out, ws, st, mk);
      break;
    }
    case Family::ConvGemm: {
      CallMaps m;
      call_maps(k, d_in, n_in, d_out, ws, m);
      launch_conv_gemm(k->cgemm, m.w, d_in[0], d_in[1], d_out, ws, st, mk);
      break;
    }
    case Family::ConvFlat: {
      CallMaps m;
      call_maps(k, d_in, n_in, d_out, ws, m);
      launch_conv_flat(k->flat, m.x, d_in[1], d_out, ws, own_ws, st, mk);
      break;
    }
    case Family::Stream:
      mk.mark(st);
      launch_stream(k->stream, d_in[0], n_in > 1 ? d_in[1] : nullptr, d_out, st);
      mk.mark(st);
      break;
  }
  if (k->timing) k->marks_used = mk.next;
}

// Median device time (ms) of `iters` executes, CUDA events on `stream` around each one (after one
// untimed warm-up execute). Used by the on-device re-ranking of the top-k schedules.
float time_execute(Kernel* k, const void* const* d_in, int n_in, void* d_out, void* stream, int iters) {
  auto st = static_cast<cudaStream_t>(stream);
  execute(k, d_in, n_in, d_out, nullptr, 0, stream);
  cudaEvent_t a, b;
  check_cuda(cudaEventCreate(&a), "cudaEventCreate");
  check_cuda(cudaEventCreate(&b), "cudaEventCreate");
  std::vector<float> ms;
  for (int i = 0; i < std::max(1, iters); ++i) {
    check_cuda(cudaEventRecord(a, st), "cudaEventRecord");
    execute(k, d_in, n_in, d_out, nullptr, 0, stream);
    check_cuda(cudaEventRecord(b, st), "cudaEventRecord");
    check_cuda(cudaEventSynchronize(b), "cudaEventSynchronize");
    float t = 0.f;
    check_cuda(cudaEventElapsedTime(&t, a, b), "cudaEventElapsedTime");
    ms.push_back(t);
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  std::sort(ms.begin(), ms.end());
  return ms[ms.size() / 2];
}

void set_timing(Kernel* k, bool on) {
  if (on && !k->ev[0])
    for (auto& e : k->ev) check_cuda(cudaEventCreate(&e), "cudaEventCreate");
  k->timing = on;
}

std::vector<std::pair<std::string, float>> timings(Kernel* k) {
  std::vector<std::pair<std::string, float>> out;
  if (!k->timing || k->marks_used < 2) return out;
  check_cuda(cudaEventSynchronize(k->ev[k->marks_used - 1]), "cudaEventSynchronize");
  for (int i = 1; i < k->marks_used; ++i) {
    float ms = 0.f;
    check_cuda(cudaEventElapsedTime(&ms, k->ev[i - 1], k->ev[i]), "cudaEventElapsedTime");
    const size_t j = static_cast<size_t>(i - 1);
    out.emplace_back(j < k->launch_names.size() ? k->launch_names[j] : "launch", ms);
  }
  return out;
}

namespace {

// The op with its split extent replaced (same JSON form as OpDesc::to_json).
std::string chunk_json(const OpDesc& op, int64_t n) {
  std::ostringstream os;
  auto p = [&](const char* name) { return op.param(name); };
  os << "{\"kind\":\"" << kind_name(op.kind) << "\"";
  switch (op.kind) {
    case Kind::Gemm:
      if (op.batch > 1)
        os << ",\"M\":" << p("M") << ",\"K\":" << p("K") << ",\"N\":" << p("N") << ",\"batch\":" << n;
      else
        os << ",\"M\":" << n << ",\"K\":" << p("K") << ",\"N\":" << p("N");
      break;
    case Kind::Gemv:
    case Kind::Softmax:
      os << ",\"M\":" << n << ",\"N\":" << p("N");
      break;
    case Kind::Conv2d:
      os << ",\"I\":[" << n << "," << p("C") << "," << p("H") << "," << p("W") << "],\"K\":[" << p("F") << ","
         << p("C") << "," << p("R") << "," << p("S") << "],\"S\":" << op.stride;
      break;
    case Kind::DwConv2d:
      os << ",\"I\":[" << n << "," << p("C") << "," << p("H") << "," << p("W") << "],\"K\":[" << p("C") << ",1,"
         << p("R") << "," << p("S") << "],\"S\":" << op.stride;
      break;
    case Kind::AvgPool2d:
      os << ",\"I\":[" << n << "," << p("C") << "," << p("H") << "," << p("W") << "],\"F\":" << p("F")
         << ",\"S\":" << op.stride;
      break;
  }
  os << ",\"dtype_bytes\":" << op.dtype_bytes << "}";
  return os.str();
}

// The state's tiles clamped to the chunk's padded extents: a complete state of the chunk op with
// the same reduce-axis walk (only the split spatial axis shrinks).
Sched clamp_state(const Sched& s, const OpDesc& op) {
  Sched c = s;
  for (int a = 0; a < op.naxes; ++a) {
    for (int l = 0; l < c.L; ++l) c.tiles[a][l] = std::min(c.tiles[a][l], op.ax[a].padded);
    if (c.L > 0) c.vts[a] = std::min(c.vts[a], c.tiles[a][c.L - 1]);
  }
  return c;
}

void plan_pipe(Kernel* k) {
  auto* hp = new HostPipe;
  k->pipe = hp;
  const OpDesc& op = k->op;
  const int nin = op.input_count();
  size_t total = 0;
  for (int t = 0; t <= nin; ++t) total += tensor_bytes(op, t);
  const bool off = dev_env("GENSOR_HOST_PIPE") && dev_env("GENSOR_HOST_PIPE")[0] == '0';
  if (off || total < (size_t(8) << 20)) return;  // small ops: one copy, one launch, one copy
  switch (op.kind) {
    case Kind::Gemm:
      hp->extent = op.batch > 1 ? op.batch : op.param("M");
      hp->split[0] = true;
      hp->split[1] = op.batch > 1;
      break;
    case Kind::Gemv:
    case Kind::Softmax:
      hp->extent = op.param("M");
      hp->split[0] = true;
      break;
    case Kind::Conv2d:
    case Kind::DwConv2d:
    case Kind::AvgPool2d:
      hp->extent = op.param("N");
      hp->split[0] = true;
      break;
  }
  if (hp->extent < 2) return;
  // chunks of ~8 MB of traffic (measured: PCIe reaches full duplex only for multi-MB copies; on
  // configs[1]'s 26.7 MB, 3 chunks 0.455 ms, 2 chunks 0.47, 4 chunks 0.465), <= 16
  const int chunk_mb = dev_env("GENSOR_HOST_PIPE_MB") ? std::atoi(dev_env("GENSOR_HOST_PIPE_MB")) : 8;
  int64_t chunks = std::min<int64_t>({hp->extent, 16, static_cast<int64_t>(total / (size_t(std::max(1, chunk_mb)) << 20))});
  if (chunks < 2) return;
  hp->q = (hp->extent + chunks - 1) / chunks;
  if (op.kind == Kind::Gemm && op.batch == 1) hp->q = (hp->q + 127) / 128 * 128;  // whole 128-row M tiles
  if (hp->q >= hp->extent) return;
  for (int t = 0; t <= nin; ++t) {
    const bool sp = t == nin || hp->split[t];
    hp->unit_bytes[t == nin ? 3 : t] = sp ? tensor_bytes(op, t) / static_cast<size_t>(hp->extent) : 0;
  }
  const int64_t rem = hp->extent % hp->q;
  for (int i = 0; i < (rem ? 2 : 1); ++i) {
    const OpDesc cop = OpDesc::parse_text(chunk_json(op, i == 0 ? hp->q : rem));
    hp->sub[i] = prepare(cop, clamp_state(k->state, cop), k->variant);
  }
  check_cuda(cudaStreamCreateWithFlags(&hp->s_in, cudaStreamNonBlocking), "pipe stream");
  check_cuda(cudaStreamCreateWithFlags(&hp->s_out, cudaStreamNonBlocking), "pipe stream");
  const int64_t n = (hp->extent + hp->q - 1) / hp->q;
  hp->ev_in.resize(static_cast<size_t>(n));
  hp->ev_k.resize(static_cast<size_t>(n));
  for (int64_t c = 0; c < n; ++c) {
    check_cuda(cudaEventCreateWithFlags(&hp->ev_in[static_cast<size_t>(c)], cudaEventDisableTiming), "pipe event");
    check_cuda(cudaEventCreateWithFlags(&hp->ev_k[static_cast<size_t>(c)], cudaEventDisableTiming), "pipe event");
  }
  check_cuda(cudaEventCreateWithFlags(&hp->ev_shared, cudaEventDisableTiming), "pipe event");
  check_cuda(cudaEventCreateWithFlags(&hp->ev_begin, cudaEventDisableTiming), "pipe event");
  hp->usable = true;
}

}  // namespace

void execute_host(Kernel* k, const void* const* h_in, int n_in, void* h_out, void* stream) {
  const OpDesc& op = k->op;
  if (n_in != op.input_count())
    throw Error(Code::ShapeMismatch,
                "expected " + std::to_string(op.input_count()) + " inputs, got " + std::to_string(n_in));
  auto st = static_cast<cudaStream_t>(stream);
  if (!k->pipe) {
    try {
      plan_pipe(k);
    } catch (const Error& e) {  // a chunk shape the family cannot run: keep the one-shot path
      if (dev_env("GENSOR_HOST_PIPE_DEBUG")) std::fprintf(stderr, "host pipe disabled: %s\n", e.what());
      if (k->pipe) {
        for (Kernel*& sk : k->pipe->sub) {
          destroy(sk);
          sk = nullptr;
        }
        k->pipe->usable = false;
      }
    }
  }
  if (k->pipe && k->pipe->usable) {
    HostPipe& hp = *k->pipe;
    for (int i = 0; i < n_in; ++i)
      if (!k->d_in[i]) check_cuda(cudaMalloc(&k->d_in[i], tensor_bytes(op, i)), "cudaMalloc input staging");
    if (!k->d_out) check_cuda(cudaMalloc(&k->d_out, tensor_bytes(op, op.output_index())), "cudaMalloc output staging");
    const bool dbg = dev_env("GENSOR_HOST_PIPE_DEBUG") != nullptr;
    std::vector<cudaEvent_t> dev_t(dbg ? 3 * hp.ev_in.size() : 0);
    cudaEvent_t dev_t0 = nullptr;
    if (dbg) {
      for (auto& e : dev_t) cudaEventCreate(&e);
      cudaEventCreate(&dev_t0);
      cudaEventRecord(dev_t0, st);
    }
    // order after prior work on the caller's stream, then the unsplit (shared) inputs
    check_cuda(cudaEventRecord(hp.ev_begin, st), "pipe event");
    check_cuda(cudaStreamWaitEvent(hp.s_in, hp.ev_begin, 0), "pipe wait");
    check_cuda(cudaStreamWaitEvent(hp.s_out, hp.ev_begin, 0), "pipe wait");
    for (int i = 0; i < n_in; ++i)
      if (!hp.split[i])
        check_cuda(cudaMemcpyAsync(k->d_in[i], h_in[i], tensor_bytes(op, i), cudaMemcpyHostToDevice, hp.s_in), "H2D");
    check_cuda(cudaEventRecord(hp.ev_shared, hp.s_in), "pipe event");
    check_cuda(cudaStreamWaitEvent(st, hp.ev_shared, 0), "pipe wait");
    const int64_t n = static_cast<int64_t>(hp.ev_in.size());
    for (int64_t c = 0; c < n; ++c) {
      const int64_t u0 = c * hp.q, cnt = std::min(hp.q, hp.extent - u0);
      Kernel* sk = hp.sub[cnt == hp.q ? 0 : 1];
      const void* din[3] = {nullptr, nullptr, nullptr};
      for (int i = 0; i < n_in; ++i) {
        if (hp.split[i]) {
          const size_t off = static_cast<size_t>(u0) * hp.unit_bytes[i], b = static_cast<size_t>(cnt) * hp.unit_bytes[i];
          check_cuda(cudaMemcpyAsync(static_cast<char*>(k->d_in[i]) + off, static_cast<const char*>(h_in[i]) + off, b,
                                     cudaMemcpyHostToDevice, hp.s_in),
                     "H2D chunk");
          din[i] = static_cast<char*>(k->d_in[i]) + off;
        } else {
          din[i] = k->d_in[i];
        }
      }
      check_cuda(cudaEventRecord(hp.ev_in[static_cast<size_t>(c)], hp.s_in), "pipe event");
      if (dbg) cudaEventRecord(dev_t[3 * c], hp.s_in);
      check_cuda(cudaStreamWaitEvent(st, hp.ev_in[static_cast<size_t>(c)], 0), "pipe wait");
      const size_t ooff = static_cast<size_t>(u0) * hp.unit_bytes[3], ob = static_cast<size_t>(cnt) * hp.unit_bytes[3];
      execute(sk, din, n_in, static_cast<char*>(k->d_out) + ooff, nullptr, 0, st);
      check_cuda(cudaEventRecord(hp.ev_k[static_cast<size_t>(c)], st), "pipe event");
      if (dbg) cudaEventRecord(dev_t[3 * c + 1], st);
      check_cuda(cudaStreamWaitEvent(hp.s_out, hp.ev_k[static_cast<size_t>(c)], 0), "pipe wait");
      check_cuda(cudaMemcpyAsync(static_cast<char*>(h_out) + ooff, static_cast<char*>(k->d_out) + ooff, ob,
                                 cudaMemcpyDeviceToHost, hp.s_out),
                 "D2H chunk");
      if (dbg) cudaEventRecord(dev_t[3 * c + 2], hp.s_out);
    }
    check_cuda(cudaStreamSynchronize(hp.s_out), "stream sync");
    check_cuda(cudaStreamSynchronize(st), "stream sync");
    if (dbg) {  // developer timeline: per chunk H2D done / kernels done / D2H done (us from begin)
      for (int64_t c = 0; c < n; ++c) {
        float t[3];
        for (int j = 0; j < 3; ++j) cudaEventElapsedTime(&t[j], dev_t0, dev_t[3 * c + j]);
        std::fprintf(stderr, "chunk %lld: h2d %.1f  kernel %.1f  d2h %.1f\n", static_cast<long long>(c), t[0] * 1e3,
                     t[1] * 1e3, t[2] * 1e3);
      }
      for (auto e : dev_t) cudaEventDestroy(e);
      cudaEventDestroy(dev_t0);
    }
    return;
  }
  for (int i = 0; i < n_in; ++i) {
    const size_t b = tensor_bytes(op, i);
    if (!k->d_in[i]) check_cuda(cudaMalloc(&k->d_in[i], b), "cudaMalloc input staging");
    check_cuda(cudaMemcpyAsync(k->d_in[i], h_in[i], b, cudaMemcpyHostToDevice, st), "H2D");
  }
  const size_t ob = tensor_bytes(op, op.output_index());
  if (!k->d_out) check_cuda(cudaMalloc(&k->d_out, ob), "cudaMalloc output staging");
  execute(k, k->d_in, n_in, k->d_out, nullptr, 0, stream);
  check_cuda(cudaMemcpyAsync(h_out, k->d_out, ob, cudaMemcpyDeviceToHost, st), "D2H");
  check_cuda(cudaStreamSynchronize(st), "stream sync");
}

}  // namespace gb::dev
