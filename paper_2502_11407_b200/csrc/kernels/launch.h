// Host-callable launchers of the kernel families (all asynchronous on the given stream).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include "flat_table.h"
#include <stddef.h>

#include "plan.h"

namespace gb::dev {

// Optional per-launch timing marks: when `ev` is non-null, ev[0] is recorded before the first
// launch and ev[i] after the i-th launch of the family, all on the launch stream.
struct Marks {
  cudaEvent_t* ev = nullptr;
  int next = 0;
  void mark(cudaStream_t st) {
    if (ev) cudaEventRecord(ev[next++], st);
  }
};

// ---- state-driven SIMT family (generic.cu) ----
int generic_max_width(bool f64);
void launch_generic(const GenericPlan& p, bool f64, bool bf16, const void* in0, const void* in1, void* out,
                    int batch, cudaStream_t st, const CUtensorMap* map = nullptr);

// ---- TMA tensor maps (gemm_tc.cu) ----
void encode_map(CUtensorMap* map, bool bf16, bool tf32, const void* ptr, int rank, const uint64_t* dims,
                const uint64_t* strides_bytes, const uint32_t* box, bool atom32 = false);
void encode_map_swizzle(CUtensorMap* map, bool bf16, bool tf32, const void* ptr, int rank, const uint64_t* dims,
                        const uint64_t* strides_bytes, const uint32_t* box, CUtensorMapSwizzle swizzle);

// ---- tensor-core GEMM family (gemm_tc.cu) ----
// The plan is immutable after prepare; tensor maps over the caller's buffers are built per
// (A, B, C) by gemm_tc_maps and passed to the launch (the kernel handle caches them).
struct GemmTcArgs {
  int M = 0, N = 0, K = 0, batch = 1, BN = 128;
  int stages = 4;  // smem ring depth (from the schedule's level-1 k tile)
  int cs = 1;      // cluster size along N (A multicast), 1 = no cluster
  int sms = 148;
  bool bf16 = false;
  bool a_shared = false;  // A is one matrix for every batch entry (1x1 conv: the filter bank)
  bool x3 = false;        // fp32-grade 3xTF32 (hi/lo operand split in the kernel), BN = 64
  bool pair = false;      // CTA pairs (cta_group::2): 256 x BN tiles, half of B staged per CTA
};
struct GemmTcMaps {
  CUtensorMap A, B, C, Am;  // Am: A slices for cluster multicast (box rows 128 / cs)
};
bool gemm_tc_supported(int M, int N, int K, int elem_bytes);
int gemm_tc_max_stages(int BN, bool bf16, bool x3 = false);
int gemm_tc_stages(const GemmTcArgs& a);
void gemm_tc_maps(const GemmTcArgs& a, const void* A, const void* B, void* C, GemmTcMaps& m);
void launch_gemm_tc(const GemmTcArgs& a, const GemmTcMaps& m, cudaStream_t st);

// ---- tensor-core implicit-GEMM conv2d family (conv_tc.cu) ----
// Workspace (caller- or per-stream-owned, conv_tc_ws_bytes): the converted filter bank W' and the
// NHWC copy of the input, both rewritten by the pre-pass launch of every execute.
struct ConvTcArgs {
  int N = 0, C = 0, H = 0, W = 0, F = 0, R = 0, S = 0, OH = 0, OW = 0;
  int sms = 148;
  bool bf16 = false;
  bool ns = false;   // conv_ns: filter columns folded into the UMMA N (4 x 32 position tiles)
  bool s2d = false;  // conv_ns over the space-to-depth form of a stride-2 conv (ResNet stem)
  size_t w_off = 0, x_off = 0, ws_bytes = 0;  // workspace layout: W' at w_off, X at x_off
};
struct ConvTcMaps {
  CUtensorMap W;  // over W' in the workspace
  CUtensorMap X;  // over the NHWC copy (conv_tc: dims permuted to (c, w, n, h))
  CUtensorMap O;  // conv_ns: the NCHW output as (w, h, f, n) for TMA stores
};
void conv_tc_maps(const ConvTcArgs& a, void* ws, void* O, ConvTcMaps& m);
// ---- general tensor-core implicit-GEMM conv2d reading NCHW in place (conv_gemm.cu) ----
struct ConvGemmArgs {
  int N = 0, C = 0, H = 0, W = 0, F = 0, R = 0, S = 0, stride = 1, OH = 0, OW = 0;
  int BN = 128;
  int packed = 0;  // few channels: the (s, c) pairs of a filter row form one K axis
  int sms = 148;
  size_t ws_bytes = 0;  // W'[r][s][f][Cp] (pre-pass launch of every execute)
};
void conv_gemm_map(const ConvGemmArgs& a, void* ws, CUtensorMap& mapW);
void launch_conv_gemm(const ConvGemmArgs& a, const CUtensorMap& mapW, const void* I, const void* K, void* O,
                      void* ws, cudaStream_t st, Marks& mk);

bool conv_tc_supported(int C, int F, int R, int S, int stride, bool bf16);
bool conv_tc_prepass_fits(int C, int W);
bool conv_ns_supported(int C, int F, int R, int S, int stride, bool bf16);
bool conv_s2d_supported(int C, int F, int R, int S, int stride, bool bf16);
size_t conv_tc_smem_need(int C, int F, int R, int S, bool bf16);
void launch_conv_tc(const ConvTcArgs& a, const ConvTcMaps& m, const void* I, const void* K, void* O, void* ws,
                    cudaStream_t st, Marks& mk);

// ---- flattened-plane stride-1 tf32 conv2d reading NCHW in place, one launch (conv_flat.cu) ----
struct ConvFlatArgs {
  int N = 0, C = 0, H = 0, W = 0, F = 0, R = 0, S = 0, OH = 0, OW = 0;
  int FN = 0;    // filter rows per tap slot: one filter group (F rounded up to 16, or the state's f tile)
  int FG = 1;    // filter groups (ceil(F / FN)): CTA b works on group b % FG with that group's bank
  int T = 0;     // taps R*S
  int nck = 0;   // 32-channel chunks
  int PW = 0;    // wide positions per image (OH * W)
  int tiles_img = 0, total = 0, stages = 0, sms = 148;
  int spec = -1; // compile-time-specialised MMA issue (3x3, FN 64: W mod 4), -1 = table-driven
  bool pair = false;  // cta_group::2 CTA pairs (flat_table pair mode: half the bank per CTA)
  int exp = 0;   // DEV build only (GENSOR_FLAT_EXP): 2048 table-driven issue, 8192 single CTAs, 65536 timeline marker
  size_t ws_bytes = 0;  // bank image W' (workspace), rewritten by every execute, + completion counter
  size_t sync_off = 0;  // counter of filter CTAs done (handle-owned workspaces)
  size_t grp_bytes = 0; // one filter group's bank image
  int filt_blocks = 0;  // CTAs of the bank-conversion launch
  FlatTable tb;         // taps, groups and the MMA op table for this W (flat_table.h)
};
// fn_req: filter group width (0 = all filters in one group), allow_pair: CTA pairs when legal
bool conv_flat_plan(int N, int C, int H, int W, int F, int R, int S, int stride, int sms, ConvFlatArgs& a,
                    int fn_req = 0, bool allow_pair = true);
void conv_flat_map(const ConvFlatArgs& a, const void* I, CUtensorMap& mapX);
void launch_conv_flat(const ConvFlatArgs& a, const CUtensorMap& mapX, const void* K, void* O, void* ws,
                      bool own_ws, cudaStream_t st, Marks& mk);

// ---- HBM-streaming family (stream.cu): gemv / softmax / avgpool2d / dwconv2d ----
enum class StreamKind : int { Gemv, Softmax, AvgPool, DwConv };
constexpr int kWinTH = 8, kWinTW = 2;  // window ops: outputs per thread (rows x cols)

// Window ops: a unit is a band of `band_rows` output rows of one (n, c) plane; its input rows
// [oh0*stride, oh0*stride + in_rows) are one contiguous range of the NCHW input.
struct StreamWinArgs {
  int64_t planes = 0;       // N * C
  int64_t C = 1, H = 0, W = 0, OH = 0, OW = 0;
  int32_t R = 1, S = 1, stride = 1, divisor = 0;  // divisor: F*F for avgpool, 0 for dwconv
  int32_t band_rows = 1, in_rows = 1;
  int64_t bands = 1, units = 0;
  int64_t buf_floats = 0;   // one staging buffer (phase slack included), floats
  int32_t threads = 256;
  int32_t sms = 148;
  int32_t vec = 0, vec_out = 0;  // set at launch from pointer alignment
  int32_t order_kind = 0;   // interpreter reduce order: 1 r-major, 2 s-major, 0 other (list below)
  int32_t n_order = 0;
  uint8_t order[64];        // (r << 4) | s in the interpreter's accumulation order
};

struct StreamArgs {
  StreamKind kind = StreamKind::Gemv;
  int64_t M = 0, N = 0;       // gemv / softmax rows x cols
  int64_t rows_per_unit = 1;  // gemv / softmax: rows per CTA work unit (level-1 m tile, split for balance)
  int32_t wpr = 1;            // gemv: warps per row (1, 2, 4, 8)
  int32_t sms = 148;
  StreamWinArgs win;
};
void launch_stream(const StreamArgs& a, const void* in0, const void* in1, void* out, cudaStream_t st);

}  // namespace gb::dev
