// Tensor-core implicit-GEMM conv2d families, instantiated from a constructed conv2d schedule:
//   O[n][f][h][w] = sum_{c,r,s} I[n][c][h*S+r][w*S+s] * K[f][c][r][s]   (op_spec.cpp:177-181)
// GEMM view: M = output positions, N = f, K = (r, s, c). Reference layouts in and out.
//
// conv_ns (the configs[1] headline; stride 1, S <= 4, S*F <= 256):
//   * launch 1 (pre-pass): NCHW -> NHWC copy of the input (2-row bands) and the K-major filter
//     bank W'[r][s][f][c]; it triggers the conv grid early (programmatic dependent launch);
//   * the filter columns s are folded into the UMMA N (N = S*F): one MMA multiplies each staged
//     input position by all S columns at full tensor-core rate, and the epilogue adds TMEM block
//     s of lane w + s into output w with warp shuffles — no s-shifted copies of A;
//   * tile = 4 output rows x 32 input columns of one image; one TMA box {32 channels, 32 columns,
//     4 + R - 1 rows} per 32-channel chunk (128 B swizzle); a filter-row shift r is +4 KB;
//   * 8 epilogue warps (two per TMEM lane quarter) store through shared memory with TMA;
//   * stride-2 few-channel convs (the ResNet stem) run as the equivalent stride-1 conv over the
//     space-to-depth form (4C channels, ceil(R/2) x ceil(S/2) filters; k_s2d_prepass).
//
// conv_tc (other stride-1 windows, and the bf16 variant):
//   * same pre-pass; output tile = 8 rows x 2 images x 8 columns laid out in shared memory as row
//     rho = h*16 + img*8 + w, so a filter-row shift r is rho + 16r (2 KB, whole 1 KB swizzle
//     atoms): ONE staged box of (8+R-1) x 2 x 8 positions per (s, 128 B channel chunk) serves all
//     R row shifts; the box is one TMA load over a (c, w, n, h)-permuted view of the NHWC copy;
//   * one thread issues tcgen05.mma (kind::tf32 or kind::f16) into two TMEM accumulators
//     (double-buffered: the epilogue of tile i overlaps the MMAs of tile i+1);
//   * 4 epilogue warps: tcgen05.ld -> streaming stores into NCHW.
#include <cuda_bf16.h>

#include <algorithm>
#include <type_traits>

#include "../host/error.hpp"
#include "common.cuh"
#include "launch.h"
#include "tc_common.cuh"

namespace gb::dev {

#ifdef GENSOR_DEV_OVERRIDES
// Developer timeline of conv_ns (make DEV=1 only): clock64 marks per CTA, 64 slots, read back by
// gensor_dev_conv_trace (tools/conv_trace.py). The product build compiles the marks away.
__device__ long long g_ns_trace[160 * 64];
#define NS_MARK(slot) \
  do {                 \
    if (blockIdx.x < 160) g_ns_trace[blockIdx.x * 64 + (slot)] = clock64(); \
  } while (0)
#else
#define NS_MARK(slot) \
  do {                 \
  } while (0)
#endif

namespace {

using namespace tc;

constexpr int kTH = 8;       // output rows per tile
constexpr int kTI = 2;       // images per tile
constexpr int kTW = 8;       // output columns per tile
constexpr int kProducerWarps = 1;  // one elected thread issues the A-box TMA loads
constexpr int kThreads = 32 * (kProducerWarps + 1 + 4);  // producer, MMA, 4 epilogue warps

template <typename T>
struct ConvTraits;
template <>
struct ConvTraits<float> {
  static constexpr uint32_t kFormat = 2;  // tf32
  static constexpr bool kF16 = false;
};
template <>
struct ConvTraits<__nv_bfloat16> {
  static constexpr uint32_t kFormat = 1;  // bf16
  static constexpr bool kF16 = true;
};

template <typename T, int FN, int STAGES, bool STREAM>
__global__ void __launch_bounds__(kThreads, 1)
    k_conv_tc(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapW, float* __restrict__ O, int N,
              int C, int H, int W, int F, int R, int S, int OH, int OW, int tiles_h, int tiles_w, int total,
              int G) {
  // G > 1 (streamed filters only): tile t = (position tile t / G, filter group t % G of FN filters)
  constexpr int CK = 128 / sizeof(T);        // channels per 128 B row
  constexpr uint32_t W_CHUNK = FN * 128;     // one (r, s, c-chunk) slice of W'
  constexpr uint32_t IDESC = instr_desc(ConvTraits<T>::kFormat, 128, FN, 0, 0);
  constexpr uint32_t TMEM_COLS = 2 * FN;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int nck = (C + CK - 1) / CK;
  const int box_rows = (kTH + R - 1) * kTI * kTW;  // staged positions per (s, c-chunk)
  // STREAM: the filter bank does not fit next to the pipeline, so every stage carries its R
  // filter-row blocks of W' (TMA) next to the A box instead of a resident bank
  const uint32_t w_bytes = STREAM ? 0u : static_cast<uint32_t>(R * S * nck) * W_CHUNK;
  const uint32_t a_bytes = static_cast<uint32_t>(box_rows * 128);
  const uint32_t stage_bytes = a_bytes + (STREAM ? static_cast<uint32_t>(R) * W_CHUNK : 0u);
  uint8_t* wsm = smem;
  uint8_t* asm_ = smem + w_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(asm_ + STAGES * stage_bytes);
  uint64_t* empty = full + STAGES;
  uint64_t* wbar = empty + STAGES;
  uint64_t* acc_full = wbar + 1;       // [2]
  uint64_t* acc_empty = acc_full + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int tiles_img = tiles_h * tiles_w;
  constexpr int kMmaWarp = kProducerWarps;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(wbar, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 4);
    }
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tmem_alloc<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < kProducerWarps) {
    // ---- producer: one TMA box per (tile, channel chunk, s): rows rho = hh*16 + img*8 + w of
    // input positions (n0 + img, h0 + hh, w0 + s + w), 128 B of channels each; out-of-range
    // positions / channels are zero-filled by the TMA unit.
    if (elect_one()) {
      asm volatile("griddepcontrol.wait;" ::: "memory");  // X is written by the preceding pre-pass
      tma_prefetch(&mapX);
      if constexpr (STREAM) tma_prefetch(&mapW);
      int it = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const int tp = t / G, f0 = (t % G) * FN;
        const int n0 = (tp / tiles_img) * kTI;
        const int h0 = ((tp % tiles_img) / tiles_w) * kTH;
        const int w0 = (tp % tiles_w) * kTW;
        for (int ck = 0; ck < nck; ++ck)
          for (int s = 0; s < S; ++s, ++it) {
            const int st = it % STAGES;
            mbar_wait(&empty[st], ((it / STAGES) & 1) ^ 1);
            mbar_arrive_expect_tx(&full[st], stage_bytes);
            tma_load_4d(asm_ + st * stage_bytes, &mapX, &full[st], ck * CK, w0 + s, n0, h0);
            if constexpr (STREAM)
              for (int r = 0; r < R; ++r)
                tma_load_3d(asm_ + st * stage_bytes + a_bytes + r * W_CHUNK, &mapW, &full[st], ck * CK, f0, r * S + s);
          }
      }
    }
  } else if (warp == kMmaWarp) {
    if (elect_one()) {
      // W' is written by the preceding conversion launch (programmatic dependent launch: this
      // grid starts early and only this thread waits for the primary grid's results)
      asm volatile("griddepcontrol.wait;" ::: "memory");
      if constexpr (!STREAM) {
        tma_prefetch(&mapW);
        mbar_arrive_expect_tx(wbar, w_bytes);
        for (int rs = 0; rs < R * S; ++rs)
          for (int ck = 0; ck < nck; ++ck) tma_load_3d(wsm + (rs * nck + ck) * W_CHUNK, &mapW, wbar, ck * CK, 0, rs);
        mbar_wait(wbar, 0);
      }
      const uint32_t w_addr = smem_u32(wsm);
      const uint32_t a_base = smem_u32(asm_);
      int it = 0, local = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++local) {
        const int acc = local & 1;
        mbar_wait(&acc_empty[acc], ((local >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * FN;
        bool first = true;
        for (int ck = 0; ck < nck; ++ck)
          for (int s = 0; s < S; ++s, ++it) {
            const int st = it % STAGES;
            mbar_wait(&full[st], (it / STAGES) & 1);
            tc_fence_after();
            const uint32_t a_addr = a_base + st * stage_bytes;
            for (int r = 0; r < R; ++r) {
              const uint32_t wa = STREAM ? a_addr + a_bytes + r * W_CHUNK : w_addr + ((r * S + s) * nck + ck) * W_CHUNK;
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const uint64_t ad = smem_desc_sw128(a_addr + r * (kTI * kTW * 128) + k * 32, 16, 1024);
                const uint64_t bd = smem_desc_sw128(wa + k * 32, 16, 1024);
                if constexpr (ConvTraits<T>::kF16)
                  mma_f16(d, ad, bd, IDESC, first ? 0u : 1u);
                else
                  mma_tf32(d, ad, bd, IDESC, first ? 0u : 1u);
                first = false;
              }
            }
            mma_commit(&empty[st]);
          }
        mma_commit(&acc_full[acc]);
      }
    }
  } else {
    // ---- epilogue warps: drain TMEM into NCHW ----
    const int q = warp & 3;  // TMEM lane quarter = tile rows m in [32q, 32q+32)
    // position of TMEM lane m = 32q + lane: rho = hh*16 + img*8 + w
    const int hh = (q * 32 + lane) / (kTI * kTW), img = (lane >> 3) & 1, wl = lane & 7;
    const int64_t fstride = static_cast<int64_t>(OH) * OW;
    int local = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++local) {
      const int acc = local & 1;
      const int tp = t / G, f0 = (t % G) * FN;
      const int n = (tp / tiles_img) * kTI + img;
      const int h = ((tp % tiles_img) / tiles_w) * kTH + hh;
      const int w = (tp % tiles_w) * kTW + wl;
      mbar_wait(&acc_full[acc], (local >> 1) & 1);
      tc_fence_after();
      const bool ok = n < N && h < OH && w < OW;
      float* obase = O + (static_cast<int64_t>(n) * F * OH + h) * OW + w + static_cast<int64_t>(f0) * fstride;
#pragma unroll 1
      for (int c = 0; c < FN; c += 32) {
        uint32_t r[32];
        tmem_ld32(tmem + acc * FN + (static_cast<uint32_t>(q * 32) << 16) + c, r);
        tmem_ld_wait();
        tmem_ld_pin(r);
        if (ok) {
#pragma unroll
          for (int v = 0; v < 32; ++v)
            if (f0 + c + v < F) __stcs(obase + (c + v) * fstride, __uint_as_float(r[v]));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc<TMEM_COLS>(tmem);
  }
}

// Pre-pass (one launch, the primary grid of the programmatic dependent launch pair):
//   blocks [0, N*H)      NCHW row (n, h) -> NHWC X[n][h][:][:] through shared memory (coalesced
//                        reads along w, 16 B writes along c);
//   blocks [N*H, ...)    K[f][c][r][s] -> W'[r][s][f][c] (K-major B rows for the conv's TMA).
constexpr int kBandRows = 2;  // pre-pass: max input rows per block (shared-memory sizing)

// rows per pre-pass block: 2 (measured: 1-row bands 10.7 us, 2-row 9.2 us for C; 464 B runs per
// channel)
constexpr int kPrepassBand = 2;

template <typename T>
__global__ void __launch_bounds__(256) k_conv_prepass(const float* __restrict__ I, const float* __restrict__ K,
                                                      T* __restrict__ X, T* __restrict__ Wt, int N, int C, int H,
                                                      int W, int F, int RS, int band) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ float tile[];  // [C][band*W + 1]
  // one block = a band of `band` input rows of one image, all channels: reads C contiguous runs
  // of band*W floats, writes one contiguous NHWC slab
  const int bands_per_img = (H + band - 1) / band;
  const int rows = N * bands_per_img;
  if (static_cast<int>(blockIdx.x) < rows) {
    const int n = blockIdx.x / bands_per_img, h0 = (blockIdx.x % bands_per_img) * band;
    const int nr = min(band, H - h0);
    const int run = nr * W;           // floats per channel in this band
    const int pitch = run + 1;        // odd pitch: transposed reads are bank-conflict free
    const float* src = I + (static_cast<int64_t>(n) * C * H + h0) * W;
    const bool v4 = (reinterpret_cast<uintptr_t>(I) & 15) == 0 && run % 4 == 0 &&
                    (static_cast<int64_t>(H) * W) % 4 == 0 && (static_cast<int64_t>(h0) * W) % 4 == 0;
    if (v4) {
      const int r4 = run / 4;
      for (int i0 = threadIdx.x; i0 < C * r4; i0 += 8 * 256) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = i0 + u * 256;
          const int c = i / r4, x = i - c * r4;
          v[u] = i < C * r4 ? __ldg(reinterpret_cast<const float4*>(src + static_cast<int64_t>(c) * H * W) + x)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = i0 + u * 256;
          const int c = i / r4, x = i - c * r4;
          if (i < C * r4) {
            float* t = tile + c * pitch + 4 * x;
            t[0] = v[u].x;
            t[1] = v[u].y;
            t[2] = v[u].z;
            t[3] = v[u].w;
          }
        }
      }
    } else if ((reinterpret_cast<uintptr_t>(I) & 7) == 0 && run % 2 == 0 && (static_cast<int64_t>(H) * W) % 2 == 0 &&
               (static_cast<int64_t>(h0) * W) % 2 == 0) {  // 8 B-aligned rows (even W): float2
      const int r2 = run / 2;
      for (int i0 = threadIdx.x; i0 < C * r2; i0 += 8 * 256) {
        float2 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = i0 + u * 256;
          const int c = i / r2, x = i - c * r2;
          v[u] = i < C * r2 ? __ldg(reinterpret_cast<const float2*>(src + static_cast<int64_t>(c) * H * W) + x)
                            : make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = i0 + u * 256;
          const int c = i / r2, x = i - c * r2;
          if (i < C * r2) {
            float* t = tile + c * pitch + 2 * x;
            t[0] = v[u].x;
            t[1] = v[u].y;
          }
        }
      }
    } else {
      for (int i = threadIdx.x; i < C * run; i += 256) {
        const int c = i / run, x = i - c * run;
        tile[c * pitch + x] = __ldg(src + static_cast<int64_t>(c) * H * W + x);
      }
    }
    __syncthreads();
    T* dst = X + (static_cast<int64_t>(n) * H + h0) * W * C;  // positions x = (h - h0)*W + w
    if (C % 4 == 0) {  // 4 consecutive channels of one position per thread: 16 B (fp32) stores
      const int c4n = C / 4;
      for (int j = threadIdx.x; j < run * c4n; j += 256) {
        const int x = j / c4n, c = (j - x * c4n) * 4;
        const float a0 = tile[c * pitch + x], a1 = tile[(c + 1) * pitch + x];
        const float a2 = tile[(c + 2) * pitch + x], a3 = tile[(c + 3) * pitch + x];
        if constexpr (sizeof(T) == 4) {
          *reinterpret_cast<float4*>(dst + static_cast<int64_t>(x) * C + c) = make_float4(a0, a1, a2, a3);
        } else {
          __nv_bfloat162 lo = __floats2bfloat162_rn(a0, a1), hi = __floats2bfloat162_rn(a2, a3);
          uint2 u;
          u.x = *reinterpret_cast<uint32_t*>(&lo);
          u.y = *reinterpret_cast<uint32_t*>(&hi);
          *reinterpret_cast<uint2*>(dst + static_cast<int64_t>(x) * C + c) = u;
        }
      }
    } else {
      for (int i = threadIdx.x; i < C * run; i += 256) {
        const int x = i / C, c = i - x * C;
        dst[i] = from_f32<T>(tile[c * pitch + x]);
      }
    }
    return;
  }
  const int64_t total = static_cast<int64_t>(F) * C * RS;
  const int nb = gridDim.x - rows;
  for (int64_t e = (blockIdx.x - rows) * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(nb) * blockDim.x) {
    const int rs = static_cast<int>(e % RS);  // source order: e = (f*C + c)*RS + rs
    const int64_t fc = e / RS;
    const int c = static_cast<int>(fc % C), f = static_cast<int>(fc / C);
    Wt[(static_cast<int64_t>(rs) * F + f) * C + c] = from_f32<T>(__ldg(K + e));
  }
}

// conv_tc geometry shared by the map builder and the launch: filters per tile group (FN),
// whether the filter bank streams per stage, the stage count.
bool tc_fits_stream(int R, int FN) {  // two streamed stages fit shared memory
  const size_t a = static_cast<size_t>((kTH + R - 1) * kTI * kTW * 128);
  return 2 * (a + static_cast<size_t>(R) * FN * 128) <= 227 * 1024 - 1024 - 256;
}

struct TcGeom {
  int FN = 32, G = 1, stages = 0, tiles_h = 0, tiles_w = 0, total = 0;
  bool stream = false;
  size_t w_bytes = 0, a_bytes = 0;
};

TcGeom tc_geom(const ConvTcArgs& a) {
  TcGeom g;
  while (g.FN < a.F) g.FN *= 2;
  if (g.FN > 128 && !tc_fits_stream(a.R, g.FN) &&
      conv_tc_smem_need(a.C, a.F, a.R, a.S, a.bf16) > 227 * 1024 - 1024 - 256)
    g.FN = 128;  // groups of 128 filters, each a tile of its own
  const int CK = a.bf16 ? 64 : 32;
  const int nck = (a.C + CK - 1) / CK;
  const size_t a_bytes0 = static_cast<size_t>((kTH + a.R - 1) * kTI * kTW * 128);
  const size_t bank = static_cast<size_t>(a.R * a.S * nck) * g.FN * 128;
  // resident filter bank when it fits next to two A stages, else filter blocks streamed per stage
  g.stream = bank + 2 * a_bytes0 > 227 * 1024 - 1024 - 256 || g.FN < a.F;
  g.G = (a.F + g.FN - 1) / g.FN;  // filter groups (FN < F only with streamed filters)
  g.w_bytes = g.stream ? 0 : bank;
  g.a_bytes = a_bytes0 + (g.stream ? static_cast<size_t>(a.R) * g.FN * 128 : 0);
  g.tiles_h = (a.OH + kTH - 1) / kTH;
  g.tiles_w = (a.OW + kTW - 1) / kTW;
  g.total = ((a.N + kTI - 1) / kTI) * g.tiles_h * g.tiles_w * g.G;
  g.stages = static_cast<int>((227 * 1024 - 1024 - 256 - g.w_bytes) / g.a_bytes);
  if (g.stages > 6) g.stages = 6;
  return g;
}

void tc_maps(const ConvTcArgs& a, void* ws, ConvTcMaps& m) {
  const TcGeom g = tc_geom(a);
  const int es = a.bf16 ? 2 : 4, CK = 128 / es;
  const uint64_t dw[3] = {static_cast<uint64_t>(a.C), static_cast<uint64_t>(a.F), static_cast<uint64_t>(a.R) * a.S};
  const uint64_t sw[2] = {static_cast<uint64_t>(a.C) * es, static_cast<uint64_t>(a.C) * a.F * es};
  const uint32_t bw[3] = {static_cast<uint32_t>(CK), static_cast<uint32_t>(g.FN), 1};
  encode_map(&m.W, es == 2, es == 4, static_cast<char*>(ws) + a.w_off, 3, dw, sw, bw);
  // NHWC copy viewed as (c, w, n, h): box {CK, 8, 2, 8+R-1} -> smem rows h*16 + img*8 + w
  const uint64_t dx[4] = {static_cast<uint64_t>(a.C), static_cast<uint64_t>(a.W), static_cast<uint64_t>(a.N),
                          static_cast<uint64_t>(a.H)};
  const uint64_t sx[3] = {static_cast<uint64_t>(a.C) * es, static_cast<uint64_t>(a.H) * a.W * a.C * es,
                          static_cast<uint64_t>(a.W) * a.C * es};
  const uint32_t bx[4] = {static_cast<uint32_t>(CK), kTW, kTI, static_cast<uint32_t>(kTH + a.R - 1)};
  encode_map(&m.X, es == 2, es == 4, static_cast<char*>(ws) + a.x_off, 4, dx, sx, bx);
}

template <typename T, int FN>
void run_conv(const ConvTcArgs& a, const ConvTcMaps& m, const float* I, const float* K, float* O, void* ws,
              cudaStream_t st, Marks& mk) {
  const TcGeom g = tc_geom(a);
  const int grid = std::min(g.total, a.sms);
  T* ws_w = reinterpret_cast<T*>(static_cast<char*>(ws) + a.w_off);
  T* ws_x = reinterpret_cast<T*>(static_cast<char*>(ws) + a.x_off);
  auto launch = [&](auto kern) {
    const size_t smem = g.w_bytes + static_cast<size_t>(g.stages) * g.a_bytes + 1024 + 256;
    set_smem_attr(kern, static_cast<int>(smem), "conv_tc smem attribute");
    mk.mark(st);
    const int64_t wt = static_cast<int64_t>(a.F) * a.C * a.R * a.S;
    const int wblocks = static_cast<int>(std::min<int64_t>(64, (wt + 255) / 256));
    const int band = kPrepassBand;
    const size_t pre_smem = static_cast<size_t>(a.C) * (band * a.W + 1) * sizeof(float);
    set_smem_attr(k_conv_prepass<T>, static_cast<int>(pre_smem), "prepass smem attribute");
    k_conv_prepass<T><<<a.N * ((a.H + band - 1) / band) + wblocks, 256, pre_smem, st>>>(I, K, ws_x, ws_w, a.N, a.C,
                                                                                         a.H, a.W, a.F, a.R * a.S, band);
    check_cuda(cudaGetLastError(), "conv prepass launch");
    count_launch();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    check_cuda(cudaLaunchKernelEx(&cfg, kern, m.X, m.W, O, a.N, a.C, a.H, a.W, a.F, a.R, a.S, a.OH, a.OW, g.tiles_h,
                                  g.tiles_w, g.total, g.G),
               "conv_tc launch");
    mk.mark(st);
    count_launch();
  };
  if (g.stream) {
    switch (g.stages) {
      case 2: launch(k_conv_tc<T, FN, 2, true>); return;
      case 3: launch(k_conv_tc<T, FN, 3, true>); return;
      case 4: launch(k_conv_tc<T, FN, 4, true>); return;
      default:
        if (g.stages >= 5) { launch(k_conv_tc<T, FN, 4, true>); return; }
        throw Error(Code::Unsupported, "conv_tc: a streamed stage does not fit in shared memory");
    }
  }
  switch (g.stages) {
    case 1: launch(k_conv_tc<T, FN, 1, false>); break;
    case 2: launch(k_conv_tc<T, FN, 2, false>); break;
    case 3: launch(k_conv_tc<T, FN, 3, false>); break;
    case 4: launch(k_conv_tc<T, FN, 4, false>); break;
    case 5: launch(k_conv_tc<T, FN, 5, false>); break;
    case 6: launch(k_conv_tc<T, FN, 6, false>); break;
    default:
      throw Error(Code::Unsupported, "conv_tc: filter bank does not fit in shared memory");
  }
}

// Space-to-depth pre-pass for stride-2 convs with few channels (the ResNet stem): blocks
// [0, xblocks) write X2[n][h2][w2][(c, dy, dx)] = I[n][c][2 h2 + dy][2 w2 + dx] (0 outside), the
// rest W2[r2][s2][f][(c, dy, dx)] = K[f][c][2 r2 + dy][2 s2 + dx] (0 past the window); conv_ns then
// runs the equivalent stride-1 conv.
__global__ void __launch_bounds__(256) k_s2d_prepass(const float* __restrict__ I, const float* __restrict__ K,
                                                     float* __restrict__ X2, float* __restrict__ W2, int N, int C,
                                                     int H, int W, int F, int R, int S, int H2, int Wd2, int R2,
                                                     int S2, int xblocks) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int C2 = 4 * C;
  if (static_cast<int>(blockIdx.x) < xblocks) {
    // block = output rows (n, h2) for h2-row ids blockIdx.x, blockIdx.x + xblocks, ...: the two
    // input rows of all C channels are read coalesced into shared memory, then the X2 row
    // [w2][(c, dy, dx)] is written contiguously
    extern __shared__ float rowsm[];  // [C][2][W]
    for (int64_t rid = blockIdx.x; rid < static_cast<int64_t>(N) * H2; rid += xblocks) {
      const int n = static_cast<int>(rid / H2), h2 = static_cast<int>(rid % H2);
      // every (channel, row) load of this thread in flight at once (C <= 8: at most 16 rows)
      const float* src = I + (static_cast<int64_t>(n) * C * H + 2 * h2) * W;
      for (int w = threadIdx.x; w < W; w += 256) {
        float v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const int c = k >> 1, dy = k & 1;
          v[k] = (c < C && 2 * h2 + dy < H) ? __ldg(src + (static_cast<int64_t>(c) * H + dy) * W + w) : 0.0f;
        }
#pragma unroll
        for (int k = 0; k < 16; ++k)
          if ((k >> 1) < C) rowsm[k * W + w] = v[k];
      }
      __syncthreads();
      float* dst = X2 + rid * Wd2 * C2;
      // thread = (output column w2, channel c): the 4 values (dy, dx) of one input channel form
      // one 16 B store
      for (int i = threadIdx.x; i < Wd2 * C; i += 256) {
        const int c = i % C, w2 = i / C, w = 2 * w2;
        const float* r0 = rowsm + (c * 2) * W;
        const float4 v = make_float4(r0[w], w + 1 < W ? r0[w + 1] : 0.0f, r0[W + w], w + 1 < W ? r0[W + w + 1] : 0.0f);
        *reinterpret_cast<float4*>(dst + static_cast<int64_t>(w2) * C2 + 4 * c) = v;
      }
      __syncthreads();
    }
    return;
  }
  const int64_t total = static_cast<int64_t>(R2) * S2 * F * C2;
  const int nb = gridDim.x - xblocks;
  for (int64_t e = (blockIdx.x - xblocks) * 256LL + threadIdx.x; e < total; e += static_cast<int64_t>(nb) * 256) {
    const int c2 = static_cast<int>(e % C2);
    const int f = static_cast<int>((e / C2) % F);
    const int rs = static_cast<int>(e / (static_cast<int64_t>(C2) * F));
    const int r2 = rs / S2, s2 = rs % S2;
    const int c = c2 >> 2, r = 2 * r2 + ((c2 >> 1) & 1), sc = 2 * s2 + (c2 & 1);
    W2[e] = (r < R && sc < S) ? __ldg(K + ((static_cast<int64_t>(f) * C + c) * R + r) * S + sc) : 0.0f;
  }
}

// ---------------------------------------------------------------------------------------------
// conv_ns: stride-1 tf32 conv with S*F <= 256, reading the NCHW input IN PLACE (no NHWC copy).
//   * tile = 4 output rows x 32 columns of one image; the A operand is MN-major (32 consecutive
//     input columns of one row = one 128 B row per channel, 32 B-atom swizzle), staged per
//     32-channel chunk as (4 + R - 1) row chunks of 4 KB: a filter-row shift r is +4 KB;
//   * the filter columns s are folded into N: B = W'[r][chunk][s][f][c] rows (s, f), so one
//     N = S*FN MMA computes, for every staged input position, its products with all S filter
//     columns (full tensor-core rate at N = 192 instead of N = 64 per s, and no s-shifted
//     copies of A); the epilogue adds column s of TMEM lane w + s into output w with a warp
//     shuffle: outputs w < 32 - (S - 1) of each tile are valid;
//   * 8 software producer warps (two groups alternating chunks) load 128 B input row segments
//     with coalesced LDG and store them swizzled (the input rows are only 8 B aligned, which
//     TMA cannot address); the filter bank is TMA-loaded once and stays resident.
constexpr int kNsRows = 4, kNsCols = 32;
constexpr int kNsEpi = 8;  // epilogue warps: two per TMEM lane quarter, splitting the filter blocks
constexpr int kNsThreads = 32 * (1 + 1 + kNsEpi);

template <int STAGES, int SMAX>
__global__ void __launch_bounds__(kNsThreads, 1)
    k_conv_ns(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapW,
              const __grid_constant__ CUtensorMap mapO, int tma_store, float* __restrict__ O, int N,
              int C, int H, int W, int F, int FN, int R, int S, int OH, int OW, int tiles_h, int tiles_w, int total,
              int valid_w) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int nck = (C + 31) / 32;
  const int rows = kNsRows + R - 1;
  const int ncol = S * FN;  // UMMA N
  const uint32_t w_bytes = static_cast<uint32_t>(R * nck * ncol) * 128;
  const uint32_t a_bytes = static_cast<uint32_t>(rows) * 4096;
  uint8_t* wsm = smem;
  uint8_t* asm_ = smem + w_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(asm_ + STAGES * a_bytes);
  uint64_t* empty = full + STAGES;
  constexpr int kWb = 8;  // filter-bank barriers: one per 32-channel chunk (the last takes the rest)
  uint64_t* wbar = empty + STAGES;
  uint64_t* acc_full = wbar + kWb;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  float* stage_o = reinterpret_cast<float*>(smem + w_bytes + STAGES * a_bytes + 1024);  // [8 warps][8][32]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_img = tiles_h * tiles_w;
  constexpr int kMma = 1;
  if (threadIdx.x == 0) NS_MARK(0);
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < kWb; ++i) mbar_init(&wbar[i], 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], kNsEpi);
    }
    fence_barrier_init();
  }
  if (warp == kMma) {
    if (2 * ncol > 256) tmem_alloc<512>(tmem_slot);
    else tmem_alloc<256>(tmem_slot);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---- producer: one TMA box per (tile, 32-channel chunk) from the NHWC copy viewed as
    // (c, w, h, n): box {32, 32, 4 + R - 1, 1} -> K-major rows rho = hh*32 + w (128 B of
    // channels each, 128 B swizzle); out-of-range positions / channels are zero-filled
    if (elect_one()) {
      asm volatile("griddepcontrol.wait;" ::: "memory");  // X is written by the preceding pre-pass
      NS_MARK(1);
      tma_prefetch(&mapX);
      int it = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const int n = t / tiles_img;
        const int h0 = ((t % tiles_img) / tiles_w) * kNsRows;
        const int w0 = (t % tiles_w) * valid_w;
        for (int ck = 0; ck < nck; ++ck, ++it) {
          const int st = it % STAGES;
          mbar_wait(&empty[st], ((it / STAGES) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[st], a_bytes);
          tma_load_4d(asm_ + st * a_bytes, &mapX, &full[st], ck * 32, w0, h0, n);
        }
      }
    }
  } else if (warp == kMma) {
    if (elect_one()) {
      asm volatile("griddepcontrol.wait;" ::: "memory");  // W' is written by the preceding launch
      tma_prefetch(&mapW);
      // chunk-major filter loads with a barrier per chunk: the first chunk's MMAs start once its
      // R*S blocks have landed instead of after the whole bank
      const uint32_t chunk_bytes = static_cast<uint32_t>(R * S * FN) * 128;
      for (int ck = 0; ck < nck; ++ck) {
        uint64_t* wb = &wbar[ck < kWb ? ck : kWb - 1];
        if (ck < kWb - 1) mbar_arrive_expect_tx(wb, chunk_bytes);
        else if (ck == kWb - 1) mbar_arrive_expect_tx(wb, chunk_bytes * static_cast<uint32_t>(nck - ck));
        for (int r = 0; r < R; ++r)
          for (int s = 0; s < S; ++s)
            tma_load_3d(wsm + ((r * nck + ck) * S + s) * FN * 128, &mapW, wb, ck * 32, 0, r * S + s);
      }
      const uint32_t idesc = instr_desc(2, 128, static_cast<uint32_t>(ncol), 0, 0);
      const uint32_t w_addr = smem_u32(wsm), a_base = smem_u32(asm_);
      int it = 0, local = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++local) {
        const int acc = local & 1;
        mbar_wait(&acc_empty[acc], ((local >> 1) & 1) ^ 1);
        if (local < 6) NS_MARK(8 + local);
        tc_fence_after();
        const uint32_t d = tmem + acc * ncol;
        bool first = true;
        for (int ck = 0; ck < nck; ++ck, ++it) {
          const int st = it % STAGES;
          mbar_wait(&full[st], (it / STAGES) & 1);
          if (local == 0 && ck < kWb) mbar_wait(&wbar[ck], 0);  // chunk ck's filters (last: the rest)
          if (local == 0 && ck == 0) NS_MARK(2);
          tc_fence_after();
          const uint32_t a_addr = a_base + st * a_bytes;
          // k-steps of 8 channels that hold real channels (a 12-channel space-to-depth chunk: 2)
          const int ksteps = min(4, (C - ck * 32 + 7) / 8);
          for (int r = 0; r < R; ++r) {
            const uint32_t wb = w_addr + (r * nck + ck) * ncol * 128;
            for (int k = 0; k < ksteps; ++k) {
              mma_tf32(d, smem_desc_sw128(a_addr + r * 4096 + k * 32, 16, 1024),
                       smem_desc_sw128(wb + k * 32, 16, 1024), idesc, first ? 0u : 1u);
              first = false;
            }
          }
          mma_commit(&empty[st]);
        }
        mma_commit(&acc_full[acc]);
        if (local < 6) NS_MARK(16 + local);
      }
    }
  } else {
    // ---- epilogue: warp q owns TMEM lanes 32q.. = tile row q; lane = input column w0 + lane.
    // out(w) = sum_s D[lane w + s][s*FN + f]: TMEM column block s of the neighbour s lanes down
    const int q = warp & 3, half = (warp - kMma - 1) >> 2;  // lane quarter, filter-block parity
    const int64_t fstride = static_cast<int64_t>(OH) * OW;
    int local = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++local) {
      const int acc = local & 1;
      const int n = t / tiles_img;
      const int h = ((t % tiles_img) / tiles_w) * kNsRows + q;
      const int w = (t % tiles_w) * valid_w + lane;
      mbar_wait(&acc_full[acc], (local >> 1) & 1);
      if (warp == kMma + 1 && lane == 0 && local < 6) NS_MARK(24 + local);
      tc_fence_after();
      const bool ok = lane < valid_w && n < N && h < OH && w < OW;
      float* obase = O + (static_cast<int64_t>(n) * F * OH + h) * OW + w;
#pragma unroll 1
      for (int c0 = half * 32; c0 < FN + 32 * half; c0 += 64) {
        if (c0 >= FN) {  // FN = 32: the second warp of the quarter has no block; release only
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&acc_empty[acc]);
          break;
        }
        uint32_t r0[32], r1[32], r2[32], r3[SMAX > 3 ? 32 : 1];
        const uint32_t base = tmem + acc * ncol + (static_cast<uint32_t>(q * 32) << 16) + c0;
        tmem_ld32(base, r0);
        if (S > 1) tmem_ld32(base + FN, r1);
        if (S > 2) tmem_ld32(base + 2 * FN, r2);
        if constexpr (SMAX > 3) {
          if (S > 3) tmem_ld32(base + 3 * FN, r3);
        }
        tmem_ld_wait();
        tmem_ld_pin(r0);
        tmem_ld_pin(r1);
        tmem_ld_pin(r2);
        tmem_ld_pin(r3);
        if (c0 + 64 >= FN) {  // this warp's last TMEM block is in registers: hand the accumulator back
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&acc_empty[acc]);
        }
        if (tma_store) {
          // four 8-filter quarters through this warp's staging slice [8 f][valid_w], each written
          // to the NCHW output by one TMA store (clipped at the tensor edges)
          float* stg = stage_o + ((warp - kMma - 1) * 8) * kNsCols;
#pragma unroll
          for (int hf = 0; hf < 4; ++hf) {
            if (lane == 0) bulk_wait_read<0>();  // the previous store has read the slice
            __syncwarp();
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
              const int j = hf * 8 + jj;
              float v = __uint_as_float(r0[j]);
              const float v1 = __shfl_down_sync(0xffffffffu, __uint_as_float(r1[j]), 1);
              const float v2 = __shfl_down_sync(0xffffffffu, __uint_as_float(r2[j]), 2);
              if (S > 1) v += v1;
              if (S > 2) v += v2;
              if constexpr (SMAX > 3) {
                const float v3 = __shfl_down_sync(0xffffffffu, __uint_as_float(r3[j]), 3);
                if (S > 3) v += v3;
              }
              if (lane < valid_w) stg[jj * valid_w + lane] = v;
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_4d(&mapO, stg, (t % tiles_w) * valid_w, ((t % tiles_img) / tiles_w) * kNsRows + q, c0 + hf * 8,
                           n);
              bulk_commit();
            }
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            float v = __uint_as_float(r0[j]);
            const float v1 = __shfl_down_sync(0xffffffffu, __uint_as_float(r1[j]), 1);
            const float v2 = __shfl_down_sync(0xffffffffu, __uint_as_float(r2[j]), 2);
            if (S > 1) v += v1;
            if (S > 2) v += v2;
            if constexpr (SMAX > 3) {
              const float v3 = __shfl_down_sync(0xffffffffu, __uint_as_float(r3[j]), 3);
              if (S > 3) v += v3;
            }
            // default write-back caching: neighbouring tiles complete the partial sectors in L2
            if (ok && c0 + j < F) obase[(c0 + j) * fstride] = v;
          }
        }
      }
      if (warp == kMma + 1 && lane == 0 && local < 6) NS_MARK(32 + local);
    }
    if (tma_store && lane == 0) bulk_wait_read<0>();  // the staging is read before the CTA retires
    if (warp == kMma + 1 && lane == 0) NS_MARK(40);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMma) {
    tc_fence_after();
    if (2 * ncol > 256) tmem_dealloc<512>(tmem);
    else tmem_dealloc<256>(tmem);
  }
}

// conv_ns geometry: the kernel's problem is the op itself, or (stride 2) its space-to-depth form —
// a stride-1 conv over C2 = 4C channels (c, dy, dx) of ceil(H/2) x ceil(W/2) positions with
// ceil(R/2) x ceil(S/2) filters (K'[f][(c,dy,dx)][r'][s'] = K[f][c][2r'+dy][2s'+dx], 0 past the window)
struct NsGeom {
  int FN = 32, gC = 0, gH = 0, gW = 0, gR = 0, gS = 0, nck = 0;
  int valid_w = 0, tiles_w = 0, tiles_h = 0, total = 0, stages = 0;
  bool tma_store = false;
  size_t w_bytes = 0, a_bytes = 0, stage_o = 0;
};

NsGeom ns_geom(const ConvTcArgs& a) {
  NsGeom g;
  while (g.FN < a.F) g.FN *= 2;
  g.gC = a.s2d ? 4 * a.C : a.C;
  g.gH = a.s2d ? (a.H + 1) / 2 : a.H;
  g.gW = a.s2d ? (a.W + 1) / 2 : a.W;
  g.gR = a.s2d ? (a.R + 1) / 2 : a.R;
  g.gS = a.s2d ? (a.S + 1) / 2 : a.S;
  g.nck = (g.gC + 31) / 32;
  g.w_bytes = static_cast<size_t>(g.gR) * g.nck * g.gS * g.FN * 128;
  g.a_bytes = static_cast<size_t>(kNsRows + g.gR - 1) * 4096;
  // output columns per tile: at most 32 - (S - 1), balanced over the row (56 -> 2 x 28); with
  // 16 B-multiple output rows the epilogue stores through TMA, which needs valid_w % 4 == 0
  g.tma_store = a.OW % 4 == 0;
  const int vmax = g.tma_store ? (kNsCols - (g.gS - 1)) & ~3 : kNsCols - (g.gS - 1);
  g.tiles_w = (a.OW + vmax - 1) / vmax;
  g.valid_w = (a.OW + g.tiles_w - 1) / g.tiles_w;
  if (g.tma_store) g.valid_w = (g.valid_w + 3) & ~3;
  g.tiles_h = (a.OH + kNsRows - 1) / kNsRows;
  g.total = a.N * g.tiles_h * g.tiles_w;
  g.stage_o = kNsEpi * 8 * kNsCols * sizeof(float);  // epilogue staging (TMA-store path)
  const size_t budget = 227 * 1024 - 2048 - g.stage_o;
  g.stages = static_cast<int>((budget - g.w_bytes) / g.a_bytes);
  if (g.stages > 6) g.stages = 6;
  return g;
}

void ns_maps(const ConvTcArgs& a, void* ws, void* O, ConvTcMaps& m) {
  const NsGeom g = ns_geom(a);
  const uint64_t dw[3] = {static_cast<uint64_t>(g.gC), static_cast<uint64_t>(a.F), static_cast<uint64_t>(g.gR) * g.gS};
  const uint64_t sw[2] = {static_cast<uint64_t>(g.gC) * 4, static_cast<uint64_t>(g.gC) * a.F * 4};
  const uint32_t bw[3] = {32, static_cast<uint32_t>(g.FN), 1};
  encode_map(&m.W, false, true, static_cast<char*>(ws) + a.w_off, 3, dw, sw, bw);
  // NHWC copy viewed as (c, w, h, n): box {32, 32, 4 + R - 1, 1} -> rows hh*32 + w
  const uint64_t dx[4] = {static_cast<uint64_t>(g.gC), static_cast<uint64_t>(g.gW), static_cast<uint64_t>(g.gH),
                          static_cast<uint64_t>(a.N)};
  const uint64_t sx[3] = {static_cast<uint64_t>(g.gC) * 4, static_cast<uint64_t>(g.gW) * g.gC * 4,
                          static_cast<uint64_t>(g.gH) * g.gW * g.gC * 4};
  const uint32_t bx[4] = {32, kNsCols, static_cast<uint32_t>(kNsRows + g.gR - 1), 1};
  encode_map(&m.X, false, true, static_cast<char*>(ws) + a.x_off, 4, dx, sx, bx);
  if (g.tma_store) {  // NCHW output as (w, h, f, n): box {valid_w, 1, 8, 1}
    const uint64_t dout[4] = {static_cast<uint64_t>(a.OW), static_cast<uint64_t>(a.OH), static_cast<uint64_t>(a.F),
                              static_cast<uint64_t>(a.N)};
    const uint64_t sout[3] = {static_cast<uint64_t>(a.OW) * 4, static_cast<uint64_t>(a.OH) * a.OW * 4,
                              static_cast<uint64_t>(a.F) * a.OH * a.OW * 4};
    const uint32_t bout[4] = {static_cast<uint32_t>(g.valid_w), 1, 8, 1};
    encode_map_swizzle(&m.O, false, false, O, 4, dout, sout, bout, CU_TENSOR_MAP_SWIZZLE_NONE);
  }
}

void run_conv_ns(const ConvTcArgs& a, const ConvTcMaps& m, const float* I, const float* K, float* O, void* ws,
                 cudaStream_t st, Marks& mk) {
  const NsGeom g = ns_geom(a);
  const int grid = std::min(g.total, a.sms);
  float* ws_w = reinterpret_cast<float*>(static_cast<char*>(ws) + a.w_off);
  float* ws_x = reinterpret_cast<float*>(static_cast<char*>(ws) + a.x_off);
  auto launch = [&](auto kern) {
    const size_t smem = g.w_bytes + static_cast<size_t>(g.stages) * g.a_bytes + 1024 + g.stage_o + 1024;
    set_smem_attr(kern, static_cast<int>(smem), "conv_ns smem attribute");
    mk.mark(st);
    const int64_t wt = static_cast<int64_t>(a.F) * g.gC * g.gR * g.gS;
    const int wblocks = static_cast<int>(std::min<int64_t>(64, (wt + 255) / 256));
    const char* skip = dev_env("GENSOR_CONV_SKIP");  // developer timing: "prepass" | "conv"
    if (skip && skip[0] == 'p') {
      // the workspace holds the previous execute's copy
    } else if (a.s2d) {
      const int xblocks = static_cast<int>(std::min<int64_t>(1 << 20, static_cast<int64_t>(a.N) * g.gH));  // a row per block
      const size_t rsm = static_cast<size_t>(a.C) * 2 * a.W * sizeof(float);
      set_smem_attr(k_s2d_prepass, static_cast<int>(rsm), "s2d smem attribute");
      k_s2d_prepass<<<xblocks + wblocks, 256, rsm, st>>>(I, K, ws_x, ws_w, a.N, a.C, a.H, a.W, a.F, a.R, a.S, g.gH,
                                                       g.gW, g.gR, g.gS, xblocks);
    } else {
      const int band = kPrepassBand;
      const size_t pre_smem = static_cast<size_t>(a.C) * (band * a.W + 1) * sizeof(float);
      set_smem_attr(k_conv_prepass<float>, static_cast<int>(pre_smem), "prepass smem attribute");
      k_conv_prepass<float><<<a.N * ((a.H + band - 1) / band) + wblocks, 256, pre_smem, st>>>(
          I, K, ws_x, ws_w, a.N, a.C, a.H, a.W, a.F, a.R * a.S, band);
    }
    check_cuda(cudaGetLastError(), "conv filter conversion launch");
    count_launch();
    if (skip && skip[0] == 'c') {
      mk.mark(st);
      return;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kNsThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    check_cuda(cudaLaunchKernelEx(&cfg, kern, m.X, m.W, m.O, g.tma_store ? 1 : 0, O, a.N, g.gC, g.gH, g.gW, a.F, g.FN,
                                  g.gR, g.gS, a.OH, a.OW, g.tiles_h, g.tiles_w, g.total, g.valid_w),
               "conv_ns launch");
    mk.mark(st);
    count_launch();
  };
  auto pick = [&](auto smax) {
    constexpr int SM = decltype(smax)::value;
    switch (g.stages) {
      case 2: launch(k_conv_ns<2, SM>); break;
      case 3: launch(k_conv_ns<3, SM>); break;
      case 4: launch(k_conv_ns<4, SM>); break;
      case 5: launch(k_conv_ns<5, SM>); break;
      case 6: launch(k_conv_ns<6, SM>); break;
      default: throw Error(Code::Unsupported, "conv_ns: filter bank does not fit in shared memory");
    }
  };
  // 4 filter columns need a fourth TMEM block in registers: a separate instantiation keeps the
  // 3-column epilogue (the headline) free of its register pressure
  if (g.gS > 3)
    pick(std::integral_constant<int, 4>{});
  else
    pick(std::integral_constant<int, 3>{});
}
}  // namespace

size_t conv_tc_smem_need(int C, int F, int R, int S, bool bf16) {
  const int CK = bf16 ? 64 : 32;
  int FN = 32;
  while (FN < F) FN *= 2;
  const size_t nck = (C + CK - 1) / CK;
  return static_cast<size_t>(R) * S * nck * FN * 128 + 2 * static_cast<size_t>((kTH + R - 1) * kTI * kTW * 128);
}

bool conv_tc_supported(int C, int F, int R, int S, int stride, bool bf16) {
  const int es = bf16 ? 2 : 4;
  if (!(stride == 1 && F >= 1 && F <= 256 && (C * es) % 16 == 0 && R >= 1 && R <= 8 && S >= 1 && S <= 8)) return false;
  if (conv_tc_smem_need(C, F, R, S, bf16) <= 227 * 1024 - 1024 - 256) return true;  // resident bank
  int FN = 32;
  while (FN < F) FN *= 2;
  return tc_fits_stream(R, FN) || tc_fits_stream(R, 128);  // streamed (split) blocks
}

bool conv_tc_prepass_fits(int C, int W) {  // a band of NCHW rows of all channels through smem
  return static_cast<size_t>(C) * (kBandRows * W + 1) * sizeof(float) <= 96 * 1024;
}

bool conv_s2d_supported(int C, int F, int R, int S, int stride, bool bf16) {
  // stride-2, few channels: the space-to-depth form is a stride-1 conv_ns problem with 4C <= 32
  // channels (one chunk) and ceil(S/2) <= 4 filter columns
  int FN = 32;
  while (FN < F) FN *= 2;
  const int R2 = (R + 1) / 2, S2 = (S + 1) / 2;
  const size_t w_bytes = static_cast<size_t>(R2) * S2 * FN * 128;
  return !bf16 && stride == 2 && 4 * C <= 32 && R2 >= 2 && R2 <= 8 && S2 <= 4 &&
         S2 * FN <= 256 && w_bytes + 2 * static_cast<size_t>(kNsRows + R2 - 1) * 4096 <= 227 * 1024 - 2048 - kNsEpi * 8 * kNsCols * 4;
}

bool conv_ns_supported(int C, int F, int R, int S, int stride, bool bf16) {
  int FN = 32;
  while (FN < F) FN *= 2;
  const size_t w_bytes = static_cast<size_t>(R) * ((C + 31) / 32) * S * FN * 128;
  return !bf16 && stride == 1 && C % 4 == 0 && S >= 1 && S <= 4 && R >= 1 && R <= 8 && S * FN <= 256 &&
         w_bytes + 2 * static_cast<size_t>(kNsRows + R - 1) * 4096 <= 227 * 1024 - 2048 - kNsEpi * 8 * kNsCols * 4;
}

#ifdef GENSOR_DEV_OVERRIDES
extern "C" int gensor_dev_conv_trace(long long* out, int n) {
  return cudaMemcpyFromSymbol(out, g_ns_trace, sizeof(long long) * std::min(n, 160 * 64)) == cudaSuccess ? 0 : 19;
}
#endif

void conv_tc_maps(const ConvTcArgs& a, void* ws, void* O, ConvTcMaps& m) {
  if (a.ns)
    ns_maps(a, ws, O, m);
  else
    tc_maps(a, ws, m);
}

void launch_conv_tc(const ConvTcArgs& a, const ConvTcMaps& m, const void* I, const void* K, void* O, void* ws,
                    cudaStream_t st, Marks& mk) {
  const float* i = static_cast<const float*>(I);
  const float* k = static_cast<const float*>(K);
  float* o = static_cast<float*>(O);
  if (a.ns) {
    run_conv_ns(a, m, i, k, o, ws, st, mk);
    return;
  }
  const int FN = tc_geom(a).FN;
  if (a.bf16) {
    switch (FN) {
      case 32: run_conv<__nv_bfloat16, 32>(a, m, i, k, o, ws, st, mk); break;
      case 64: run_conv<__nv_bfloat16, 64>(a, m, i, k, o, ws, st, mk); break;
      case 128: run_conv<__nv_bfloat16, 128>(a, m, i, k, o, ws, st, mk); break;
      default: run_conv<__nv_bfloat16, 256>(a, m, i, k, o, ws, st, mk); break;
    }
  } else {
    switch (FN) {
      case 32: run_conv<float, 32>(a, m, i, k, o, ws, st, mk); break;
      case 64: run_conv<float, 64>(a, m, i, k, o, ws, st, mk); break;
      case 128: run_conv<float, 128>(a, m, i, k, o, ws, st, mk); break;
      default: run_conv<float, 256>(a, m, i, k, o, ws, st, mk); break;
    }
  }
}

}  // namespace gb::dev
