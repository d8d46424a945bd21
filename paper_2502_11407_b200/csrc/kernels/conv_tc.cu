// Tensor-core implicit-GEMM conv2d (stride 1), instantiated from a constructed conv2d schedule:
//   O[n][f][h][w] = sum_{c,r,s} I[n][c][h+r][w+s] * K[f][c][r][s]   (op_spec.cpp:177-181)
// GEMM view: M = output positions (h, w), N = f, K = (r, s, c).
//
// Step 1 (pre-pass, HBM-bound): NCHW input -> NHWC X (so c is the contiguous K dim a TMA box
// can load as 128 B swizzled rows) and K[f][c][r][s] -> W'[r][s][f][c].
// Step 2 (persistent tcgen05 kernel, one CTA per SM):
//   * the whole W' lives in shared memory for the CTA's lifetime (loaded once by TMA);
//   * an output tile is BH=4 rows x BW=32 columns of one image (M = 128 = one UMMA M);
//   * for each (s, 128 B c-chunk) the producer loads ONE box of (BH+R-1) x BW positions; the R
//     row shifts are 1024 B-aligned sub-views of that box, so each A row is fetched once per s
//     instead of once per (r, s) — a 3x cut of the L2->SM operand traffic for 3x3 filters;
//   * TMEM holds two 128 x FN fp32 accumulators so the epilogue of tile i overlaps tile i+1;
//   * epilogue warp q owns output row h0+q: lane = w, each tcgen05.ld column f is one coalesced
//     128 B store to O[n][f][h][w0..w0+31].
#include <cuda_bf16.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../host/error.hpp"
#include "common.cuh"
#include "launch.h"
#include "tc_common.cuh"

namespace gb::dev {

namespace {

using namespace tc;

constexpr int kBH = 4;
constexpr int kBW = 32;

// NCHW fp32 -> NHWC (fp32 or bf16), 32x32 tiles of [c][w] per (n, h) through shared memory.
template <typename TX>
__global__ void __launch_bounds__(256) k_nchw_to_nhwc(const float* __restrict__ in, TX* __restrict__ out, int C, int H,
                                                      int W) {
  __shared__ float tile[32][33];
  const int nh = blockIdx.z;  // n * H + h
  const int c0 = blockIdx.y * 32, w0 = blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t n = nh / H, h = nh % H;
  const float* src = in + (n * C) * static_cast<int64_t>(H) * W + h * W;
#pragma unroll
  for (int i = ty; i < 32; i += 8) {
    const int c = c0 + i, w = w0 + tx;
    tile[i][tx] = (c < C && w < W) ? src[static_cast<int64_t>(c) * H * W + w] : 0.0f;
  }
  __syncthreads();
  TX* dst = out + (static_cast<int64_t>(nh) * W) * C;
#pragma unroll
  for (int i = ty; i < 32; i += 8) {
    const int w = w0 + i, c = c0 + tx;
    if (w < W && c < C) dst[static_cast<int64_t>(w) * C + c] = from_f32<TX>(tile[tx][i]);
  }
}

template <typename TX>
__global__ void k_weights_rsfc(const float* __restrict__ k, TX* __restrict__ out, int F, int C, int R, int S) {
  const int64_t total = static_cast<int64_t>(F) * C * R * S;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    // out index (r, s, f, c)
    int64_t t = i;
    const int c = t % C;
    t /= C;
    const int f = t % F;
    t /= F;
    const int s = t % S;
    const int r = static_cast<int>(t / S);
    out[i] = from_f32<TX>(k[((static_cast<int64_t>(f) * C + c) * R + r) * S + s]);
  }
}

template <typename T>
struct ConvTraits;
template <>
struct ConvTraits<float> {
  static constexpr uint32_t kFormat = 2;
  static constexpr bool kF16 = false;
};
template <>
struct ConvTraits<__nv_bfloat16> {
  static constexpr uint32_t kFormat = 1;
  static constexpr bool kF16 = true;
};

template <typename T, int FN, int STAGES>
__global__ void __launch_bounds__(192, 1)
    k_conv_tc(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapW,
              float* __restrict__ O, int F, int C, int R, int S, int OH, int OW, int tiles_h, int tiles_w,
              int total_tiles, long long* __restrict__ trace, int xflags) {
#define CONV_TRACE(slot, v) \
  if (trace) trace[blockIdx.x * 64 + (slot)] = (v)
  auto gtimer = []() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return static_cast<long long>(t);
  };
  if (threadIdx.x == 0) CONV_TRACE(62, gtimer());
  constexpr int CK = 128 / sizeof(T);  // channels per 128 B row
  constexpr uint32_t W_CHUNK = FN * 128;
  constexpr uint32_t IDESC = instr_desc(ConvTraits<T>::kFormat, 128, FN, 0, 0);
  constexpr uint32_t TMEM_COLS = 2 * FN;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int nck = (C + CK - 1) / CK;
  const uint32_t w_bytes = static_cast<uint32_t>(R * S * nck) * W_CHUNK;
  const uint32_t a_bytes = static_cast<uint32_t>((kBH + R - 1) * kBW * 128);
  uint8_t* wsm = smem;
  uint8_t* asm_ = smem + w_bytes;  // STAGES x a_bytes (each a multiple of 1024)
  uint64_t* full = reinterpret_cast<uint64_t*>(asm_ + STAGES * a_bytes);
  uint64_t* empty = full + STAGES;
  uint64_t* wbar = empty + STAGES;
  uint64_t* acc_full = wbar + 1;   // [2]
  uint64_t* acc_empty = acc_full + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int tiles_img = tiles_h * tiles_w;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(wbar, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 4);  // one arrival per epilogue warp
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      tma_prefetch(&mapX);
      tma_prefetch(&mapW);
      // resident weights: one (F x 128 B) K-major chunk per (r, s, c-chunk)
      mbar_arrive_expect_tx(wbar, w_bytes);
      for (int rs = 0; rs < R * S; ++rs)
        for (int ck = 0; ck < nck; ++ck)
          tma_load_3d(wsm + (rs * nck + ck) * W_CHUNK, &mapW, wbar, ck * CK, 0, rs);
      int it = 0;
      long long pw = 0;
      int pt = 0;
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x, ++pt) {
        const int n = t / tiles_img;
        const int th = (t % tiles_img) / tiles_w;
        const int tw = t % tiles_w;
        for (int s = 0; s < S; ++s)
          for (int ck = 0; ck < nck; ++ck, ++it) {
            const int st = it % STAGES;
            const uint32_t ph = (it / STAGES) & 1;
            const long long w0 = trace ? clock64() : 0;
            mbar_wait(&empty[st], ph ^ 1);
            if (trace) pw += clock64() - w0;
            if (xflags & 4) {
              mbar_arrive(&full[st]);
            } else {
              mbar_arrive_expect_tx(&full[st], a_bytes);
              tma_load_4d(asm_ + st * a_bytes, &mapX, &full[st], ck * CK, tw * kBW + s, th * kBH, n);
            }
          }
        CONV_TRACE(20 + pt, clock64());
      }
      CONV_TRACE(61, pw);
    }
  } else if (warp == 1) {
    if (elect_one()) {
      CONV_TRACE(0, clock64());
      mbar_wait(wbar, 0);
      CONV_TRACE(1, clock64());
      long long fw = 0;
      const uint32_t w_addr = smem_u32(wsm);
      const uint32_t a_base = smem_u32(asm_);
      int it = 0, local = 0;
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x, ++local) {
        const int acc = local & 1;
        mbar_wait(&acc_empty[acc], ((local >> 1) & 1) ^ 1);
        CONV_TRACE(2 + 2 * local, clock64());
        tc_fence_after();
        const uint32_t d = tmem + acc * FN;
        bool first = true;
        for (int s = 0; s < S; ++s)
          for (int ck = 0; ck < nck; ++ck, ++it) {
            const int st = it % STAGES;
            const long long w0 = trace ? clock64() : 0;
            mbar_wait(&full[st], (it / STAGES) & 1);
            if (trace) fw += clock64() - w0;
            tc_fence_after();
            const uint32_t a_addr = a_base + st * a_bytes;
            for (int r = 0; r < R; ++r) {
              const uint32_t wa = w_addr + ((r * S + s) * nck + ck) * W_CHUNK;
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const uint64_t ad = smem_desc_sw128(a_addr + r * (kBW * 128) + k * 32, 16, 1024);
                const uint64_t bd = smem_desc_sw128(wa + k * 32, 16, 1024);
                if (xflags & 2) {
                } else if constexpr (ConvTraits<T>::kF16)
                  mma_f16(d, ad, bd, IDESC, first ? 0u : 1u);
                else
                  mma_tf32(d, ad, bd, IDESC, first ? 0u : 1u);
                first = false;
              }
            }
            mma_commit(&empty[st]);
          }
        mma_commit(&acc_full[acc]);
        CONV_TRACE(3 + 2 * local, clock64());
      }
      CONV_TRACE(60, fw);
    }
  } else {
    const int q = warp & 3;  // lane quarter = output row offset within the tile
    int local = 0;
    for (int t = blockIdx.x; t < total_tiles; t += gridDim.x, ++local) {
      const int acc = local & 1;
      const int n = t / tiles_img;
      const int h = ((t % tiles_img) / tiles_w) * kBH + q;
      const int w = (t % tiles_w) * kBW + lane;
      mbar_wait(&acc_full[acc], (local >> 1) & 1);
      tc_fence_after();
      const bool ok = h < OH && w < OW;
      float* obase = O + ((static_cast<int64_t>(n) * F) * OH + h) * OW + w;
      const int64_t fstride = static_cast<int64_t>(OH) * OW;
#pragma unroll 1
      for (int c = 0; c < FN; c += 16) {
        uint32_t r[16];
        tmem_ld16(tmem + acc * FN + (static_cast<uint32_t>(q * 32) << 16) + c, r);
        tmem_ld_wait();
        if (ok && !(xflags & 1)) {
#pragma unroll
          for (int v = 0; v < 16; ++v)
            if (c + v < F) obase[(c + v) * fstride] = __uint_as_float(r[v]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[acc]);
      if (warp == 2 && lane == 0) CONV_TRACE(40 + local, clock64());
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<TMEM_COLS>(tmem);
  }
  if (threadIdx.x == 0) CONV_TRACE(63, gtimer());
}

template <typename T, int FN>
void run_conv(ConvTcArgs& a, const float* I, const float* K, float* O, cudaStream_t st, Marks& mk) {
  constexpr int CK = 128 / sizeof(T);
  const int nck = (a.C + CK - 1) / CK;
  const size_t w_bytes = static_cast<size_t>(a.R * a.S * nck) * FN * 128;
  const size_t a_bytes = static_cast<size_t>((kBH + a.R - 1) * kBW * 128);
  T* X = static_cast<T*>(a.ws_x);
  T* Wt = static_cast<T*>(a.ws_w);
  // pre-pass: layouts for TMA
  mk.mark(st);
  {
    dim3 grid((a.W + 31) / 32, (a.C + 31) / 32, a.N * a.H);
    k_nchw_to_nhwc<T><<<grid, 256, 0, st>>>(I, X, a.C, a.H, a.W);
    check_cuda(cudaGetLastError(), "nchw_to_nhwc");
    mk.mark(st);
    const int64_t wt = static_cast<int64_t>(a.F) * a.C * a.R * a.S;
    k_weights_rsfc<T><<<static_cast<unsigned>(std::min<int64_t>(1184, (wt + 255) / 256)), 256, 0, st>>>(
        K, Wt, a.F, a.C, a.R, a.S);
    check_cuda(cudaGetLastError(), "weights_rsfc");
    mk.mark(st);
    count_launch(2);
  }
  if (!a.maps_ready) {
    const int es = sizeof(T);
    const uint64_t dx[4] = {static_cast<uint64_t>(a.C), static_cast<uint64_t>(a.W), static_cast<uint64_t>(a.H),
                            static_cast<uint64_t>(a.N)};
    const uint64_t sx[3] = {static_cast<uint64_t>(a.C) * es, static_cast<uint64_t>(a.C) * a.W * es,
                            static_cast<uint64_t>(a.C) * a.W * a.H * es};
    const uint32_t bx[4] = {static_cast<uint32_t>(CK), static_cast<uint32_t>(kBW),
                            static_cast<uint32_t>(kBH + a.R - 1), 1};
    encode_map(&a.mapX, es == 2, es == 4, X, 4, dx, sx, bx);
    const uint64_t dw[3] = {static_cast<uint64_t>(a.C), static_cast<uint64_t>(a.F),
                            static_cast<uint64_t>(a.R) * a.S};
    const uint64_t sw[2] = {static_cast<uint64_t>(a.C) * es, static_cast<uint64_t>(a.C) * a.F * es};
    const uint32_t bw[3] = {static_cast<uint32_t>(CK), static_cast<uint32_t>(FN), 1};
    encode_map(&a.mapW, es == 2, es == 4, Wt, 3, dw, sw, bw);
    a.maps_ready = true;
  }
  const int tiles_h = (a.OH + kBH - 1) / kBH, tiles_w = (a.OW + kBW - 1) / kBW;
  const int total = a.N * tiles_h * tiles_w;
  const size_t budget = 227 * 1024 - 1024 - 256;
  int stages = static_cast<int>((budget - w_bytes) / a_bytes);
  if (stages >= 4) stages = 4;
  auto launch = [&](auto kern) {
    const size_t smem = w_bytes + static_cast<size_t>(stages) * a_bytes + 1024 + 256;
    check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
               "conv_tc smem attribute");
    const int grid = std::min(total, a.sms);
    static long long* trace = nullptr;  // developer knob: GENSOR_CONV_TRACE=<file> dumps clock64 marks
    static const char* trace_path = std::getenv("GENSOR_CONV_TRACE");
    if (trace_path && !trace) check_cuda(cudaMalloc(&trace, 148 * 64 * sizeof(long long) * 2), "trace");
    if (trace) check_cuda(cudaMemsetAsync(trace, 0, 148 * 64 * sizeof(long long) * 2, st), "trace");
    static const int xflags = std::getenv("GENSOR_CONV_XFLAGS") ? std::atoi(std::getenv("GENSOR_CONV_XFLAGS")) : 0;
    kern<<<grid, 192, smem, st>>>(a.mapX, a.mapW, O, a.F, a.C, a.R, a.S, a.OH, a.OW, tiles_h, tiles_w, total, trace,
                                  xflags);
    if (trace) {
      std::vector<long long> h(static_cast<size_t>(grid) * 64);
      check_cuda(cudaMemcpy(h.data(), trace, h.size() * sizeof(long long), cudaMemcpyDeviceToHost), "trace");
      if (FILE* f = std::fopen(trace_path, "w")) {
        for (int b = 0; b < grid; ++b) {
          for (int i = 0; i < 64; ++i) std::fprintf(f, "%lld%c", h[static_cast<size_t>(b) * 64 + i], i == 63 ? '\n' : ' ');
        }
        std::fclose(f);
      }
    }
    check_cuda(cudaGetLastError(), "conv_tc launch");
    mk.mark(st);
    count_launch();
  };
  if (stages >= 4)
    launch(k_conv_tc<T, FN, 4>);
  else if (stages == 3)
    launch(k_conv_tc<T, FN, 3>);
  else if (stages == 2)
    launch(k_conv_tc<T, FN, 2>);
  else
    throw Error(Code::Unsupported, "conv_tc: filter bank does not fit in shared memory");
}

}  // namespace

size_t conv_tc_smem_need(int C, int F, int R, int S, bool bf16) {
  const int CK = bf16 ? 64 : 32;
  int FN = 32;
  while (FN < F) FN *= 2;
  const size_t nck = (C + CK - 1) / CK;
  return static_cast<size_t>(R) * S * nck * FN * 128 + 2 * static_cast<size_t>((kBH + R - 1) * kBW * 128);
}

bool conv_tc_supported(int C, int F, int R, int S, int stride, bool bf16) {
  const int es = bf16 ? 2 : 4;
  return stride == 1 && F >= 1 && F <= 256 && (C * es) % 16 == 0 && R >= 1 && R <= 8 && S >= 1 &&
         conv_tc_smem_need(C, F, R, S, bf16) <= 227 * 1024 - 1024 - 256;
}

void launch_conv_tc(ConvTcArgs& a, const void* I, const void* K, void* O, cudaStream_t st, Marks& mk) {
  if (I != a.last_I || K != a.last_K) a.last_I = I, a.last_K = K;
  const float* i = static_cast<const float*>(I);
  const float* k = static_cast<const float*>(K);
  float* o = static_cast<float*>(O);
  int FN = 32;
  while (FN < a.F) FN *= 2;
  if (a.bf16) {
    switch (FN) {
      case 32: run_conv<__nv_bfloat16, 32>(a, i, k, o, st, mk); break;
      case 64: run_conv<__nv_bfloat16, 64>(a, i, k, o, st, mk); break;
      case 128: run_conv<__nv_bfloat16, 128>(a, i, k, o, st, mk); break;
      default: run_conv<__nv_bfloat16, 256>(a, i, k, o, st, mk); break;
    }
  } else {
    switch (FN) {
      case 32: run_conv<float, 32>(a, i, k, o, st, mk); break;
      case 64: run_conv<float, 64>(a, i, k, o, st, mk); break;
      case 128: run_conv<float, 128>(a, i, k, o, st, mk); break;
      default: run_conv<float, 256>(a, i, k, o, st, mk); break;
    }
  }
}

}  // namespace gb::dev
