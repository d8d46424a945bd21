// HBM-streaming kernel family ("stream" variant), instantiated from a constructed schedule:
//   gemv       y[m] = sum_n A[m][n] x[n]                       (op_spec.cpp:163-167; row sum: x = 1)
//   softmax    Y[m][n] = exp(X[m][n] - max_n X) / sum_n exp(.)  (extension op, no reference kind)
//   avgpool2d  O[p][h][w] = sum_{i,j} I[p][hS+i][wS+j] / F^2    (op_spec.cpp:190-193)
//   dwconv2d   O[n][c][h][w] = sum_{r,s} I[n][c][hS+r][wS+s] K[c][r][s]   (extension op)
// All four move every byte of HBM once; the design goal is bytes in flight, not FLOPs:
//   * persistent grid (SMs x resident CTAs), the schedule's level-1 spatial tile is the CTA's
//     work unit (rows for gemv/softmax, an output-row band of one plane for the window ops);
//   * gemv: one warp per row, 128-bit streaming loads (ld.global.cs) 8 deep per lane, fp64
//     accumulation of the exact fp32 products, warp-shuffle reduction;
//   * softmax: one CTA per row, the row held in registers (single HBM read), block max / sum
//     reductions by warp shuffles, 128-bit streaming stores;
//   * window ops: the input band of a unit is one contiguous HBM range, copied into shared memory
//     with 16 B cp.async (double-buffered: band u+1 streams in while band u is computed); each
//     thread computes a 4x4 output tile from a register patch, accumulating the reduce axes in the
//     interpreter's order (oracle/gensor_oracle.c) so integer inputs are
//     bit-exact; fp32 results of random inputs are within the stated tolerance.
#include <cuda_runtime.h>

#include <algorithm>
#include <stdint.h>

#include "../host/error.hpp"
#include "common.cuh"
#include "launch.h"
#include "tc_common.cuh"

namespace gb::dev {

namespace {

// ---- small PTX helpers ---------------------------------------------------------------------
__device__ __forceinline__ float4 ld_stream4(const float* p) {
  float4 v;
  asm volatile("ld.global.cs.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ void st_stream4(float* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(gmem)
               : "memory");
}

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(gmem)
               : "memory");
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// 1-D TMA bulk copy global -> shared (16 B aligned, size a multiple of 16), completion counted
// on an mbarrier's transaction count.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   tc::smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(tc::smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ---- gemv / row reduction ------------------------------------------------------------------
// A row is split over WPR warps (each warp streams an interleaved 512 B-granular share with D
// 128-bit loads in flight per lane); the CTA's 8 warps cover 8/WPR rows per step. Partial sums
// meet in shared memory and are added in a fixed order, so results are deterministic.
constexpr int kGemvThreads = 256;
constexpr int kGemvD = 8;

template <bool VEC>
__global__ void __launch_bounds__(kGemvThreads) k_gemv(const float* __restrict__ A, const float* __restrict__ x,
                                                       float* __restrict__ y, int64_t M, int64_t N,
                                                       int64_t rows_per_unit, int64_t units, int wpr) {
  __shared__ double red[kGemvThreads / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rows_per_step = (kGemvThreads / 32) / wpr;
  const int sub = warp / wpr, part = warp % wpr;
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    const int64_t r_end = min(M, (u + 1) * rows_per_unit);
    for (int64_t m0 = u * rows_per_unit; m0 < r_end; m0 += rows_per_step) {
      const int64_t m = m0 + sub;
      // D independent fp32 FMA chains per lane (one per load slot), combined in fp64: integer
      // inputs stay exact, random inputs keep ~1e-7 normwise error.
      float p[kGemvD];
#pragma unroll
      for (int d = 0; d < kGemvD; ++d) p[d] = 0.0f;
      if (m < r_end) {
        const float* row = A + m * N;
        if constexpr (VEC) {
          const int64_t nv = N >> 2;
          const float4* xv = reinterpret_cast<const float4*>(x);
          const int64_t step = 32 * wpr;
          int64_t i = part * 32 + lane;
          for (; i + (kGemvD - 1) * step < nv; i += kGemvD * step) {
            float4 a[kGemvD];
#pragma unroll
            for (int d = 0; d < kGemvD; ++d) a[d] = ld_stream4(row + 4 * (i + d * step));
#pragma unroll
            for (int d = 0; d < kGemvD; ++d) {
              const float4 b = __ldg(xv + i + d * step);
              p[d] = fmaf(a[d].x, b.x, p[d]);
              p[d] = fmaf(a[d].y, b.y, p[d]);
              p[d] = fmaf(a[d].z, b.z, p[d]);
              p[d] = fmaf(a[d].w, b.w, p[d]);
            }
          }
#pragma unroll
          for (int d = 0; d < kGemvD; ++d) {  // tail: at most D-1 more loads per lane
            const int64_t j = i + d * step;
            if (j < nv) {
              const float4 a = ld_stream4(row + 4 * j);
              const float4 b = __ldg(xv + j);
              p[d] = fmaf(a.x, b.x, p[d]);
              p[d] = fmaf(a.y, b.y, p[d]);
              p[d] = fmaf(a.z, b.z, p[d]);
              p[d] = fmaf(a.w, b.w, p[d]);
            }
          }
        } else {
          for (int64_t n = part * 32 + lane; n < N; n += kGemvD * 32 * wpr) {
#pragma unroll
            for (int d = 0; d < kGemvD; ++d) {
              const int64_t j = n + static_cast<int64_t>(d) * 32 * wpr;
              if (j < N) p[d] = fmaf(__ldcs(row + j), __ldg(x + j), p[d]);
            }
          }
        }
      }
      double acc = 0.0;
#pragma unroll
      for (int d = 0; d < kGemvD; ++d) acc += static_cast<double>(p[d]);
      acc = warp_sum(acc);
      if (wpr == 1) {
        if (lane == 0 && m < r_end) y[m] = static_cast<float>(acc);
      } else {
        if (lane == 0) red[warp] = acc;
        __syncthreads();
        if (threadIdx.x < rows_per_step && m0 + threadIdx.x < r_end) {
          double t = 0.0;
          for (int q = 0; q < wpr; ++q) t += red[threadIdx.x * wpr + q];
          y[m0 + threadIdx.x] = static_cast<float>(t);
        }
        __syncthreads();
      }
    }
  }
}

// TMA-bulk gemv: CTA b owns a contiguous range of row units; a producer warp streams one row per
// stage (cp.async.bulk, mbarrier transaction counts) into a ring of `stages` (a multiple of 8) row
// buffers; consumer
// warp w reduces rows i = w (mod 8) of the range against x (staged once in shared memory) — 8 rows
// in flight per CTA, each reduced by one warp in a fixed order (deterministic) — and releases the
// stage as soon as its row is done.
constexpr int kGemvBulkConsumers = 8;

__global__ void __launch_bounds__(32 * (kGemvBulkConsumers + 1), 1)
    k_gemv_bulk(const float* __restrict__ A, const float* __restrict__ x, float* __restrict__ y, int64_t M, int64_t N,
                int64_t rows_per_unit, int64_t units, int stages) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t row_bytes = static_cast<uint32_t>(N * 4);
  float* xs = reinterpret_cast<float*>(smem_raw);
  float* ring = xs + N;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + static_cast<int64_t>(stages) * N);
  uint64_t* empty = full + stages;
  uint64_t* xbar = empty + stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t u0 = units * blockIdx.x / gridDim.x, u1 = units * (blockIdx.x + 1) / gridDim.x;
  const int64_t r0 = min(M, u0 * rows_per_unit), r1 = min(M, u1 * rows_per_unit);
  const int64_t rows = r1 - r0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&empty[i], 1);
    }
    tc::mbar_init(xbar, 1);
    tc::fence_barrier_init();
  }
  __syncthreads();
  if (warp == kGemvBulkConsumers) {  // producer
    if (lane == 0) {
      tc::mbar_arrive_expect_tx(xbar, row_bytes);
      bulk_g2s(xs, x, row_bytes, xbar);
      for (int64_t i = 0; i < rows; ++i) {
        const int st = static_cast<int>(i % stages);
        if (i >= stages) tc::mbar_wait(&empty[st], static_cast<uint32_t>(((i / stages) & 1) ^ 1));
        tc::mbar_arrive_expect_tx(&full[st], row_bytes);
        bulk_g2s(ring + static_cast<int64_t>(st) * N, A + (r0 + i) * N, row_bytes, &full[st]);
      }
    }
    return;
  }
  tc::mbar_wait(xbar, 0);
  const int64_t nv = N >> 2;
  const float4* xv = reinterpret_cast<const float4*>(xs);
  for (int64_t i = warp; i < rows; i += kGemvBulkConsumers) {
    const int st = static_cast<int>(i % stages);
    tc::mbar_wait(&full[st], static_cast<uint32_t>((i / stages) & 1));
    const float4* rv = reinterpret_cast<const float4*>(ring + static_cast<int64_t>(st) * N);
    // 4 independent fp32 FMA chains per lane, combined in fp64
    float p[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    int64_t j = lane;
    for (; j + 3 * 32 < nv; j += 4 * 32) {
#pragma unroll
      for (int d = 0; d < 4; ++d) {
        const float4 a = rv[j + d * 32], b = xv[j + d * 32];
        p[d] = fmaf(a.x, b.x, p[d]);
        p[d] = fmaf(a.y, b.y, p[d]);
        p[d] = fmaf(a.z, b.z, p[d]);
        p[d] = fmaf(a.w, b.w, p[d]);
      }
    }
    for (; j < nv; j += 32) {
      const float4 a = rv[j], b = xv[j];
      p[0] = fmaf(a.x, b.x, p[0]);
      p[0] = fmaf(a.y, b.y, p[0]);
      p[0] = fmaf(a.z, b.z, p[0]);
      p[0] = fmaf(a.w, b.w, p[0]);
    }
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(&empty[st]);  // the row is in registers: free the stage
    const double v = warp_sum((static_cast<double>(p[0]) + static_cast<double>(p[1])) +
                              (static_cast<double>(p[2]) + static_cast<double>(p[3])));
    if (lane == 0) y[r0 + i] = static_cast<float>(v);
  }
}

// ---- softmax ---------------------------------------------------------------------------------
constexpr int kSoftmaxThreads = 256;

__device__ __forceinline__ float block_max(float v, float* red) {
  v = warp_max(v);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();  // red[] reuse across calls
  if (lane == 0) red[warp] = v;
  __syncthreads();
  float r = red[0];
  for (int w = 1; w < kSoftmaxThreads / 32; ++w) r = fmaxf(r, red[w]);
  return r;
}

__device__ __forceinline__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double r = red[0];
  for (int w = 1; w < kSoftmaxThreads / 32; ++w) r += red[w];
  return r;
}

// exp(x - mx) with the subtraction made exact by Knuth's TwoSum (d = hi + lo exactly), then
// exp(hi + lo) = exp(hi) * (1 + lo): the argument's rounding never reaches the result.
__device__ __forceinline__ float exp_shift(float x, float mx) {
  const float hi = __fsub_rn(x, mx);
  const float bb = __fsub_rn(hi, x);
  const float lo = __fadd_rn(__fsub_rn(x, __fsub_rn(hi, bb)), __fsub_rn(-mx, bb));
  const float e = expf(hi);
  return fmaf(e, lo, e);
}

// Single HBM pass: row in registers (VPT float4 per thread), N <= 4 * VPT * 256.
template <int VPT>
__global__ void __launch_bounds__(kSoftmaxThreads) k_softmax_reg(const float* __restrict__ X, float* __restrict__ Y,
                                                                 int64_t M, int64_t N, int64_t rows_per_unit,
                                                                 int64_t units) {
  __shared__ double red_d[kSoftmaxThreads / 32];
  __shared__ float red_f[kSoftmaxThreads / 32];
  const int64_t nv = N >> 2;
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    const int64_t r_end = min(M, (u + 1) * rows_per_unit);
    for (int64_t m = u * rows_per_unit; m < r_end; ++m) {
      const float* row = X + m * N;
      float4 v[VPT];
      float mx = -INFINITY;
#pragma unroll
      for (int q = 0; q < VPT; ++q) {
        const int64_t i = threadIdx.x + static_cast<int64_t>(q) * kSoftmaxThreads;
        if (i < nv) {
          v[q] = ld_stream4(row + 4 * i);
          mx = fmaxf(mx, fmaxf(fmaxf(v[q].x, v[q].y), fmaxf(v[q].z, v[q].w)));
        }
      }
      mx = block_max(mx, red_f);
      float ts = 0.0f;  // <= 4*VPT positive terms per thread in fp32, then fp64 across the block
#pragma unroll
      for (int q = 0; q < VPT; ++q) {
        const int64_t i = threadIdx.x + static_cast<int64_t>(q) * kSoftmaxThreads;
        if (i < nv) {
          v[q].x = exp_shift(v[q].x, mx);
          v[q].y = exp_shift(v[q].y, mx);
          v[q].z = exp_shift(v[q].z, mx);
          v[q].w = exp_shift(v[q].w, mx);
          ts += (v[q].x + v[q].y) + (v[q].z + v[q].w);
        }
      }
      const double s = block_sum(static_cast<double>(ts), red_d);
      const float inv = static_cast<float>(1.0 / s);
      float* out = Y + m * N;
#pragma unroll
      for (int q = 0; q < VPT; ++q) {
        const int64_t i = threadIdx.x + static_cast<int64_t>(q) * kSoftmaxThreads;
        if (i < nv)
          st_stream4(out + 4 * i, make_float4(v[q].x * inv, v[q].y * inv, v[q].z * inv, v[q].w * inv));
      }
    }
  }
}

// Short rows (N <= 32 * 4 * VPL): one warp per row, the row in registers, warp-shuffle max and
// fp64 sum — no shared memory, no block barriers (GPT-2 attention rows, N = 512).
template <int VPL>
__global__ void __launch_bounds__(kSoftmaxThreads) k_softmax_warp(const float* __restrict__ X, float* __restrict__ Y,
                                                                  int64_t M, int64_t N, int64_t rows_per_unit,
                                                                  int64_t units) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nv = N >> 2;
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    const int64_t r_end = min(M, (u + 1) * rows_per_unit);
    constexpr int64_t kStep = kSoftmaxThreads / 32;
    // software pipeline: the next row of this warp is in flight while the current one is reduced,
    // exponentiated and stored
    float4 nxt[VPL];
    auto load_row = [&](int64_t m, float4 (&dst)[VPL]) {
#pragma unroll
      for (int q = 0; q < VPL; ++q) {
        const int64_t i = lane + 32 * q;
        dst[q] = (m < r_end && i < nv) ? ld_stream4(X + m * N + 4 * i) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
    load_row(u * rows_per_unit + warp, nxt);
    for (int64_t m = u * rows_per_unit + warp; m < r_end; m += kStep) {
      float4 v[VPL];
#pragma unroll
      for (int q = 0; q < VPL; ++q) v[q] = nxt[q];
      load_row(m + kStep, nxt);
      float mx = -INFINITY;
#pragma unroll
      for (int q = 0; q < VPL; ++q) {
        const int64_t i = lane + 32 * q;
        if (i < nv) mx = fmaxf(mx, fmaxf(fmaxf(v[q].x, v[q].y), fmaxf(v[q].z, v[q].w)));
      }
      mx = warp_max(mx);
      float ts = 0.0f;
#pragma unroll
      for (int q = 0; q < VPL; ++q) {
        const int64_t i = lane + 32 * q;
        if (i < nv) {
          v[q].x = exp_shift(v[q].x, mx);
          v[q].y = exp_shift(v[q].y, mx);
          v[q].z = exp_shift(v[q].z, mx);
          v[q].w = exp_shift(v[q].w, mx);
          ts += (v[q].x + v[q].y) + (v[q].z + v[q].w);
        }
      }
      const float inv = static_cast<float>(1.0 / warp_sum(static_cast<double>(ts)));
      float* out = Y + m * N;
#pragma unroll
      for (int q = 0; q < VPL; ++q) {
        const int64_t i = lane + 32 * q;
        if (i < nv) st_stream4(out + 4 * i, make_float4(v[q].x * inv, v[q].y * inv, v[q].z * inv, v[q].w * inv));
      }
    }
  }
}

// Any N (unaligned or longer than the register budget): max pass, sum pass, write pass.
__global__ void __launch_bounds__(kSoftmaxThreads) k_softmax_any(const float* __restrict__ X, float* __restrict__ Y,
                                                                 int64_t M, int64_t N, int64_t rows_per_unit,
                                                                 int64_t units) {
  __shared__ double red_d[kSoftmaxThreads / 32];
  __shared__ float red_f[kSoftmaxThreads / 32];
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    const int64_t r_end = min(M, (u + 1) * rows_per_unit);
    for (int64_t m = u * rows_per_unit; m < r_end; ++m) {
      const float* row = X + m * N;
      float mx = -INFINITY;
      for (int64_t n = threadIdx.x; n < N; n += kSoftmaxThreads) mx = fmaxf(mx, row[n]);
      mx = block_max(mx, red_f);
      double s = 0.0;
      for (int64_t n = threadIdx.x; n < N; n += kSoftmaxThreads) s += static_cast<double>(exp_shift(row[n], mx));
      s = block_sum(s, red_d);
      const double inv = 1.0 / s;
      for (int64_t n = threadIdx.x; n < N; n += kSoftmaxThreads)
        Y[m * N + n] = static_cast<float>(static_cast<double>(exp_shift(row[n], mx)) * inv);
    }
  }
}

// ---- window ops: avgpool2d / dwconv2d --------------------------------------------------------
// outputs per thread: a column strip of kTH rows (launch.h); adjacent lanes own adjacent columns,
// so every shared-memory read of a warp is conflict-free (stride 1)
constexpr int kTH = kWinTH, kTW = kWinTW;
constexpr int kWinStages = 3;   // band staging buffers per CTA

// Band geometry of unit u. Plane/row offsets stay 64-bit; everything inside a band is 32-bit.
struct Band {
  int64_t g0;      // element offset of the band's first input row
  int64_t out0;    // element offset of the band's first output row
  int32_t oh0;     // first output row
  int32_t len;     // input elements in the band
  int32_t ph;      // smem phase: sm[ph + i] = in[g0 + i]
  int32_t plane;
};

__device__ __forceinline__ Band band_of(const StreamWinArgs& a, int64_t u) {
  Band b;
  const int64_t plane = u / a.bands;
  const int32_t band = static_cast<int32_t>(u - plane * a.bands);
  b.plane = static_cast<int32_t>(plane);
  b.oh0 = band * a.band_rows;
  const int32_t ih0 = b.oh0 * a.stride;
  const int32_t rows = min(a.in_rows, static_cast<int32_t>(a.H) - ih0);
  b.g0 = plane * a.H * a.W + static_cast<int64_t>(ih0) * a.W;
  b.out0 = plane * a.OH * a.OW + static_cast<int64_t>(b.oh0) * a.OW;
  b.len = rows * static_cast<int32_t>(a.W);
  b.ph = static_cast<int32_t>(b.g0 & 3);
  return b;
}

__device__ __forceinline__ void issue_band(const StreamWinArgs& a, const float* __restrict__ in, float* buf,
                                           const Band& b) {
  const float* src = in + b.g0;
  float* dst = buf + b.ph;
  const int nt = blockDim.x;
  if (a.vec) {
    const int head = min((4 - b.ph) & 3, b.len);
    const int body = (b.len - head) >> 2;
    for (int i = threadIdx.x; i < head; i += nt) cp_async4(dst + i, src + i);
    for (int i = threadIdx.x; i < body; i += nt) cp_async16(dst + head + 4 * i, src + head + 4 * i);
    for (int i = head + 4 * body + threadIdx.x; i < b.len; i += nt) cp_async4(dst + i, src + i);
  } else {
    for (int i = threadIdx.x; i < b.len; i += nt) cp_async4(dst + i, src + i);
  }
}

// Correctly rounded acc / F^2 (the oracle divides the window sum by the true F^2,
// oracle_interpret): Markstein's sequence q0 = acc*y, r = acc - F^2*q0 (exact by FMA),
// q = q0 + r*y with y = RN(1/F^2) is correctly rounded for normal results (checked against exact
// rational division for F^2 in {9, 25, 49}); tiny / non-finite sums take the IEEE division.
__device__ __noinline__ float div_window_slow(float acc, float d) { return __fdiv_rn(acc, d); }

__device__ __forceinline__ float div_window(float acc, float d, float y) {
  const float q0 = acc * y;
  const float r = fmaf(-q0, d, acc);
  float q = fmaf(r, y, q0);
  // Out-of-line IEEE division only where the Markstein step could over/underflow; keeping it a
  // real (not if-converted) branch leaves 3 FMA-pipe ops per output on the hot path.
  if (__builtin_expect(!(fabsf(acc) > 1e-30f && fabsf(acc) < 1e30f), 0)) q = div_window_slow(acc, d);
  return q;
}

template <bool DW>
__device__ __forceinline__ void store_row(const StreamWinArgs& a, float* orow, int ox, const float (&acc)[kTW]) {
  float o[kTW];
  const float d = static_cast<float>(a.divisor), y = __frcp_rn(d);
#pragma unroll
  for (int j = 0; j < kTW; ++j) o[j] = DW ? acc[j] : div_window(acc[j], d, y);
  if constexpr (kTW == 2) {
    if (a.vec_out && ox + 2 <= a.OW) {
      __stcs(reinterpret_cast<float2*>(orow), make_float2(o[0], o[1]));
      return;
    }
  }
#pragma unroll
  for (int j = 0; j < kTW; ++j)
    if (ox + j < a.OW) __stcs(orow + j, o[j]);
}

// 3x3 window fast path. The (kTH-1)*STRIDE+3 x (kTW-1)*STRIDE+3 input patch is loaded into
// registers first (independent shared loads, 64-bit pairs when rows are 8 B aligned), then every
// output accumulates its 9 taps in the interpreter's order — r-major (r outer, s inner: the
// lexicographic order) or s-major — with the kTH*kTW outputs as independent FMA chains.
template <bool DW, int STRIDE, bool SMAJOR>
__device__ __forceinline__ void tile3x3(const StreamWinArgs& a, const float* band, bool pairs, const float (&w)[9],
                                        float* __restrict__ out_band, int oy, int ox, int rows_out) {
  constexpr int PH = (kTH - 1) * STRIDE + 3, PW = (kTW - 1) * STRIDE + 3;
  const int W = static_cast<int>(a.W);
  const float* src = band + (oy * STRIDE) * W + ox * STRIDE;
  float p[PH][PW];
  if (pairs) {  // src is 8 B aligned on every row
#pragma unroll
    for (int y = 0; y < PH; ++y) {
#pragma unroll
      for (int x = 0; x + 1 < PW; x += 2) {
        const float2 v = *reinterpret_cast<const float2*>(src + y * W + x);
        p[y][x] = v.x;
        p[y][x + 1] = v.y;
      }
      if constexpr (PW % 2) p[y][PW - 1] = src[y * W + PW - 1];
    }
  } else {
#pragma unroll
    for (int y = 0; y < PH; ++y)
#pragma unroll
      for (int x = 0; x < PW; ++x) p[y][x] = src[y * W + x];
  }
  float acc[kTH][kTW];
#pragma unroll
  for (int i = 0; i < kTH; ++i)
#pragma unroll
    for (int j = 0; j < kTW; ++j) acc[i][j] = 0.0f;
#pragma unroll
  for (int q = 0; q < 9; ++q) {
    const int r = SMAJOR ? q % 3 : q / 3;
    const int sx = SMAJOR ? q / 3 : q % 3;
#pragma unroll
    for (int i = 0; i < kTH; ++i)
#pragma unroll
      for (int j = 0; j < kTW; ++j) {
        const float v = p[i * STRIDE + r][j * STRIDE + sx];
        if constexpr (DW)
          acc[i][j] = fmaf(v, w[r * 3 + sx], acc[i][j]);
        else
          acc[i][j] += v;
      }
  }
  const int OW = static_cast<int>(a.OW);
#pragma unroll
  for (int i = 0; i < kTH; ++i) {
    if (oy + i >= rows_out) break;
    store_row<DW>(a, out_band + (oy + i) * OW + ox, ox, acc[i]);
  }
}

// Generic path: any window / stride / interpreter order (order list from the host).
template <bool DW>
__device__ __forceinline__ void tile_generic(const StreamWinArgs& a, const float* band,
                                             const float* __restrict__ wplane, float* __restrict__ out_band, int oy0,
                                             int ox0, int rows_out) {
  const int W = static_cast<int>(a.W), OW = static_cast<int>(a.OW);
  for (int i = 0; i < kTH; ++i) {
    const int oy = oy0 + i;
    if (oy >= rows_out) break;
    for (int j = 0; j < kTW; ++j) {
      const int ox = ox0 + j;
      if (ox >= OW) break;
      float acc = 0.0f;
      for (int q = 0; q < a.n_order; ++q) {
        const int r = a.order[q] >> 4, sx = a.order[q] & 15;
        const float v = band[(oy * a.stride + r) * W + ox * a.stride + sx];
        if constexpr (DW)
          acc = fmaf(v, wplane[r * a.S + sx], acc);
        else
          acc += v;
      }
      out_band[oy * OW + ox] = DW ? acc : __fdiv_rn(acc, static_cast<float>(a.divisor));
    }
  }
}

// MODE: 0 generic, 1 3x3 s1 r-major, 2 3x3 s1 s-major, 3 3x3 s2 r-major, 4 3x3 s2 s-major.
// Persistent CTAs; band u+gridDim streams into the other buffer while band u is computed.
template <bool DW, int MODE>
__global__ void __launch_bounds__(256) k_window(const StreamWinArgs a, const float* __restrict__ in,
                                                const float* __restrict__ wts, float* __restrict__ out) {
  extern __shared__ __align__(16) float sm[];
  // kWinStages-deep ring: the bands of the next kWinStages-1 units stream in while one computes
  const int64_t g = gridDim.x;
#pragma unroll
  for (int k = 0; k < kWinStages - 1; ++k) {
    const int64_t uk = blockIdx.x + k * g;
    if (uk < a.units) issue_band(a, in, sm + k * a.buf_floats, band_of(a, uk));
    cp_async_commit();
  }
  int cur = 0;
  const int tiles_x = static_cast<int>((a.OW + kTW - 1) / kTW);
  const int tiles = tiles_x * ((a.band_rows + kTH - 1) / kTH);
  for (int64_t u = blockIdx.x; u < a.units; u += g) {
    const int64_t nu = u + (kWinStages - 1) * g;
    const int nb = cur == 0 ? kWinStages - 1 : cur - 1;  // the slot freed last iteration
    if (nu < a.units) issue_band(a, in, sm + nb * a.buf_floats, band_of(a, nu));
    cp_async_commit();
    cp_async_wait<kWinStages - 1>();
    __syncthreads();
    const Band b = band_of(a, u);
    // rows past the plane's last output row belong to no output of this band
    const int rows_out = min(a.band_rows, static_cast<int32_t>(a.OH) - b.oh0);
    const float* band = sm + cur * a.buf_floats + b.ph;
    const bool pairs = (a.W % 2 == 0) && (b.ph % 2 == 0);  // 8 B aligned patch rows (ox*STRIDE even)
    float* out_band = out + b.out0;
    const int c = static_cast<int>(b.plane % a.C);
    float w[9];
    if constexpr (DW && MODE != 0) {
#pragma unroll
      for (int q = 0; q < 9; ++q) w[q] = __ldg(wts + c * 9 + q);
    }
    for (int t = threadIdx.x; t < tiles; t += blockDim.x) {
      const int oy = (t / tiles_x) * kTH, ox = (t % tiles_x) * kTW;
      if (oy >= rows_out) continue;
      if constexpr (MODE == 1) tile3x3<DW, 1, false>(a, band, pairs, w, out_band, oy, ox, rows_out);
      else if constexpr (MODE == 2) tile3x3<DW, 1, true>(a, band, pairs, w, out_band, oy, ox, rows_out);
      else if constexpr (MODE == 3) tile3x3<DW, 2, false>(a, band, pairs, w, out_band, oy, ox, rows_out);
      else if constexpr (MODE == 4) tile3x3<DW, 2, true>(a, band, pairs, w, out_band, oy, ox, rows_out);
      else tile_generic<DW>(a, band, DW ? wts + static_cast<int64_t>(c) * a.R * a.S : nullptr, out_band, oy, ox, rows_out);
    }
    __syncthreads();  // this buffer is refilled next iteration
    cur = cur + 1 == kWinStages ? 0 : cur + 1;
  }
  cp_async_wait<0>();
}

// TMA-bulk window kernel: a producer warp streams each band's input range — widened to 16 B
// boundaries, so one cp.async.bulk moves it and sm[ph + i] = in[g0 + i] still holds — into a
// kWinBulkStages ring; consumer warps compute 4x4 tiles and release the stage per warp.
constexpr int kWinBulkStages = 4;

template <bool DW, int MODE>
__global__ void __launch_bounds__(288) k_window_bulk(const StreamWinArgs a, const float* __restrict__ in,
                                                     const float* __restrict__ wts, float* __restrict__ out,
                                                     int64_t total_in) {
  extern __shared__ __align__(16) float sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + kWinBulkStages * a.buf_floats);
  uint64_t* empty = full + kWinBulkStages;
  const int cwarps = (blockDim.x >> 5) - 1;
  const int consumers = cwarps * 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t g = gridDim.x;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kWinBulkStages; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&empty[i], cwarps);
    }
    tc::fence_barrier_init();
  }
  __syncthreads();
  if (warp == cwarps) {  // producer
    if (lane == 0) {
      const int64_t aligned_end = total_in & ~int64_t(3);
      int k = 0;
      for (int64_t u = blockIdx.x; u < a.units; u += g, ++k) {
        const int st = k % kWinBulkStages;
        tc::mbar_wait(&empty[st], ((k / kWinBulkStages) & 1) ^ 1);
        const Band b = band_of(a, u);
        const int64_t lo = b.g0 - b.ph;                                   // 16 B aligned
        const int64_t hi = min((b.g0 + b.len + 3) & ~int64_t(3), aligned_end);
        float* dst = sm + st * a.buf_floats;
        // tail past the last aligned 16 B of the whole tensor (last band only): plain loads
        for (int64_t i = hi; i < b.g0 + b.len; ++i) dst[i - lo] = in[i];
        tc::mbar_arrive_expect_tx(&full[st], static_cast<uint32_t>((hi - lo) * 4));
        if (hi > lo) bulk_g2s(dst, in + lo, static_cast<uint32_t>((hi - lo) * 4), &full[st]);
      }
    }
    return;
  }
  const int tiles_x = static_cast<int>((a.OW + kTW - 1) / kTW);
  const int tiles = tiles_x * ((a.band_rows + kTH - 1) / kTH);
  int k = 0;
  for (int64_t u = blockIdx.x; u < a.units; u += g, ++k) {
    const int st = k % kWinBulkStages;
    tc::mbar_wait(&full[st], (k / kWinBulkStages) & 1);
    const Band b = band_of(a, u);
    const int rows_out = min(a.band_rows, static_cast<int32_t>(a.OH) - b.oh0);
    const float* band = sm + st * a.buf_floats + b.ph;
    const bool pairs = (a.W % 2 == 0) && (b.ph % 2 == 0);  // 8 B aligned patch rows (ox*STRIDE even)
    float* out_band = out + b.out0;
    const int c = static_cast<int>(b.plane % a.C);
    float w[9];
    if constexpr (DW && MODE != 0) {
#pragma unroll
      for (int q = 0; q < 9; ++q) w[q] = __ldg(wts + c * 9 + q);
    }
    for (int t = threadIdx.x; t < tiles; t += consumers) {
      const int oy = (t / tiles_x) * kTH, ox = (t % tiles_x) * kTW;
      if (oy >= rows_out) continue;
      if constexpr (MODE == 1) tile3x3<DW, 1, false>(a, band, pairs, w, out_band, oy, ox, rows_out);
      else if constexpr (MODE == 2) tile3x3<DW, 1, true>(a, band, pairs, w, out_band, oy, ox, rows_out);
      else if constexpr (MODE == 3) tile3x3<DW, 2, false>(a, band, pairs, w, out_band, oy, ox, rows_out);
      else if constexpr (MODE == 4) tile3x3<DW, 2, true>(a, band, pairs, w, out_band, oy, ox, rows_out);
      else tile_generic<DW>(a, band, DW ? wts + static_cast<int64_t>(c) * a.R * a.S : nullptr, out_band, oy, ox, rows_out);
    }
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(&empty[st]);
  }
}

// Global window (OH = OW = 1: the window covers the whole plane, e.g. ResNet's final 7x7 pool):
// planes are contiguous, so a CTA stages kGlobalPlanes whole planes with coalesced loads and each
// thread reduces one plane from shared memory in the interpreter's order (odd plane pitch in
// words when H*W is odd keeps the per-thread reads conflict-free).
constexpr int kGlobalPlanes = 256;

template <bool DW>
__global__ void __launch_bounds__(kGlobalPlanes) k_window_global(const StreamWinArgs a, const float* __restrict__ in,
                                                                 const float* __restrict__ wts,
                                                                 float* __restrict__ out) {
  extern __shared__ float pl[];
  const int hw = static_cast<int>(a.H * a.W);
  const float dv = static_cast<float>(a.divisor), y = __frcp_rn(dv);
  for (int64_t g0 = static_cast<int64_t>(blockIdx.x) * kGlobalPlanes; g0 < a.planes;
       g0 += static_cast<int64_t>(gridDim.x) * kGlobalPlanes) {
    const int np = static_cast<int>(min(static_cast<int64_t>(kGlobalPlanes), a.planes - g0));
    const float* src = in + g0 * hw;
    __syncthreads();
    for (int i = threadIdx.x; i < np * hw; i += kGlobalPlanes) pl[i] = __ldg(src + i);
    __syncthreads();
    if (threadIdx.x < np) {
      const float* p = pl + threadIdx.x * hw;
      const int64_t plane = g0 + threadIdx.x;
      const int c = static_cast<int>(plane % a.C);
      float acc = 0.0f;
      for (int q = 0; q < a.n_order; ++q) {
        const int r = a.order[q] >> 4, sx = a.order[q] & 15;
        const float v = p[r * a.W + sx];
        if constexpr (DW)
          acc = fmaf(v, __ldg(wts + c * a.R * a.S + r * a.S + sx), acc);
        else
          acc += v;
      }
      out[plane] = DW ? acc : div_window(acc, dv, y);
    }
  }
}

template <bool DW, int MODE>
void run_window(const StreamWinArgs& a, const void* in, const void* w, void* out, cudaStream_t st) {
  const int64_t total_in = a.planes * a.H * a.W;
  int per_sm = 0;
  if (a.vec) {  // 16 B aligned input: TMA bulk band loads
    auto kern = k_window_bulk<DW, MODE>;
    const size_t smem = kWinBulkStages * (a.buf_floats * sizeof(float) + 16);
    set_smem_attr(kern, static_cast<int>(smem), "window smem attribute");
    const int threads = a.threads + 32;
    check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem), "window occupancy");
    const int64_t grid = std::min<int64_t>(a.units, static_cast<int64_t>(std::max(1, per_sm)) * a.sms);
    kern<<<static_cast<unsigned>(grid), threads, smem, st>>>(a, static_cast<const float*>(in),
                                                           static_cast<const float*>(w), static_cast<float*>(out),
                                                           total_in);
  } else {  // 4 B aligned input: per-thread cp.async staging
    auto kern = k_window<DW, MODE>;
    const size_t smem = kWinStages * a.buf_floats * sizeof(float);
    set_smem_attr(kern, static_cast<int>(smem), "window smem attribute");
    check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, a.threads, smem), "window occupancy");
    const int64_t grid = std::min<int64_t>(a.units, static_cast<int64_t>(std::max(1, per_sm)) * a.sms);
    kern<<<static_cast<unsigned>(grid), a.threads, smem, st>>>(a, static_cast<const float*>(in),
                                                             static_cast<const float*>(w), static_cast<float*>(out));
  }
  check_cuda(cudaGetLastError(), "window launch");
  count_launch();
}

template <typename K>
int64_t persistent_grid(K kern, int threads, size_t smem, int sms, int64_t units) {
  int per_sm = 0;
  check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem), "occupancy");
  return std::max<int64_t>(1, std::min<int64_t>(units, static_cast<int64_t>(std::max(1, per_sm)) * sms));
}

}  // namespace

void launch_stream(const StreamArgs& a, const void* in0, const void* in1, void* out, cudaStream_t st) {
  switch (a.kind) {
    case StreamKind::Gemv: {
      const bool vec = (a.N % 4 == 0) && (reinterpret_cast<uintptr_t>(in0) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(in1) % 16 == 0);
      const int64_t units = (a.M + a.rows_per_unit - 1) / a.rows_per_unit;
      auto go = [&](auto kern) {
        const int64_t grid = persistent_grid(kern, kGemvThreads, 0, a.sms, units);
        kern<<<static_cast<unsigned>(grid), kGemvThreads, 0, st>>>(static_cast<const float*>(in0),
                                                                   static_cast<const float*>(in1),
                                                                   static_cast<float*>(out), a.M, a.N,
                                                                   a.rows_per_unit, units, a.wpr);
      };
      const size_t row_bytes = static_cast<size_t>(a.N) * 4;
      const size_t budget = 200 * 1024;  // x + ring + 2 barriers per stage
      // stages: a multiple of the 8 consumer warps, so stage s is always consumed by warp s % 8 and
      // a warp never waits on a fill more than one mbarrier phase ahead of the last one it consumed
      int stages = static_cast<int>(std::min<size_t>(16, (budget - std::min(budget, row_bytes + 16)) / (row_bytes + 16)));
      stages = stages / kGemvBulkConsumers * kGemvBulkConsumers;
      if (vec && a.N >= 256 && stages >= kGemvBulkConsumers) {
        const size_t smem = row_bytes * (stages + 1) + static_cast<size_t>(stages) * 16 + 16;
        set_smem_attr(k_gemv_bulk, static_cast<int>(smem), "gemv smem attribute");
        const int64_t grid = std::min<int64_t>(units, a.sms);
        k_gemv_bulk<<<static_cast<unsigned>(grid), 32 * (kGemvBulkConsumers + 1), smem, st>>>(
            static_cast<const float*>(in0), static_cast<const float*>(in1), static_cast<float*>(out), a.M, a.N,
            a.rows_per_unit, units, stages);
      } else if (vec) {
        go(k_gemv<true>);
      } else {
        go(k_gemv<false>);
      }
      check_cuda(cudaGetLastError(), "gemv launch");
      count_launch();
      return;
    }
    case StreamKind::Softmax: {
      const bool vec = (a.N % 4 == 0) && (reinterpret_cast<uintptr_t>(in0) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(out) % 16 == 0);
      const int64_t units = (a.M + a.rows_per_unit - 1) / a.rows_per_unit;
      const int64_t nv = a.N / 4;
      auto go = [&](auto kern) {
        const int64_t grid = persistent_grid(kern, kSoftmaxThreads, 0, a.sms, units);
        kern<<<static_cast<unsigned>(grid), kSoftmaxThreads, 0, st>>>(static_cast<const float*>(in0),
                                                                      static_cast<float*>(out), a.M, a.N,
                                                                      a.rows_per_unit, units);
      };
      if (vec && nv <= 32 * 2) go(k_softmax_warp<2>);
      else if (vec && nv <= 32 * 4) go(k_softmax_warp<4>);
      else if (vec && nv <= 32 * 8) go(k_softmax_warp<8>);
      else if (vec && nv <= kSoftmaxThreads * 1) go(k_softmax_reg<1>);
      else if (vec && nv <= kSoftmaxThreads * 2) go(k_softmax_reg<2>);
      else if (vec && nv <= kSoftmaxThreads * 4) go(k_softmax_reg<4>);
      else if (vec && nv <= kSoftmaxThreads * 8) go(k_softmax_reg<8>);
      else go(k_softmax_any);
      check_cuda(cudaGetLastError(), "softmax launch");
      count_launch();
      return;
    }
    case StreamKind::AvgPool:
    case StreamKind::DwConv: {
      StreamWinArgs w = a.win;
      w.vec = reinterpret_cast<uintptr_t>(in0) % 16 == 0;
      w.vec_out = (w.OW % 2 == 0) && (reinterpret_cast<uintptr_t>(out) % 8 == 0);
      const bool dw = a.kind == StreamKind::DwConv;
      if (w.OH == 1 && w.OW == 1 && w.H * w.W <= 128) {  // global window over small planes
        const size_t smem = static_cast<size_t>(kGlobalPlanes) * w.H * w.W * sizeof(float);
        const int64_t groups = (w.planes + kGlobalPlanes - 1) / kGlobalPlanes;
        const unsigned grid = static_cast<unsigned>(std::min<int64_t>(groups, static_cast<int64_t>(w.sms) * 4));
        auto kern = dw ? k_window_global<true> : k_window_global<false>;
        set_smem_attr(kern, static_cast<int>(smem), "global window smem attribute");
        kern<<<grid, kGlobalPlanes, smem, st>>>(w, static_cast<const float*>(in0), static_cast<const float*>(in1),
                                                static_cast<float*>(out));
        check_cuda(cudaGetLastError(), "global window launch");
        count_launch();
        return;
      }
      int mode = 0;
      if (w.R == 3 && w.S == 3 && (w.stride == 1 || w.stride == 2) && w.order_kind != 0)
        mode = (w.stride == 1 ? 1 : 3) + (w.order_kind == 2 ? 1 : 0);
      if (dw) {
        switch (mode) {
          case 1: run_window<true, 1>(w, in0, in1, out, st); break;
          case 2: run_window<true, 2>(w, in0, in1, out, st); break;
          case 3: run_window<true, 3>(w, in0, in1, out, st); break;
          case 4: run_window<true, 4>(w, in0, in1, out, st); break;
          default: run_window<true, 0>(w, in0, in1, out, st); break;
        }
      } else {
        switch (mode) {
          case 1: run_window<false, 1>(w, in0, in1, out, st); break;
          case 2: run_window<false, 2>(w, in0, in1, out, st); break;
          case 3: run_window<false, 3>(w, in0, in1, out, st); break;
          case 4: run_window<false, 4>(w, in0, in1, out, st); break;
          default: run_window<false, 0>(w, in0, in1, out, st); break;
        }
      }
      return;
    }
  }
}

}  // namespace gb::dev
