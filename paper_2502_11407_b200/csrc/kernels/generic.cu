// State-driven SIMT kernel: executes ANY complete schedule of a contraction-form operator
// (gemm, gemv, conv2d, avgpool2d, dwconv2d; batched gemm via grid.y) exactly as the schedule
// tiles it. This is the execute step the reference's (absent) interpreter performs on the CPU
// (SPEC.md:479-487), moved onto the GPU:
//   * one CTA per level-1 spatial tile; one thread slot per level-L thread tile;
//   * virtual threads = strided slices of the thread tile;
//   * each level-1 reduce chunk's input boxes staged in shared memory, then the deeper reduce
//     digits walked in the interpreter's order, guarded (padding) iterations skipped.
// Acc = double gives the parity variant: products of fp32/bf16 inputs are exact in double and
// the additions happen in the interpreter's order, so outputs equal the oracle's interpret()
// bit for bit. Acc = float is the fp32 FFMA variant.
#include "../host/error.hpp"
#include "common.cuh"
#include "launch.h"
#include "plan.h"
#include "tc_common.cuh"

#include <type_traits>

namespace gb::dev {

namespace {

template <typename In, typename Out, typename Acc, int ACC>
__global__ void __launch_bounds__(256) k_generic(const GenericPlan p, const In* __restrict__ in0,
                                                  const In* __restrict__ in1, Out* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  In* sm = reinterpret_cast<In*>(smem_raw);
  const int64_t b = blockIdx.y;
  in0 += b * p.batch_stride[0];
  if (p.n_in == 2) in1 += b * p.batch_stride[1];
  out += b * p.batch_stride[2];

  int64_t org[8];
#pragma unroll
  for (int a = 0; a < 8; ++a) org[a] = 0;
  {
    int64_t c = blockIdx.x;
    for (int i = p.nsp - 1; i >= 0; --i) {
      org[p.sp[i]] = (c % p.tiles[i]) * p.B[i];
      c /= p.tiles[i];
    }
  }

  for (int round = 0; round < p.rounds; ++round) {
    const int slot = round * p.block + threadIdx.x;
    const bool active = slot < p.slots;
    int th[4] = {0, 0, 0, 0};
    {
      int c = active ? slot : 0;
      for (int i = p.nsp - 1; i >= 0; --i) {
        const int n = p.B[i] / p.T[i];
        th[i] = c % n;
        c /= n;
      }
    }
    for (int ch = 0; ch < p.acc_chunks; ++ch) {
      int64_t o0[ACC], o1[ACC], og[ACC];
      bool ok[ACC];
#pragma unroll
      for (int j = 0; j < ACC; ++j) {
        int e = ch * ACC + j;
        int64_t g0 = 0, g1 = 0, go = 0;
        bool inb = active;
        for (int i = p.nsp - 1; i >= 0; --i) {
          const int Ti = p.T[i];
          const int ei = e % Ti;
          e /= Ti;
          const int per = Ti / p.V[i];
          const int rel = (ei / per) * (p.B[i] / p.V[i]) + th[i] * per + (ei % per);
          const int a = p.sp[i];
          const int64_t ab = org[a] + rel;
          inb = inb && ab < p.ext[a];
          if (p.staged) {
            g0 += rel * p.scoef[0][a];
            g1 += rel * p.scoef[1][a];
          } else {
            g0 += ab * p.coef[0][a];
            g1 += ab * p.coef[1][a];
          }
          go += ab * p.coef[2][a];
        }
        o0[j] = g0;
        o1[j] = g1;
        og[j] = go;
        ok[j] = inb;
      }
      Acc acc[ACC];
#pragma unroll
      for (int j = 0; j < ACC; ++j) acc[j] = Acc(0);

      for (int c = 0; c < p.n_chunks; ++c) {
        int64_t ro[3] = {0, 0, 0};
        {
          int x = c;
          for (int q = p.nred - 1; q >= 0; --q) {
            ro[q] = static_cast<int64_t>(x % p.outer_radix[q]) * p.chunk_tile[q];
            x /= p.outer_radix[q];
          }
        }
        if (p.staged) {
          for (int q = 0; q < p.nred; ++q) org[p.red[q]] = ro[q];
          __syncthreads();  // previous chunk fully consumed
          for (int t = 0; t < p.n_in; ++t) {
            const In* src = t == 0 ? in0 : in1;
            int64_t bo[4];
            for (int d = 0; d < p.sm_nd[t]; ++d) {
              const int w = p.sm_win[t][d];
              bo[d] = w < 0 ? org[p.sm_axis[t][d]] : org[p.sm_axis[t][d]] * p.stride + org[w];
            }
            In* dst = sm + p.sm_base[t];
            for (int e = threadIdx.x; e < p.sm_elems[t]; e += blockDim.x) {
              int x = e;
              int64_t ga = 0;
              bool inb = true;
              for (int d = p.sm_nd[t] - 1; d >= 0; --d) {
                const int rel = x % p.sm_range[t][d];
                x /= p.sm_range[t][d];
                const int64_t coord = bo[d] + rel;
                inb = inb && coord < p.sm_gdim[t][d];
                ga += coord * p.sm_gstride[t][d];
              }
              dst[e] = inb ? src[ga] : In(0.0f);
            }
          }
          __syncthreads();
        }
        const In* s0 = p.staged ? sm + p.sm_base[0] : in0;
        const In* s1 = p.staged ? sm + p.sm_base[1] : in1;
        for (int i = 0; i < p.chunk_len; ++i) {
          int rr[3] = {0, 0, 0};
          {
            int x = i;
            for (int d = p.n_inner - 1; d >= 0; --d) {
              const int r = x % p.inner_radix[d];
              x /= p.inner_radix[d];
              rr[p.inner_slot[d]] += r * p.inner_mul[d];
            }
          }
          bool guard = false;
          int64_t r0 = 0, r1 = 0;
          for (int q = 0; q < p.nred; ++q) {
            const int a = p.red[q];
            const int64_t ab = ro[q] + rr[q];
            guard = guard || ab >= p.ext[a];
            if (p.staged) {
              r0 += rr[q] * p.scoef[0][a];
              r1 += rr[q] * p.scoef[1][a];
            } else {
              r0 += ab * p.coef[0][a];
              r1 += ab * p.coef[1][a];
            }
          }
          if (guard) continue;  // padded iteration: skipped, as the interpreter does
#pragma unroll
          for (int j = 0; j < ACC; ++j) {
            if (!ok[j]) continue;
            Acc v = static_cast<Acc>(to_f32(s0[o0[j] + r0]));
            if (p.n_in == 2) v *= static_cast<Acc>(to_f32(s1[o1[j] + r1]));
            acc[j] += v;
          }
        }
      }
#pragma unroll
      for (int j = 0; j < ACC; ++j) {
        if (!ok[j]) continue;
        Acc v = acc[j];
        if (p.divisor) v = v / static_cast<Acc>(p.divisor);
        out[og[j]] = from_f32<Out>(static_cast<float>(v));
      }
    }
  }
}

// ---- register-tiled fast paths of the same plans (simt_f32) --------------------------------
// The program is the plan's: CTA = level-1 spatial tile, thread = level-L thread tile split into
// vthread slices (slice e of a thread covers (e / per) * (B / V) + th * per + e % per), the reduce
// axis walked in ascending order through level-1 chunks staged in shared memory — for a single
// reduce axis that IS the interpreter's order (chunks, then level-2.. digits, then scalars), so
// outputs equal k_generic<float>'s. What changes is mechanical: compile-time thread tiles, the A
// chunk staged k-major so a thread's rows are adjacent words (float4 loads when a slice holds >= 4),
// no index decoding in the k loop.
__device__ __forceinline__ void cp_async4(void* dst, const void* src, bool valid) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(src), "r"(valid ? 4 : 0) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, int bytes) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

template <typename In, int TM, int TN>
__global__ void __launch_bounds__(256) k_simt_gemm(const GenericPlan p, const In* __restrict__ A,
                                                   const In* __restrict__ Bm, In* __restrict__ C) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int BM = p.B[0], BN = p.B[1], BK = p.chunk_tile[0];
  // A chunk row-major [BM][BK], 16 B granules of row mm XOR-swizzled by ((mm >> 3) & 7): a warp's
  // TM-row reads (4 row groups x 8 rows apart) hit distinct banks, and 16 B copies stay aligned
  float* As = reinterpret_cast<float*>(smem_raw);
  float* Bs = As + BM * BK;  // [BK][BN]
  const int am = p.sp[0], an = p.sp[1], ak = p.red[0];
  const int64_t M = p.ext[am], N = p.ext[an], K = p.ext[ak];
  const int64_t b = blockIdx.y;
  A += b * p.batch_stride[0];
  Bm += b * p.batch_stride[1];
  C += b * p.batch_stride[2];
  const int64_t m0 = static_cast<int64_t>(blockIdx.x / p.tiles[1]) * BM;
  const int64_t n0 = static_cast<int64_t>(blockIdx.x % p.tiles[1]) * BN;
  const int sn = BN / TN;
  const bool active = static_cast<int>(threadIdx.x) < p.slots;
  const int thm = active ? threadIdx.x / sn : 0, thn = active ? threadIdx.x % sn : 0;
  const int perm = TM / p.V[0], pern = TN / p.V[1];
  const int strm = BM / p.V[0], strn = BN / p.V[1];
  int ra[TM], fx[TM], rn[TN];
#pragma unroll
  for (int e = 0; e < TM; ++e) {
    const int mm = (e / perm) * strm + thm * perm + e % perm;
    ra[e] = mm * BK;
    fx[e] = BK >= 32 ? ((mm >> 3) & 7) << 2 : 0;
  }
#pragma unroll
  for (int e = 0; e < TN; ++e) rn[e] = (e / pern) * strn + thn * pern + e % pern;
  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.0f;
  const int64_t a_m = p.coef[0][am], a_k = p.coef[0][ak], b_k = p.coef[1][ak], b_n = p.coef[1][an];
  const bool bvec = pern % 4 == 0 && BN % 4 == 0;
  // 16 B asynchronous copies when both operands are fp32 with unit-stride, 16 B-aligned rows
  const bool v16 = sizeof(In) == 4 && a_k == 1 && b_n == 1 && (a_m & 3) == 0 && (b_k & 3) == 0 && (n0 & 3) == 0 &&
                   (reinterpret_cast<uintptr_t>(A) & 15) == 0 && (reinterpret_cast<uintptr_t>(Bm) & 15) == 0 &&
                   BK % 4 == 0 && BN % 4 == 0;
  const int kshift = __ffs(BK) - 1, nshift = __ffs(BN) - 1;  // level-1 tiles are powers of two
  auto swz = [&](int mm, int kk) { return mm * BK + (kk ^ (BK >= 32 ? ((mm >> 3) & 7) << 2 : 0)); };
  for (int64_t k0 = 0; k0 < K; k0 += BK) {
    const int kc = static_cast<int>(K - k0 < BK ? K - k0 : BK);
    __syncthreads();  // the previous chunk is consumed
    if constexpr (sizeof(In) == 4) {
      if (v16) {
        // A: BM rows x BK/4 granules; B: BK rows x BN/4 granules (zero-filled out of range)
        for (int e = threadIdx.x; e < (BM * BK) >> 2; e += blockDim.x) {
          const int mm = (4 * e) >> kshift, kk = (4 * e) & (BK - 1);
          const int64_t krem = kc - kk;
          const int bytes = m0 + mm < M ? static_cast<int>(krem >= 4 ? 16 : krem > 0 ? 4 * krem : 0) : 0;
          cp_async16(As + swz(mm, kk), bytes ? A + (m0 + mm) * a_m + (k0 + kk) : A, bytes);
        }
        for (int e = threadIdx.x; e < (BK * BN) >> 2; e += blockDim.x) {
          const int kk = (4 * e) >> nshift, nn = (4 * e) & (BN - 1);
          const int64_t nrem = N - (n0 + nn);
          const int bytes = kk < kc ? static_cast<int>(nrem >= 4 ? 16 : nrem > 0 ? 4 * nrem : 0) : 0;
          cp_async16(Bs + kk * BN + nn, bytes ? Bm + (k0 + kk) * b_k + (n0 + nn) : Bm, bytes);
        }
      } else {
        for (int e = threadIdx.x; e < BM * BK; e += blockDim.x) {  // coalesced along k
          const int mm = e >> kshift, kk = e & (BK - 1);
          const bool ok = kk < kc && m0 + mm < M;
          cp_async4(As + swz(mm, kk), ok ? A + (m0 + mm) * a_m + (k0 + kk) * a_k : A, ok);
        }
        for (int e = threadIdx.x; e < BK * BN; e += blockDim.x) {
          const int kk = e >> nshift, nn = e & (BN - 1);
          const bool ok = kk < kc && n0 + nn < N;
          cp_async4(Bs + kk * BN + nn, ok ? Bm + (k0 + kk) * b_k + (n0 + nn) * b_n : Bm, ok);
        }
      }
      cp_async_wait_all();
    } else {
      for (int e = threadIdx.x; e < BM * BK; e += blockDim.x) {
        const int mm = e >> kshift, kk = e & (BK - 1);
        As[swz(mm, kk)] = kk < kc && m0 + mm < M ? to_f32(A[(m0 + mm) * a_m + (k0 + kk) * a_k]) : 0.0f;
      }
      for (int e = threadIdx.x; e < BK * BN; e += blockDim.x) {
        const int kk = e >> nshift, nn = e & (BN - 1);
        Bs[kk * BN + nn] = kk < kc && n0 + nn < N ? to_f32(Bm[(k0 + kk) * b_k + (n0 + nn) * b_n]) : 0.0f;
      }
    }
    __syncthreads();
    if (!active) continue;
    auto step = [&](int kk, const int (&abase)[TM], int r) {
      float a[TM], bv[TN];
#pragma unroll
      for (int e = 0; e < TM; ++e) a[e] = As[abase[e] + r];
      if (bvec) {
#pragma unroll
        for (int e = 0; e < TN; e += 4) {
          const float4 x = *reinterpret_cast<const float4*>(Bs + kk * BN + rn[e]);
          bv[e] = x.x, bv[e + 1] = x.y, bv[e + 2] = x.z, bv[e + 3] = x.w;
        }
      } else {
#pragma unroll
        for (int e = 0; e < TN; ++e) bv[e] = Bs[kk * BN + rn[e]];
      }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], bv[j], acc[i][j]);
    };
    int kq = 0;
    for (; kq + 4 <= kc; kq += 4) {  // ascending k; the swizzle is constant inside a 16 B granule
      int abase[TM];
#pragma unroll
      for (int e = 0; e < TM; ++e) abase[e] = ra[e] + (kq ^ fx[e]);
#pragma unroll
      for (int r = 0; r < 4; ++r) step(kq + r, abase, r);
    }
    for (; kq < kc; ++kq) {
      int abase[TM];
#pragma unroll
      for (int e = 0; e < TM; ++e) abase[e] = ra[e] + ((kq & ~3) ^ fx[e]);
      step(kq, abase, kq & 3);
    }
  }
  if (!active) return;
  const int64_t c_m = p.coef[2][am], c_n = p.coef[2][an];
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int64_t m = m0 + ra[i] / BK;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int64_t n = n0 + rn[j];
      if (n < N) C[m * c_m + n * c_n] = from_f32<In>(acc[i][j]);
    }
  }
}

// gemv: CTA = level-1 m tile, thread = TM rows (vthread slices), n ascending; x staged once in
// shared memory when it fits; each row streamed with float4 loads (4 consecutive n, summed in
// order), U loads per row in flight.
template <int TM>
__global__ void __launch_bounds__(256) k_simt_gemv(const GenericPlan p, const float* __restrict__ A,
                                                   const float* __restrict__ x, float* __restrict__ y) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* xs = reinterpret_cast<float*>(smem_raw);
  const int am = p.sp[0], an = p.red[0];
  const int64_t M = p.ext[am], N = p.ext[an];
  const int64_t b = blockIdx.y;
  A += b * p.batch_stride[0];
  x += b * p.batch_stride[1];
  y += b * p.batch_stride[2];
  const bool xin = p.fast_pad != 0;  // x staged
  if (xin) {
    for (int64_t i = threadIdx.x; i < N; i += blockDim.x) xs[i] = x[i * p.coef[1][an]];
    __syncthreads();
  }
  const int BM = p.B[0];
  const int64_t m0 = static_cast<int64_t>(blockIdx.x) * BM;
  if (static_cast<int>(threadIdx.x) >= p.slots) return;
  const int per = TM / p.V[0], str = BM / p.V[0];
  const float* row[TM];
  bool ok[TM];
  float acc[TM];
#pragma unroll
  for (int e = 0; e < TM; ++e) {
    const int64_t m = m0 + (e / per) * str + static_cast<int>(threadIdx.x) * per + e % per;
    ok[e] = m < M;
    row[e] = A + (ok[e] ? m : 0) * p.coef[0][am];
    acc[e] = 0.0f;
  }
  const int64_t a_n = p.coef[0][an];
  const float* xv = xin ? xs : x;
  const int64_t x_n = xin ? 1 : p.coef[1][an];
  int64_t n = 0;
  if (a_n == 1 && x_n == 1 && (p.coef[0][am] & 3) == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0) {
    constexpr int U = TM <= 4 ? 4 : 2;  // float4 loads per row in flight
    for (; n + 4 * U <= N; n += 4 * U) {
      float4 v[TM][U];
#pragma unroll
      for (int e = 0; e < TM; ++e)
#pragma unroll
        for (int u = 0; u < U; ++u) v[e][u] = __ldg(reinterpret_cast<const float4*>(row[e] + n) + u);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const float4 xx = *reinterpret_cast<const float4*>(xv + n + 4 * u);
#pragma unroll
        for (int e = 0; e < TM; ++e) {
          acc[e] = fmaf(v[e][u].x, xx.x, acc[e]);
          acc[e] = fmaf(v[e][u].y, xx.y, acc[e]);
          acc[e] = fmaf(v[e][u].z, xx.z, acc[e]);
          acc[e] = fmaf(v[e][u].w, xx.w, acc[e]);
        }
      }
    }
  }
  for (; n < N; ++n) {
    const float xx = xv[n * x_n];
#pragma unroll
    for (int e = 0; e < TM; ++e) acc[e] = fmaf(__ldg(row[e] + n * a_n), xx, acc[e]);
  }
#pragma unroll
  for (int e = 0; e < TM; ++e) {
    const int64_t m = m0 + (e / per) * str + static_cast<int>(threadIdx.x) * per + e % per;
    if (ok[e]) y[m * p.coef[2][am]] = acc[e];
  }
}

// gemv through TMA (plan.fast == 3: one row per thread per row group, i.e. vthreads == thread tile):
// stage s holds, for row group e, the CTA's `slots` consecutive rows x 32 columns per 4 KB box
// (128 B swizzle), 8 boxes per stage (256 columns); thread t reduces row (e * slots + t) from its
// 128 B row of each box — the swizzle puts the 8 lanes of a shared-memory phase on distinct banks —
// in ascending column order. Whole lines from HBM, one TMA op per 4 KB.
constexpr int kGvBoxCols = 32, kGvBoxes = 8, kGvStages = 3;

template <int TM>
__global__ void __launch_bounds__(256) k_simt_gemv_tma(const __grid_constant__ CUtensorMap mapA, const GenericPlan p,
                                                       const float* __restrict__ x, float* __restrict__ y) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);  // swizzle atoms
  __shared__ uint64_t full[kGvStages], empty[kGvStages];
  const int am = p.sp[0], an = p.red[0];
  const int64_t M = p.ext[am], N = p.ext[an];
  const int slots = p.slots;                        // rows per row group = threads that own rows
  const uint32_t stage_bytes = static_cast<uint32_t>(slots) * 128 * kGvBoxes;
  float* xs = reinterpret_cast<float*>(smem + kGvStages * stage_bytes);
  const int64_t m0 = static_cast<int64_t>(blockIdx.x) * p.B[0];
  const int cols = kGvBoxCols * kGvBoxes;
  const int nchunks = static_cast<int>((N + cols - 1) / cols);
  const int nsteps = TM * nchunks;                  // (row group e, column chunk c), e-major
  if (threadIdx.x == 0) {
    for (int i = 0; i < kGvStages; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&empty[i], blockDim.x);
    }
    tc::fence_barrier_init();
  }
  for (int64_t i = threadIdx.x; i < N; i += blockDim.x) xs[i] = x[i * p.coef[1][an]];
  __syncthreads();
  auto issue = [&](int s, int k) {  // thread 0: stage s <- step k
    const int e = k / nchunks, c = k - e * nchunks;
    tc::mbar_arrive_expect_tx(&full[s], stage_bytes);
    uint8_t* dst = smem + s * stage_bytes;
    for (int b = 0; b < kGvBoxes; ++b)
      tc::tma_load_2d(dst + b * slots * 128, &mapA, &full[s], c * cols + b * kGvBoxCols,
                      static_cast<int>(m0 + static_cast<int64_t>(e) * slots));
  };
  if (threadIdx.x == 0)
    for (int k = 0; k < kGvStages && k < nsteps; ++k) issue(k, k);
  const int t = threadIdx.x;
  const bool active = t < slots;
  float acc = 0.0f;
  for (int k = 0; k < nsteps; ++k) {
    const int s = k % kGvStages;
    const int e = k / nchunks, c = k - e * nchunks;
    tc::mbar_wait(&full[s], (k / kGvStages) & 1);
    if (active) {
      const uint8_t* src = smem + s * stage_bytes + t * 128;
      const int64_t n0 = static_cast<int64_t>(c) * cols;
      if (n0 + cols <= N) {
#pragma unroll
        for (int b = 0; b < kGvBoxes; ++b) {
#pragma unroll
          for (int g = 0; g < 8; ++g) {
            const float4 v = *reinterpret_cast<const float4*>(src + b * slots * 128 + ((g ^ (t & 7)) << 4));
            const float4 xx = *reinterpret_cast<const float4*>(xs + n0 + b * kGvBoxCols + 4 * g);
            acc = fmaf(v.x, xx.x, acc);
            acc = fmaf(v.y, xx.y, acc);
            acc = fmaf(v.z, xx.z, acc);
            acc = fmaf(v.w, xx.w, acc);
          }
        }
      } else {
        for (int q = 0; n0 + q < N; ++q) {
          const int b = q / kGvBoxCols, w = q % kGvBoxCols;
          const float v = *reinterpret_cast<const float*>(src + b * slots * 128 + (((w >> 2) ^ (t & 7)) << 4) + (w & 3) * 4);
          acc = fmaf(v, xs[n0 + q], acc);
        }
      }
      if (c == nchunks - 1) {  // row (e, t) complete
        const int64_t m = m0 + static_cast<int64_t>(e) * slots + t;
        if (m < M) y[m * p.coef[2][am]] = acc;
        acc = 0.0f;
      }
    }
    tc::mbar_arrive(&empty[s]);
    if (threadIdx.x == 0 && k + kGvStages < nsteps) {
      tc::mbar_wait(&empty[s], (k / kGvStages) & 1);
      issue(s, k + kGvStages);
    }
  }
}

void launch_simt_gemv_tma(const GenericPlan& p, const CUtensorMap& mapA, const void* in1, void* out, int batch,
                          cudaStream_t st) {
  dim3 g(static_cast<unsigned>(p.tiles[0]), static_cast<unsigned>(batch));
  auto go = [&](auto kern) {
    set_smem_attr(kern, p.smem_bytes, "simt gemv smem attribute");
    kern<<<g, p.block, p.smem_bytes, st>>>(mapA, p, static_cast<const float*>(in1), static_cast<float*>(out));
    check_cuda(cudaGetLastError(), "simt gemv launch");
    count_launch();
  };
  switch (p.T[0]) {
    case 1: go(k_simt_gemv_tma<1>); break;
    case 2: go(k_simt_gemv_tma<2>); break;
    case 4: go(k_simt_gemv_tma<4>); break;
    case 8: go(k_simt_gemv_tma<8>); break;
    default: throw Error(Code::Unsupported, "simt gemv thread tile");
  }
}

template <typename In>
void launch_simt_gemm(const GenericPlan& p, const void* in0, const void* in1, void* out, int batch, cudaStream_t st) {
  dim3 g(static_cast<unsigned>(p.tiles[0]) * static_cast<unsigned>(p.tiles[1]), static_cast<unsigned>(batch));
  auto go = [&](auto kern) {
    if (p.smem_bytes > 48 * 1024)
      set_smem_attr(kern, p.smem_bytes, "simt gemm smem attribute");
    kern<<<g, p.block, p.smem_bytes, st>>>(p, static_cast<const In*>(in0), static_cast<const In*>(in1),
                                          static_cast<In*>(out));
    check_cuda(cudaGetLastError(), "simt gemm launch");
    count_launch();
  };
  auto pick_n = [&](auto tm) {
    constexpr int TM = decltype(tm)::value;
    switch (p.T[1]) {
      case 1: go(k_simt_gemm<In, TM, 1>); break;
      case 2: go(k_simt_gemm<In, TM, 2>); break;
      case 4: go(k_simt_gemm<In, TM, 4>); break;
      case 8: go(k_simt_gemm<In, TM, 8>); break;
      default: throw Error(Code::Unsupported, "simt gemm thread tile");
    }
  };
  switch (p.T[0]) {
    case 1: pick_n(std::integral_constant<int, 1>{}); break;
    case 2: pick_n(std::integral_constant<int, 2>{}); break;
    case 4: pick_n(std::integral_constant<int, 4>{}); break;
    case 8: pick_n(std::integral_constant<int, 8>{}); break;
    default: throw Error(Code::Unsupported, "simt gemm thread tile");
  }
}

void launch_simt_gemv(const GenericPlan& p, const void* in0, const void* in1, void* out, int batch, cudaStream_t st) {
  dim3 g(static_cast<unsigned>(p.tiles[0]), static_cast<unsigned>(batch));
  auto go = [&](auto kern) {
    if (p.smem_bytes > 48 * 1024)
      set_smem_attr(kern, p.smem_bytes, "simt gemv smem attribute");
    kern<<<g, p.block, p.smem_bytes, st>>>(p, static_cast<const float*>(in0), static_cast<const float*>(in1),
                                          static_cast<float*>(out));
    check_cuda(cudaGetLastError(), "simt gemv launch");
    count_launch();
  };
  switch (p.T[0]) {
    case 1: go(k_simt_gemv<1>); break;
    case 2: go(k_simt_gemv<2>); break;
    case 4: go(k_simt_gemv<4>); break;
    case 8: go(k_simt_gemv<8>); break;
    default: throw Error(Code::Unsupported, "simt gemv thread tile");
  }
}

template <typename In, typename Out, typename Acc>
void dispatch(const GenericPlan& p, int width, const void* in0, const void* in1, void* out, int batch,
              cudaStream_t st) {
  int64_t grid = 1;
  for (int i = 0; i < p.nsp; ++i) grid *= p.tiles[i];
  dim3 g(static_cast<unsigned>(grid), static_cast<unsigned>(batch));
  auto go = [&](auto kern) {
    if (p.smem_bytes > 48 * 1024)
      set_smem_attr(kern, p.smem_bytes, "generic smem attribute");
    kern<<<g, p.block, p.smem_bytes, st>>>(p, static_cast<const In*>(in0), static_cast<const In*>(in1),
                                          static_cast<Out*>(out));
    check_cuda(cudaGetLastError(), "generic launch");
    count_launch();
  };
  switch (width) {
    case 1: go(k_generic<In, Out, Acc, 1>); break;
    case 2: go(k_generic<In, Out, Acc, 2>); break;
    case 4: go(k_generic<In, Out, Acc, 4>); break;
    case 8: go(k_generic<In, Out, Acc, 8>); break;
    case 16: go(k_generic<In, Out, Acc, 16>); break;
    case 32: go(k_generic<In, Out, Acc, 32>); break;
    default: throw Error(Code::Unsupported, "generic accumulator width " + std::to_string(width));
  }
}

}  // namespace

int generic_max_width(bool f64) { return f64 ? 16 : 32; }

void launch_generic(const GenericPlan& p, bool f64, bool bf16, const void* in0, const void* in1, void* out,
                    int batch, cudaStream_t st, const CUtensorMap* map) {
  if (!f64 && !bf16 && p.fast == 3 && map) {
    launch_simt_gemv_tma(p, *map, in1, out, batch, st);
    return;
  }
  if (!f64 && p.fast == 1) {
    if (bf16)
      launch_simt_gemm<__nv_bfloat16>(p, in0, in1, out, batch, st);
    else
      launch_simt_gemm<float>(p, in0, in1, out, batch, st);
    return;
  }
  if (!f64 && !bf16 && p.fast == 2) {
    launch_simt_gemv(p, in0, in1, out, batch, st);
    return;
  }
  const int width = p.acc / p.acc_chunks;
  if (bf16) {
    if (f64)
      dispatch<__nv_bfloat16, __nv_bfloat16, double>(p, width, in0, in1, out, batch, st);
    else
      dispatch<__nv_bfloat16, __nv_bfloat16, float>(p, width, in0, in1, out, batch, st);
  } else {
    if (f64)
      dispatch<float, float, double>(p, width, in0, in1, out, batch, st);
    else
      dispatch<float, float, float>(p, width, in0, in1, out, batch, st);
  }
}

}  // namespace gb::dev
