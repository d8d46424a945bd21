// conv_flat: stride-1 tf32 conv2d that reads the caller's NCHW input IN PLACE through TMA (no
// NHWC copy of the activations).
//
// Flattened planes. With stride 1, output (h, w) of image n reads input position
// p + r*W + s of every channel plane, where p = h*W + w is the output's position in the INPUT's
// row pitch ("wide" positions; the W - OW columns past each output row are computed and
// dropped). So every tap (r, s) is a 1-D shift o = r*W + s of one flat plane, and a tile of 128
// consecutive wide positions is an M = 128 UMMA tile whose A operand (positions x channels) is
// MN-major: 32 consecutive positions of one channel are one 128 B row, exactly what a TMA box
// over the plane-major input {H*W, N*C} delivers (32 B-atom swizzle, the tf32 MN-major layout).
//
// Alignment. TMA can only start a box at a 16 B-aligned position (tools/tma_align_probe.cu), so a
// tap is split as o = a + b with a = o & ~3 (the A box offset) and b = o & 3. The MMA for tap
// (r, s) multiplies the box at P0 + a and lands in TMEM accumulator block b; the epilogue adds
// block b of TMEM lane j + b into output j. Taps sharing an offset a share one staged A box and
// are folded into the UMMA N (3x3 over a 58-wide plane: a = 0 {b 0,1,2 -> N 192}, 56 {b 2,3 ->
// N 128}, 60 {b 0 -> N 64}, 116 {b 0,1,2 -> N 192}); their filter rows sit next to each other in
// the resident bank. Lanes j + b >= 32 belong to the next warp's lane quarter: the first three
// lanes of each warp publish their blocks 1..3 through shared memory. Tiles advance by 124
// positions (multiple of 4, lanes 124..127 only feed their neighbours).
//
// Two launches, chained by programmatic dependent launch: k_flat_filters converts K[f][c][r][s]
// into the bank image W' (K-major, 128 B-swizzled, tf32-rounded; one 147 KB copy per execute in
// the workspace) while the conv grid starts and streams its first input stages; the conv CTAs
// then copy W' into shared memory with one bulk copy per 32-channel chunk.
//
// Filter groups: the plan may split F into FG groups of FN filters (the constructed state's
// level-1 f tile): CTA b works on group b % FG with that group's resident bank and walks the
// position tiles b / FG, b / FG + grid / FG, ...; every group re-reads the input tiles (L2).
//
// Roles: warp 0 = TMA producer (one 16 KB stage per (tile, 32-channel chunk, offset group)),
// warp 1 = MMA issuer (a precomputed op table: accumulator column, filter rows, UMMA N, first-touch
// flag), warps 2.. = epilogue (EPW warps per TMEM lane quarter, splitting the 16-filter blocks).
// Accumulators: 4 blocks of FN columns, double-buffered (2 x 256 TMEM columns), so tile i's
// epilogue overlaps tile i+1's MMAs.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>
#include <utility>
#include <cstdlib>
#include <string>

#include "../host/error.hpp"
#include "common.cuh"
#include "launch.h"
#include "tc_common.cuh"

namespace gb::dev {
using namespace tc;

#ifdef GENSOR_DEV_OVERRIDES
// Developer timeline (make DEV=1 only): clock64 marks per CTA, 64 slots (tools/conv_trace.py):
// 0 start, 1 bank requested, 8+i MMA tile i start, 16+i tile i committed, 24+i epilogue got tile i,
// 32+i epilogue done with tile i, 40 MMA loop end, 44/45 epilogue of tile 1: blocks read /
// boundary values exchanged.
__device__ long long g_flat_trace[160 * 64];
// per epilogue warp, tile 1: [0] acc_full seen, [1] TMEM read, [2] at the quarter barrier, [3] past it, [4] done
__device__ long long g_flat_warp[160 * 16 * 5];
#define FL_WMARK(k)                                                                                   \
  do {                                                                                                \
    if (blockIdx.x < 160 && lane == 0 && local == 1 && warp >= 2)                                    \
      g_flat_warp[(blockIdx.x * 16 + (warp - 2)) * 5 + (k)] = clock64() - g_flat_trace[blockIdx.x * 64]; \
  } while (0)
extern "C" int gensor_dev_flat_warp(long long* out, int n) {
  return cudaMemcpyFromSymbol(out, g_flat_warp, sizeof(long long) * std::min(n, 160 * 16 * 5)) == cudaSuccess ? 0 : 19;
}
#define FL_MARK(slot) \
  do {                 \
    if (blockIdx.x < 160) g_flat_trace[blockIdx.x * 64 + (slot)] = clock64(); \
  } while (0)
#define FL_CLOCK() clock64()
#define FL_STORE(slot, v) \
  do {                     \
    if (blockIdx.x < 160) g_flat_trace[blockIdx.x * 64 + (slot)] = (v); \
  } while (0)
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ unsigned long long g_flat_filt[5];  // [3]: last counter increment, [4]: first conv observation  // filters kernel: min start, max end; marker kernel (globaltimer ns)
__global__ void k_flat_marker() { g_flat_filt[2] = gtimer(); }
#define FL_GT(slot) \
  do {               \
    if (blockIdx.x < 160) g_flat_trace[blockIdx.x * 64 + (slot)] = gtimer(); \
  } while (0)
extern "C" int gensor_dev_flat_filt(unsigned long long* out) {
  const int r = cudaMemcpyFromSymbol(out, g_flat_filt, sizeof(g_flat_filt)) == cudaSuccess ? 0 : 19;
  const unsigned long long init[5] = {~0ull, 0ull, 0ull, 0ull, ~0ull};
  cudaMemcpyToSymbol(g_flat_filt, init, sizeof(init));
  return r;
}
extern "C" int gensor_dev_flat_trace(long long* out, int n) {
  return cudaMemcpyFromSymbol(out, g_flat_trace, sizeof(long long) * std::min(n, 160 * 64)) == cudaSuccess ? 0 : 19;
}
#else
#define FL_GT(slot) \
  do {               \
  } while (0)
#define FL_MARK(slot) \
  do {                 \
  } while (0)
#define FL_CLOCK() 0ll
#define FL_WMARK(k) \
  do {              \
  } while (0)
#define FL_STORE(slot, v) \
  do {                     \
  } while (0)
#endif

namespace {

constexpr int kFlatStep = 124;     // tile advance (lanes 124..127 are only read by their neighbours)
constexpr int kFlatStage = 16384;  // one A stage: 4 boxes of 32 positions x 32 channels x 4 B
constexpr int kFlatXFloats = 96;   // per warp and 16-filter block: [b1 L0][b2 L0,L1][b3 L0,L1,L2]
constexpr int kFlatMaxChunks = 8;  // bank barriers (one per 32-channel chunk, the last takes the rest)
constexpr int kFlatEpw = 4;        // epilogue warps per TMEM lane quarter (one 16-filter block each at FN = 64)
constexpr int kFlatNfbh = 1;       // 16-filter blocks per epilogue warp (FN <= 64)

// round to tf32 (nearest, ties away — cvt.rna.tf32.f32) with two integer ops; Inf / NaN unchanged
__device__ __forceinline__ uint32_t f32_to_tf32(float x) {
  const uint32_t u = __float_as_uint(x);
  return (u & 0x7f800000u) == 0x7f800000u ? u : (u + 0x1000u) & 0xffffe000u;
}

__device__ __forceinline__ void named_bar(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// The filter-bank image comes from the preceding launch. With a handle-owned workspace the conv
// CTAs poll a completion counter the filter CTAs raise (their stores are published with a
// device-scope fence before the increment); griddepcontrol.wait would instead wait for the whole
// primary grid to retire, measured ~5.5 us after its last store on these boxes. The last conv CTA
// through resets the counter (the next execute's filter launch runs after this grid). A caller
// workspace (sync == nullptr) keeps griddepcontrol.wait.
__device__ __forceinline__ void flat_wait_bank_image(unsigned* sync, unsigned filt_blocks) {
  if (!sync) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    return;
  }
  unsigned v;
  for (;;) {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(sync) : "memory");
    if (v >= filt_blocks) break;
    __nanosleep(64);
  }
#ifdef GENSOR_DEV_OVERRIDES
  atomicMin(&g_flat_filt[4], static_cast<unsigned long long>(gtimer()));
#endif
  asm volatile("fence.proxy.async.global;" ::: "memory");  // the generic-proxy image -> this thread's bulk copies
}

// After this CTA's bank copies are issued (the returning atomic stays off the bank's critical
// path): the last conv CTA through resets the counter for the next execute.
__device__ __forceinline__ void flat_done_with_counter(unsigned* sync) {
  if (sync && atomicAdd(sync + 1, 1u) == gridDim.x - 1) {
    atomicExch(sync, 0u);
    atomicExch(sync + 1, 0u);
  }
}

__device__ __forceinline__ void flat_signal_bank_image(unsigned* sync) {
  __syncthreads();
  if (sync && threadIdx.x == 0) {
    // release at gpu scope: cumulative over the CTA's image stores ordered before it by the barrier
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(sync) : "memory");
#ifdef GENSOR_DEV_OVERRIDES
    atomicMax(&g_flat_filt[3], static_cast<unsigned long long>(gtimer()));
#endif
  }
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// ---- bank image W'[chunk][slot(t)][f][32 c] (K-major rows of 128 B, 128 B swizzle: 16 B granule
// g of row rho stored at g ^ (rho & 7)), tf32-rounded, rows f >= F zero. One thread per (f, 4
// channels, tap): four strided loads of K, one 16 B store.
__global__ void __launch_bounds__(128) k_flat_filters(const float* __restrict__ K, uint8_t* __restrict__ Wp,
                                                      const __grid_constant__ ConvFlatArgs a, unsigned* sync) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the conv grid may start now
#ifdef GENSOR_DEV_OVERRIDES
  if (threadIdx.x == 0) atomicMin(&g_flat_filt[0], static_cast<unsigned long long>(gtimer()));
#endif
  const int c4n = a.C >> 2;
  const int total = a.FG * a.FN * c4n * a.T;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < total) {
  const int t = e % a.T;
  const int u = e / a.T;
  const int f = u / c4n, c4 = u - f * c4n;  // f = group * FN + row in the group
  const int fg = f / a.FN, fl = f - fg * a.FN;
  uint4 v = make_uint4(0u, 0u, 0u, 0u);
  if (f < a.F) {
    const float* src = K + (static_cast<int64_t>(f) * a.C + 4 * c4) * a.T + t;
    v = make_uint4(f32_to_tf32(__ldg(src)), f32_to_tf32(__ldg(src + a.T)), f32_to_tf32(__ldg(src + 2 * a.T)),
                   f32_to_tf32(__ldg(src + 3 * a.T)));
  }
  const int row = a.tb.tap_slot[t] * a.FN + fl;
  const size_t off = static_cast<size_t>(fg) * a.grp_bytes + static_cast<size_t>(c4 >> 3) * a.T * a.FN * 128 +
                     static_cast<size_t>(row) * 128 + ((((c4 & 7) ^ (row & 7))) << 4);
  *reinterpret_cast<uint4*>(Wp + off) = v;
#ifdef GENSOR_DEV_OVERRIDES
  if ((threadIdx.x & 31) == 0) atomicMax(&g_flat_filt[1], static_cast<unsigned long long>(gtimer()));
#endif
  }
  flat_signal_bank_image(sync);
}

// ---- MMA issue: the table-driven loop (any shape) and the compile-time-specialised one (the op
// table is a template constant: every descriptor offset, N and flag folds into the instruction
// stream; tools/flat_rate.cu measured the table-driven issue at 3.7 k vs 2.6 k cycles per tile)
struct FlatIssueCtx {
  uint64_t* full;
  uint64_t* empty;
  uint64_t* bank_bar;
  uint64_t adesc0, bdesc_ck;
  uint32_t d;
  int it, local, ck;
};

template <int R, int S, int WM, int FN>
struct FlatSpec {
  static constexpr FlatTable t = flat_table(R, S, flat_rep_w(S, WM), FN);
};

template <class TB, int PASS, int G, int I>
__device__ __forceinline__ void flat_op(const FlatIssueCtx& c, uint64_t ad) {
  constexpr int o = TB::t.grp_op0[PASS][G] + I;
  constexpr uint32_t idesc = instr_desc(2, 128, static_cast<uint32_t>(TB::t.op_n[o]), 1, 0);
  constexpr uint32_t dcol = static_cast<uint32_t>(TB::t.op_dcol[o]);
  constexpr uint64_t boff = static_cast<uint64_t>(TB::t.op_brow[o]) * 128 / 16;
  constexpr uint32_t acc0 = TB::t.op_zero[o] ? 0u : 1u;
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) mma_tf32(c.d + dcol, ad + kk * 64, c.bdesc_ck + boff + kk * 2, idesc, kk == 0 ? acc0 : 1u);
}

template <int STAGES, class TB, int PASS, int G, int... I>
__device__ __forceinline__ void flat_stage(FlatIssueCtx& c, std::integer_sequence<int, I...>) {
  const int st = c.it % STAGES;
  mbar_wait(&c.full[st], (c.it / STAGES) & 1);
  if (c.local == 0 && G == 0 && c.ck < kFlatMaxChunks) mbar_wait(&c.bank_bar[c.ck], 0);
  tc_fence_after();
  const uint64_t ad = c.adesc0 + static_cast<uint64_t>(st * (kFlatStage >> 4));
  (flat_op<TB, PASS, G, I>(c, ad), ...);
  mma_commit(&c.empty[st]);
  ++c.it;
}

template <int STAGES, class TB, int PASS, int... G>
__device__ __forceinline__ void flat_chunk(FlatIssueCtx& c, std::integer_sequence<int, G...>) {
  (flat_stage<STAGES, TB, PASS, G>(c, std::make_integer_sequence<int, TB::t.grp_nop[PASS][G]>{}), ...);
}

template <int STAGES, class TB>
__global__ void __launch_bounds__(32 * (2 + 4 * kFlatEpw), 1)
    k_conv_flat(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ ConvFlatArgs a,
                const uint8_t* __restrict__ Wp, float* __restrict__ O, unsigned* sync) {
  constexpr int EPW = kFlatEpw;
  extern __shared__ uint8_t smem_raw[];
  // 1024 B-aligned base derived by pointer arithmetic (keeps the shared state space: LDS/STS)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int FN = a.FN, nck = a.nck;
  const FlatTable& tb = a.tb;
  const uint32_t blk = static_cast<uint32_t>(a.T * FN) * 128;  // one 32-channel chunk of the bank
  uint8_t* bank = smem;
  uint8_t* ring = smem + nck * blk;
  const int nfb = FN / 16;
  float* xbuf = reinterpret_cast<float*>(ring + STAGES * kFlatStage);
  uint64_t* full = reinterpret_cast<uint64_t*>(xbuf + 2 * kFlatNfbh * EPW * 4 * kFlatXFloats);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* bank_bar = acc_empty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bank_bar + kFlatMaxChunks);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // filter group of this CTA and its position-tile stream (the grid is a multiple of FG)
  const int fg = blockIdx.x % a.FG, t_first = blockIdx.x / a.FG, t_step = gridDim.x / a.FG;
  if (threadIdx.x == 0) FL_MARK(0);
  if (threadIdx.x == 0) FL_GT(50);

  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 4 * min(EPW, nfb));  // epilogue warps that own a filter block
    }
    for (int i = 0; i < kFlatMaxChunks; ++i) mbar_init(&bank_bar[i], 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---- producer: per (tile, chunk, offset group) one stage of 4 boxes {32 positions, 32 planes}
    // (the input does not depend on the filter launch: no griddepcontrol.wait here)
    if (elect_one()) {
      tma_prefetch(&mapX);
      int it = 0;
      for (int t = t_first; t < a.total; t += t_step) {
        const int n = t / a.tiles_img;
        const int p0 = (t - n * a.tiles_img) * kFlatStep;
        for (int ck = 0; ck < nck; ++ck) {
          const int plane = n * a.C + ck * 32;
          for (int g = 0; g < tb.ngroups; ++g, ++it) {
            const int st = it % STAGES;
            mbar_wait_sleep(&empty[st], ((it / STAGES) & 1) ^ 1);
            mbar_arrive_expect_tx(&full[st], kFlatStage);
            uint8_t* dst = ring + st * kFlatStage;
            const int x0 = p0 + (tb.group_o[g] & ~3);
#pragma unroll
            for (int m = 0; m < 4; ++m) tma_load_2d(dst + m * 4096, &mapX, &full[st], x0 + 32 * m, plane);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---- MMA issuer. The bank comes from the preceding filter launch: wait for it, then one bulk
    // copy per 32-channel chunk (the first tile's MMAs on chunk 0 start before chunk 1 lands).
    if (elect_one()) {
      flat_wait_bank_image(sync, static_cast<unsigned>(a.filt_blocks));
      for (int ck = 0; ck < nck; ++ck) {
        uint64_t* bb = &bank_bar[ck < kFlatMaxChunks ? ck : kFlatMaxChunks - 1];
        if (ck < kFlatMaxChunks - 1) mbar_arrive_expect_tx(bb, blk);
        else if (ck == kFlatMaxChunks - 1) mbar_arrive_expect_tx(bb, blk * (nck - ck));
        bulk_g2s(bank + ck * blk, Wp + static_cast<size_t>(fg) * a.grp_bytes + static_cast<size_t>(ck) * blk, blk, bb);
      }
      flat_done_with_counter(sync);
      FL_MARK(1);
      FlatIssueCtx c;
      c.full = full;
      c.empty = empty;
      c.bank_bar = bank_bar;
      c.adesc0 = smem_desc_sw128(smem_u32(ring), 4096, 512, 1);
      const uint64_t bdesc0 = smem_desc_sw128(smem_u32(bank), 16, 1024);
      c.it = 0;
      c.local = 0;
      for (int t = t_first; t < a.total; t += t_step, ++c.local) {
        const int acc = c.local & 1;
        mbar_wait(&acc_empty[acc], ((c.local >> 1) & 1) ^ 1);
        if (c.local < 6) FL_MARK(8 + c.local);
        tc_fence_after();
        c.d = tmem + acc * 256;
        for (c.ck = 0; c.ck < nck; ++c.ck) {
          c.bdesc_ck = bdesc0 + ((static_cast<uint64_t>(c.ck) * blk) >> 4);
          if constexpr (!std::is_same_v<TB, void>) {
            if (c.ck == 0)
              flat_chunk<STAGES, TB, 0>(c, std::make_integer_sequence<int, TB::t.ngroups>{});
            else
              flat_chunk<STAGES, TB, 1>(c, std::make_integer_sequence<int, TB::t.ngroups>{});
          } else {
            const int pass = c.ck == 0 ? 0 : 1;
            for (int g = 0; g < tb.ngroups; ++g) {
              const int st = c.it % STAGES;
              mbar_wait(&full[st], (c.it / STAGES) & 1);
              if (c.local == 0 && g == 0 && c.ck < kFlatMaxChunks) mbar_wait(&bank_bar[c.ck], 0);
              tc_fence_after();
              const uint64_t ad = c.adesc0 + static_cast<uint64_t>(st * (kFlatStage >> 4));
              const int o0 = tb.grp_op0[pass][g], o1 = o0 + tb.grp_nop[pass][g];
              for (int o = o0; o < o1; ++o) {
                const uint32_t dc = c.d + tb.op_dcol[o];
                const uint64_t bd = c.bdesc_ck + static_cast<uint64_t>(tb.op_brow[o]) * 8;  // rows * 128 B >> 4
                const uint32_t idesc = instr_desc(2, 128, static_cast<uint32_t>(tb.op_n[o]), 1, 0);
                const uint32_t acc0 = tb.op_zero[o] ? 0u : 1u;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) mma_tf32(dc, ad + kk * 64, bd + kk * 2, idesc, kk == 0 ? acc0 : 1u);
              }
              mma_commit(&empty[st]);
              ++c.it;
            }
          }
        }
        mma_commit(&acc_full[acc]);
        if (c.local < 6) FL_MARK(16 + c.local);
      }
      FL_MARK(40);
    }
    __syncwarp();
  } else {
    // ---- epilogue: warp w owns TMEM lane quarter q = w % 4 (tile rows 32q..32q+31) and the
    // 16-filter blocks fb = h, h + EPW (at most kFlatNfbh); out(j) = sum_b D[lane j + b][block b].
    // All of a warp's blocks are read first (the accumulator is released right away), published,
    // one barrier per tile, then summed and stored.
    const int q = warp & 3, h = (warp - 2) >> 2;
    const int nmine = h < nfb ? (nfb - h + EPW - 1) / EPW : 0;  // this warp's 16-filter blocks
    const int nloop = nmine ? a.total : 0;
    const int plane_out = a.OH * a.OW;
    const uint32_t bm = tb.bmask;
    int local = 0;
    for (int t = t_first; t < nloop; t += t_step, ++local) {
      const int acc = local & 1;
      const int n = t / a.tiles_img;
      const int p0 = (t - n * a.tiles_img) * kFlatStep;
      const int vt = min(kFlatStep, a.PW - p0);
      const int j = q * 32 + lane;
      const int p = p0 + j;
      const int hrow = p / a.W, wcol = p - hrow * a.W;
      const bool ok = j < vt && wcol < a.OW;
      mbar_wait(&acc_full[acc], (local >> 1) & 1);
      if (warp == 2 && lane == 0 && local < 6) FL_MARK(24 + local);
      tc_fence_after();
      uint32_t r[kFlatNfbh][4][16];
#pragma unroll
      for (int x = 0; x < kFlatNfbh; ++x) {
        if (x < nmine) {
          const uint32_t base =
              tmem + acc * 256 + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>((h + x * EPW) * 16);
          if (bm & 1u) tmem_ld16(base, r[x][0]);
          if (bm & 2u) tmem_ld16(base + FN, r[x][1]);
          if (bm & 4u) tmem_ld16(base + 2 * FN, r[x][2]);
          if (bm & 8u) tmem_ld16(base + 3 * FN, r[x][3]);
        }
      }
      tmem_ld_wait();
#pragma unroll
      for (int x = 0; x < kFlatNfbh; ++x)
#pragma unroll
        for (int b = 0; b < 4; ++b) tmem_ld_pin(r[x][b]);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[acc]);  // the accumulator may take tile t + 2 now
      if (warp == 2 && lane == 0 && local == 1) FL_MARK(44);
      if (bm != 15u) {  // blocks no tap lands in are zero (the sums below need no per-block test)
#pragma unroll
        for (int x = 0; x < kFlatNfbh; ++x)
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            if (!(bm & 1u)) r[x][0][i] = 0u;
            if (!(bm & 2u)) r[x][1][i] = 0u;
            if (!(bm & 4u)) r[x][2][i] = 0u;
            if (!(bm & 8u)) r[x][3][i] = 0u;
          }
      }
      // lanes L < 3 publish their blocks b > L (the previous quarter's lanes 32 - b + L need
      // them), then take the NEXT quarter's lane-L values of those blocks into the same registers:
      // after that, block b of output lane l is lane (l + b) & 31 of this warp (records parity-
      // double-buffered; quarter 3's lanes 29..31 are rows >= 125, never stored)
      auto put16 = [&](float* dst, const uint32_t(&v)[16]) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          reinterpret_cast<uint4*>(dst)[k] = make_uint4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
      };
      auto get16 = [&](const float* src, uint32_t(&v)[16]) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint4 y = reinterpret_cast<const uint4*>(src)[k];
          v[4 * k] = y.x, v[4 * k + 1] = y.y, v[4 * k + 2] = y.z, v[4 * k + 3] = y.w;
        }
      };
      float* rec = xbuf + (((local & 1) * EPW + h) * 4) * (kFlatNfbh * kFlatXFloats);
      if (lane < 3) {
#pragma unroll
        for (int x = 0; x < kFlatNfbh; ++x) {
          float* mine = rec + (q * kFlatNfbh + x) * kFlatXFloats;
          if (lane == 0) put16(mine, r[x][1]);
          if (lane < 2) put16(mine + 16 + 16 * lane, r[x][2]);
          put16(mine + 48 + 16 * lane, r[x][3]);
        }
      }
      if (warp == 2 && lane == 0 && local == 1) FL_MARK(46);
      named_bar(1 + h, 128);
      if (warp == 2 && lane == 0 && local == 1) FL_MARK(47);
      if (lane < 3 && q < 3) {
#pragma unroll
        for (int x = 0; x < kFlatNfbh; ++x) {
          const float* nx = rec + ((q + 1) * kFlatNfbh + x) * kFlatXFloats;
          if (lane == 0) get16(nx, r[x][1]);
          if (lane < 2) get16(nx + 16 + 16 * lane, r[x][2]);
          get16(nx + 48 + 16 * lane, r[x][3]);
        }
      }
      if (warp == 2 && lane == 0 && local == 1) FL_MARK(45);
      const int l1 = (lane + 1) & 31, l2 = (lane + 2) & 31, l3 = (lane + 3) & 31;
#pragma unroll
      for (int x = 0; x < kFlatNfbh; ++x) {
        if (x < nmine) {
          const int f0 = fg * FN + (h + x * EPW) * 16;
          float* op = O + (static_cast<int64_t>(n) * a.F + f0) * plane_out + static_cast<int64_t>(hrow) * a.OW + wcol;
          if (a.F - f0 >= 16) {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float v = __uint_as_float(r[x][0][i]) + __shfl_sync(0xffffffffu, __uint_as_float(r[x][1][i]), l1) +
                              __shfl_sync(0xffffffffu, __uint_as_float(r[x][2][i]), l2) +
                              __shfl_sync(0xffffffffu, __uint_as_float(r[x][3][i]), l3);
              if (ok) *op = v;
              op += plane_out;
            }
          } else {
            const int fmax = a.F - f0;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float v = __uint_as_float(r[x][0][i]) + __shfl_sync(0xffffffffu, __uint_as_float(r[x][1][i]), l1) +
                              __shfl_sync(0xffffffffu, __uint_as_float(r[x][2][i]), l2) +
                              __shfl_sync(0xffffffffu, __uint_as_float(r[x][3][i]), l3);
              if (ok && i < fmax) *op = v;
              op += plane_out;
            }
          }
        }
      }
      if (warp == 2 && lane == 0 && local < 6) FL_MARK(32 + local);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
  if (threadIdx.x == 0) FL_GT(51);
}

// ---- conv_flat over a CTA pair (cta_group::2) -------------------------------------------------
// Two CTAs of a cluster own two position tiles; the leader issues UMMA M = 256 (rows 0..127 = its
// tile, 128..255 = the peer's), each CTA holds HALF of every run's filter rows (the UMMA splits B
// by rows across the pair), so the resident bank halves (74 KB instead of 147 KB at the headline),
// the freed shared memory doubles the input ring, and the tensor cores read half the filter bytes
// per output. Protocol: both producers' TMA loads complete on the leader's full barrier (the
// leader registers both halves' bytes); the leader's commits multicast to both CTAs' empty and
// accumulator-full barriers; both CTAs' epilogue warps release the accumulator on the leader's
// barrier. Runs are never split (prezero: the epilogue zeroes the blocks a run would only partly
// find written, flat_table.h), so each run is one UMMA at one bank offset in both passes.
__global__ void __launch_bounds__(128) k_flat_filters_pair(const float* __restrict__ K, uint8_t* __restrict__ Wp,
                                                           const __grid_constant__ ConvFlatArgs a, unsigned* sync) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#ifdef GENSOR_DEV_OVERRIDES
  if (threadIdx.x == 0) atomicMin(&g_flat_filt[0], static_cast<unsigned long long>(gtimer()));
#endif
  const FlatTable& tb = a.tb;
  const int c4n = a.C >> 2;
  const int total = a.FN * c4n * a.T;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < total) {
  const int t = e % a.T;
  const int u = e / a.T;
  const int f = u / c4n, c4 = u - f * c4n;
  uint4 v = make_uint4(0u, 0u, 0u, 0u);
  if (f < a.F) {
    const float* src = K + (static_cast<int64_t>(f) * a.C + 4 * c4) * a.T + t;
    v = make_uint4(f32_to_tf32(__ldg(src)), f32_to_tf32(__ldg(src + a.T)), f32_to_tf32(__ldg(src + 2 * a.T)),
                   f32_to_tf32(__ldg(src + 3 * a.T)));
  }
  const int run = tb.tap_run[t];
  const int rr = tb.tap_rrow[t] + f, nh = tb.run_rows[run] / 2;
  const int half = rr >= nh ? 1 : 0;
  const int row = tb.run_hbase[run] + rr - half * nh;
  const size_t blkh = static_cast<size_t>(tb.half_rows) * 128;
  const size_t off = static_cast<size_t>(half) * a.nck * blkh + static_cast<size_t>(c4 >> 3) * blkh +
                     static_cast<size_t>(row) * 128 + ((((c4 & 7) ^ (row & 7))) << 4);
  *reinterpret_cast<uint4*>(Wp + off) = v;
#ifdef GENSOR_DEV_OVERRIDES
  if ((threadIdx.x & 31) == 0) atomicMax(&g_flat_filt[1], static_cast<unsigned long long>(gtimer()));
#endif
  }
  flat_signal_bank_image(sync);
}

template <int R, int S, int WM, int FN>
struct FlatSpecPair {
  static constexpr FlatTable t = flat_table(R, S, flat_rep_w(S, WM), FN, true);
};

__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra.uni DONE_%=;\n\t"
      "bra.uni WAIT_%=;\n"
      "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive_remote_release(uint64_t* bar, uint32_t cta) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar)),
      "r"(cta)
      : "memory");
}

struct FlatPairCtx {
  uint64_t* full;
  uint64_t* empty;
  uint64_t* bank_bar;
  uint64_t* peer_bar;
  uint64_t adesc0, bdesc_ck;
  uint32_t d;
  int it, local, ck;
};

template <class TB, int PASS, int G, int I>
__device__ __forceinline__ void flat_op_pair(const FlatPairCtx& c, uint64_t ad) {
  constexpr int o = TB::t.grp_op0[PASS][G] + I;
  constexpr uint32_t idesc = instr_desc(2, 256, static_cast<uint32_t>(TB::t.op_n[o]), 1, 0);
  constexpr uint32_t dcol = static_cast<uint32_t>(TB::t.op_dcol[o]);
  constexpr uint64_t boff = static_cast<uint64_t>(TB::t.op_brow[o]) * 128 / 16;
  constexpr uint32_t acc0 = TB::t.op_zero[o] ? 0u : 1u;
#pragma unroll
  for (int kk = 0; kk < 4; ++kk)
    mma_tf32_pair(c.d + dcol, ad + kk * 64, c.bdesc_ck + boff + kk * 2, idesc, kk == 0 ? acc0 : 1u);
}

template <int STAGES, class TB, int PASS, int G, int... I>
__device__ __forceinline__ void flat_stage_pair(FlatPairCtx& c, std::integer_sequence<int, I...>) {
  const int st = c.it % STAGES;
  mbar_wait(&c.full[st], (c.it / STAGES) & 1);
  if (c.local == 0 && G == 0 && c.ck < kFlatMaxChunks) {
    mbar_wait(&c.bank_bar[c.ck], 0);
    if (c.ck == 0) mbar_wait_cluster(c.peer_bar, 0);  // the peer's bank half has landed
  }
  tc_fence_after();
  const uint64_t ad = c.adesc0 + static_cast<uint64_t>(st * (kFlatStage >> 4));
  (flat_op_pair<TB, PASS, G, I>(c, ad), ...);
  mma_commit_pair(&c.empty[st], 3);
  ++c.it;
}

template <int STAGES, class TB, int PASS, int... G>
__device__ __forceinline__ void flat_chunk_pair(FlatPairCtx& c, std::integer_sequence<int, G...>) {
  (flat_stage_pair<STAGES, TB, PASS, G>(c, std::make_integer_sequence<int, TB::t.grp_nop[PASS][G]>{}), ...);
}

template <int STAGES, class TB>
__global__ void __launch_bounds__(32 * (2 + 4 * kFlatEpw), 1)
    k_conv_flat_pair(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ ConvFlatArgs a,
                     const uint8_t* __restrict__ Wp, float* __restrict__ O, unsigned* sync) {
  constexpr int EPW = kFlatEpw;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int FN = a.FN, nck = a.nck;
  const FlatTable& tb = a.tb;
  const uint32_t blkh = static_cast<uint32_t>(tb.half_rows) * 128;  // one chunk of this CTA's bank half
  uint8_t* bank = smem;
  uint8_t* ring = smem + nck * blkh;
  const int nfb = FN / 16;
  float* xbuf = reinterpret_cast<float*>(ring + STAGES * kFlatStage);
  uint64_t* full = reinterpret_cast<uint64_t*>(xbuf + 2 * kFlatNfbh * EPW * 4 * kFlatXFloats);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* bank_bar = acc_empty + 2;
  uint64_t* peer_bar = bank_bar + kFlatMaxChunks;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(peer_bar + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int pairs_total = (a.total + 1) >> 1;
  if (threadIdx.x == 0) FL_MARK(0);
  if (threadIdx.x == 0) FL_GT(50);

  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 2 * 4 * min(EPW, nfb));  // both CTAs' epilogue warps that own a block
    }
    for (int i = 0; i < kFlatMaxChunks; ++i) mbar_init(&bank_bar[i], 1);
    mbar_init(peer_bar, 1);
    fence_barrier_init();
    FL_MARK(5);
  }
  cluster_sync_relaxed();
  if (threadIdx.x == 0) FL_MARK(6);  // both CTAs' barriers initialised before any cross-CTA arrive / TMA completion (init fence: release.cluster)
  if (warp == 1) tmem_alloc_pair<512>(tmem_slot);
  if (threadIdx.x == 32) FL_MARK(7);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) FL_MARK(2);
  const uint32_t tmem = *tmem_slot;
  const int q = warp & 3, h = (warp - 2) >> 2;
  const int nmine = warp >= 2 && h < nfb ? (nfb - h + EPW - 1) / EPW : 0;
  // blocks a run only partly finds written start each tile at zero (the epilogue re-zeroes a
  // buffer right after reading it); the first zeroing of both buffers is the epilogue warps'
  // initial release of the accumulators, so nothing waits on it before the first MMA
  auto prezero = [&](int acc) {
    uint32_t z[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) z[i] = 0u;
    for (int b = 0; b < 4; ++b) {
      if (!(tb.prezero & (1u << b))) continue;
      for (int x = 0; x < nmine; ++x)
        tmem_st16(tmem + acc * 256 + (static_cast<uint32_t>(q * 32) << 16) + b * FN + (h + x * EPW) * 16, z);
    }
    tmem_st_wait();
  };
  auto release = [&](int acc) {  // this warp is done with accumulator buffer acc
    tc_fence_before();
    __syncwarp();
    if (lane == 0) {
      if (leader) mbar_arrive(&acc_empty[acc]);
      else mbar_arrive_remote(&acc_empty[acc], 0);
    }
  };
  if (threadIdx.x == 0) FL_MARK(3);

  if (warp == 0) {
    // ---- producer (each CTA): its tile's stages; completion counted on the leader's full barrier
    if (elect_one()) {
      tma_prefetch(&mapX);
      int it = 0;
      for (int tp = pair; tp < pairs_total; tp += npairs) {
        int t = 2 * tp + static_cast<int>(rank);
        if (t >= a.total) t = a.total - 1;  // odd tile count: the peer recomputes a tile, stores nothing
        const int n = t / a.tiles_img;
        const int p0 = (t - n * a.tiles_img) * kFlatStep;
        for (int ck = 0; ck < nck; ++ck) {
          const int plane = n * a.C + ck * 32;
          for (int g = 0; g < tb.ngroups; ++g, ++it) {
            const int st = it % STAGES;
            mbar_wait_sleep(&empty[st], ((it / STAGES) & 1) ^ 1);
            if (leader) mbar_arrive_expect_tx(&full[st], 2 * kFlatStage);
            uint8_t* dst = ring + st * kFlatStage;
            const int x0 = p0 + (tb.group_o[g] & ~3);
#pragma unroll
            for (int m = 0; m < 4; ++m) tma_load_2d_pair(dst + m * 4096, &mapX, &full[st], x0 + 32 * m, plane);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (elect_one()) {
      flat_wait_bank_image(sync, static_cast<unsigned>(a.filt_blocks));  // W' comes from the preceding launch
      FL_MARK(4);
      const uint8_t* mine = Wp + static_cast<size_t>(rank) * nck * blkh;
      for (int ck = 0; ck < nck; ++ck) {
        uint64_t* bb = &bank_bar[ck < kFlatMaxChunks ? ck : kFlatMaxChunks - 1];
        if (ck < kFlatMaxChunks - 1) mbar_arrive_expect_tx(bb, blkh);
        else if (ck == kFlatMaxChunks - 1) mbar_arrive_expect_tx(bb, blkh * (nck - ck));
        bulk_g2s(bank + ck * blkh, mine + static_cast<size_t>(ck) * blkh, blkh, bb);
      }
      flat_done_with_counter(sync);
      if (!leader) {
        for (int ck = 0; ck < nck && ck < kFlatMaxChunks; ++ck) mbar_wait(&bank_bar[ck], 0);
        mbar_arrive_remote_release(peer_bar, 0);  // the leader's MMAs may read this bank half now
      } else {
        FL_MARK(1);
        FlatPairCtx c;
        c.full = full;
        c.empty = empty;
        c.bank_bar = bank_bar;
        c.peer_bar = peer_bar;
        c.adesc0 = smem_desc_sw128(smem_u32(ring), 4096, 512, 1);
        const uint64_t bdesc0 = smem_desc_sw128(smem_u32(bank), 16, 1024);
        c.it = 0;
        c.local = 0;
        for (int tp = pair; tp < pairs_total; tp += npairs, ++c.local) {
          const int acc = c.local & 1;
          mbar_wait(&acc_empty[acc], (c.local >> 1) & 1);  // phase 0 = the epilogue's initial release
          if (c.local < 6) FL_MARK(8 + c.local);
          tc_fence_after();
          c.d = tmem + acc * 256;
          for (c.ck = 0; c.ck < nck; ++c.ck) {
            c.bdesc_ck = bdesc0 + ((static_cast<uint64_t>(c.ck) * blkh) >> 4);
            if (c.ck == 0)
              flat_chunk_pair<STAGES, TB, 0>(c, std::make_integer_sequence<int, TB::t.ngroups>{});
            else
              flat_chunk_pair<STAGES, TB, 1>(c, std::make_integer_sequence<int, TB::t.ngroups>{});
          }
          mma_commit_pair(&acc_full[acc], 3);
          if (c.local < 6) FL_MARK(16 + c.local);
        }
        FL_MARK(40);
      }
    }
    __syncwarp();
  } else {
    // ---- epilogue (each CTA, its own TMEM lanes = its tile): as k_conv_flat, plus the prezero
    // and the release on the leader's accumulator barrier
    const int nloop = nmine ? pairs_total : 0;
    const int plane_out = a.OH * a.OW;
    const uint32_t bm = tb.bmask;
    // tiles of this CTA; the accumulator releases no MMA will wait for (the last two tiles') are
    // skipped, so no remote arrive can be in flight when the pair exits
    const int nlocal = nloop > pair ? (nloop - pair + npairs - 1) / npairs : 0;
    if (nmine) {
      for (int acc = 0; acc < 2 && acc < nlocal; ++acc) {
        if (tb.prezero) prezero(acc);
        release(acc);
      }
    }
    int local = 0;
    for (int tp = pair; tp < nloop; tp += npairs, ++local) {
      const int acc = local & 1;
      int t = 2 * tp + static_cast<int>(rank);
      const bool own = t < a.total;
      if (!own) t = a.total - 1;
      const int n = t / a.tiles_img;
      const int p0 = (t - n * a.tiles_img) * kFlatStep;
      const int vt = min(kFlatStep, a.PW - p0);
      const int j = q * 32 + lane;
      const int p = p0 + j;
      const int hrow = p / a.W, wcol = p - hrow * a.W;
      const bool ok = own && j < vt && wcol < a.OW;
      mbar_wait(&acc_full[acc], (local >> 1) & 1);
      if (warp == 2 && lane == 0 && local < 6) FL_MARK(24 + local);
      FL_WMARK(0);
      tc_fence_after();
      uint32_t r[kFlatNfbh][4][16];
#pragma unroll
      for (int x = 0; x < kFlatNfbh; ++x) {
        if (x < nmine) {
          const uint32_t base =
              tmem + acc * 256 + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>((h + x * EPW) * 16);
          if (bm & 1u) tmem_ld16(base, r[x][0]);
          if (bm & 2u) tmem_ld16(base + FN, r[x][1]);
          if (bm & 4u) tmem_ld16(base + 2 * FN, r[x][2]);
          if (bm & 8u) tmem_ld16(base + 3 * FN, r[x][3]);
        }
      }
      tmem_ld_wait();
#pragma unroll
      for (int x = 0; x < kFlatNfbh; ++x)
#pragma unroll
        for (int b = 0; b < 4; ++b) tmem_ld_pin(r[x][b]);
      FL_WMARK(1);
      if (local + 2 < nlocal) {
        if (tb.prezero) prezero(acc);
        release(acc);  // (no data is published: the TMEM reads are complete, a plain arrive suffices)
      }
      if (bm != 15u) {
#pragma unroll
        for (int x = 0; x < kFlatNfbh; ++x)
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            if (!(bm & 1u)) r[x][0][i] = 0u;
            if (!(bm & 2u)) r[x][1][i] = 0u;
            if (!(bm & 4u)) r[x][2][i] = 0u;
            if (!(bm & 8u)) r[x][3][i] = 0u;
          }
      }
      auto put16 = [&](float* dst, const uint32_t(&v)[16]) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          reinterpret_cast<uint4*>(dst)[k] = make_uint4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
      };
      auto get16 = [&](const float* src, uint32_t(&v)[16]) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint4 y = reinterpret_cast<const uint4*>(src)[k];
          v[4 * k] = y.x, v[4 * k + 1] = y.y, v[4 * k + 2] = y.z, v[4 * k + 3] = y.w;
        }
      };
      float* rec = xbuf + (((local & 1) * EPW + h) * 4) * (kFlatNfbh * kFlatXFloats);
      if (lane < 3) {
#pragma unroll
        for (int x = 0; x < kFlatNfbh; ++x) {
          float* mine = rec + (q * kFlatNfbh + x) * kFlatXFloats;
          if (lane == 0) put16(mine, r[x][1]);
          if (lane < 2) put16(mine + 16 + 16 * lane, r[x][2]);
          put16(mine + 48 + 16 * lane, r[x][3]);
        }
      }
      FL_WMARK(2);
      named_bar(1 + h, 128);
      FL_WMARK(3);
      if (lane < 3 && q < 3) {
#pragma unroll
        for (int x = 0; x < kFlatNfbh; ++x) {
          const float* nx = rec + ((q + 1) * kFlatNfbh + x) * kFlatXFloats;
          if (lane == 0) get16(nx, r[x][1]);
          if (lane < 2) get16(nx + 16 + 16 * lane, r[x][2]);
          get16(nx + 48 + 16 * lane, r[x][3]);
        }
      }
      const int l1 = (lane + 1) & 31, l2 = (lane + 2) & 31, l3 = (lane + 3) & 31;
#pragma unroll
      for (int x = 0; x < kFlatNfbh; ++x) {
        if (x < nmine) {
          const int f0 = (h + x * EPW) * 16;
          float* op = O + (static_cast<int64_t>(n) * a.F + f0) * plane_out + static_cast<int64_t>(hrow) * a.OW + wcol;
          const int fmax = a.F - f0;
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float v = __uint_as_float(r[x][0][i]) + __shfl_sync(0xffffffffu, __uint_as_float(r[x][1][i]), l1) +
                            __shfl_sync(0xffffffffu, __uint_as_float(r[x][2][i]), l2) +
                            __shfl_sync(0xffffffffu, __uint_as_float(r[x][3][i]), l3);
            if (ok && i < fmax) *op = v;
            op += plane_out;
          }
        }
      }
      if (warp == 2 && lane == 0 && local < 6) FL_MARK(32 + local);
      FL_WMARK(4);
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_relaxed();  // the pair's MMAs, TMEM reads and every awaited remote arrival are done
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair<512>(tmem);
  }
  if (threadIdx.x == 0) FL_GT(51);
}

size_t flat_smem(const ConvFlatArgs& a, int stages) {
  const size_t bank = a.pair ? static_cast<size_t>(a.nck) * a.tb.half_rows * 128 : static_cast<size_t>(a.nck) * a.T * a.FN * 128;
  return 1024 + bank + static_cast<size_t>(stages) * kFlatStage +
         static_cast<size_t>(2 * kFlatNfbh * kFlatEpw * 4 * kFlatXFloats) * 4 + (2 * stages + 4 + kFlatMaxChunks + 1) * 8 +
         16;
}

}  // namespace

// Host plan: the tap / op table for this W (flat_table.h), tiling, shared-memory ring depth, and
// whether a compile-time-specialised kernel issues the MMAs (3x3, FN = 64, W >= S + 3: the table
// depends on W mod 4 only).
bool conv_flat_plan(int N, int C, int H, int W, int F, int R, int S, int stride, int sms, ConvFlatArgs& a, int fn_req,
                    bool allow_pair) {
  if (stride != 1 || C % 32 != 0 || F < 1 || F > 64 || R < 1 || S < 1 || R > H || S > W) return false;
  if ((static_cast<int64_t>(H) * W) % 4 != 0) return false;  // plane pitch must be 16 B aligned for TMA
  const int T = R * S;
  if (T > kFlatMaxTaps) return false;
  if (static_cast<int64_t>(N) * C > (int64_t{1} << 31) - 1 || static_cast<int64_t>(H) * W > (int64_t{1} << 30) ||
      static_cast<int64_t>(F) * (H - R + 1) * (W - S + 1) > (int64_t{1} << 31) - 1)
    return false;
  a = ConvFlatArgs{};
  a.N = N, a.C = C, a.H = H, a.W = W, a.F = F, a.R = R, a.S = S;
  a.OH = H - R + 1, a.OW = W - S + 1;
  a.FN = (F + 15) / 16 * 16;
  if (fn_req > 0) {  // filter groups of fn_req filters (the state's level-1 f tile)
    if (fn_req % 16 || fn_req > 64) return false;
    a.FN = std::min(a.FN, fn_req);
  }
  a.FG = (F + a.FN - 1) / a.FN;
  if (a.FG > sms) return false;
  a.T = T;
  a.nck = C / 32;
  a.tb = flat_table(R, S, W, a.FN);
  if (!a.tb.ok) return false;
  a.PW = a.OH * W;
  a.tiles_img = (a.PW + kFlatStep - 1) / kFlatStep;
  a.total = N * a.tiles_img;
  a.sms = sms;
  if (const char* e = dev_env("GENSOR_FLAT_EXP")) a.exp = std::atoi(e);
  a.grp_bytes = static_cast<size_t>(a.nck) * T * a.FN * 128;
  a.sync_off = a.FG * a.grp_bytes;  // the bank images of the FG groups, then the completion counter
  a.ws_bytes = a.sync_off + 256;
  a.filt_blocks = (a.FG * a.FN * (C / 4) * T + 127) / 128;
  a.stages = 0;
  for (int s = 6; s >= 4; --s)
    if (flat_smem(a, s) <= 227 * 1024) {
      a.stages = s;
      break;
    }
  if (a.stages < 4) return false;
  // specialised issue when the op table equals the class representative's (W mod 4)
  a.spec = -1;
  if (R == 3 && S == 3 && ((a.FN == 64 && a.stages == 4) || (a.FN == 32 && a.stages == 6)) && W >= S + 3 &&
      !(a.exp & 2048)) {
    const FlatTable rep = flat_table(R, S, flat_rep_w(S, W & 3), a.FN);
    bool same = rep.ok && rep.ngroups == a.tb.ngroups && rep.bmask == a.tb.bmask;
    for (int g = 0; same && g < rep.ngroups; ++g)
      for (int pass = 0; pass < 2; ++pass) {
        same = same && rep.grp_op0[pass][g] == a.tb.grp_op0[pass][g] && rep.grp_nop[pass][g] == a.tb.grp_nop[pass][g];
        for (int o = rep.grp_op0[pass][g]; same && o < rep.grp_op0[pass][g] + rep.grp_nop[pass][g]; ++o)
          same = rep.op_dcol[o] == a.tb.op_dcol[o] && rep.op_n[o] == a.tb.op_n[o] && rep.op_brow[o] == a.tb.op_brow[o] &&
                 rep.op_zero[o] == a.tb.op_zero[o];
      }
    for (int t = 0; same && t < T; ++t) same = rep.tap_slot[t] == a.tb.tap_slot[t];
    if (same) a.spec = W & 3;
  }
  // CTA pairs (cta_group::2) on the specialised path: the pair table must equal its class
  // representative's as well (the kernel reads the runs, half-bank offsets and prezero blocks)
  if (allow_pair && a.spec >= 0 && a.FN == 64 && a.FG == 1 && a.total >= 2 && !(a.exp & 8192)) {
    const FlatTable tp = flat_table(R, S, W, a.FN, true);
    const FlatTable rp = flat_table(R, S, flat_rep_w(S, W & 3), a.FN, true);
    bool same = tp.ok && rp.ok && tp.ngroups == rp.ngroups && tp.bmask == rp.bmask && tp.prezero == rp.prezero &&
                tp.nruns == rp.nruns && tp.half_rows == rp.half_rows;
    for (int g = 0; same && g < tp.ngroups; ++g)
      for (int pass = 0; pass < 2; ++pass) {
        same = same && tp.grp_op0[pass][g] == rp.grp_op0[pass][g] && tp.grp_nop[pass][g] == rp.grp_nop[pass][g];
        for (int o = tp.grp_op0[pass][g]; same && o < tp.grp_op0[pass][g] + tp.grp_nop[pass][g]; ++o)
          same = tp.op_dcol[o] == rp.op_dcol[o] && tp.op_n[o] == rp.op_n[o] && tp.op_brow[o] == rp.op_brow[o] &&
                 tp.op_zero[o] == rp.op_zero[o];
      }
    for (int t = 0; same && t < T; ++t)
      same = tp.tap_run[t] == rp.tap_run[t] && tp.tap_rrow[t] == rp.tap_rrow[t];
    for (int ri = 0; same && ri < tp.nruns; ++ri)
      same = tp.run_rows[ri] == rp.run_rows[ri] && tp.run_hbase[ri] == rp.run_hbase[ri];
    if (same) {
      ConvFlatArgs b = a;
      b.pair = true;
      b.tb = tp;
      b.stages = flat_smem(b, 8) <= 227 * 1024 ? 8 : flat_smem(b, 6) <= 227 * 1024 ? 6 : 0;
      if (b.stages) a = b;
    }
  }
  return true;
}

void conv_flat_map(const ConvFlatArgs& a, const void* I, CUtensorMap& mapX) {
  // the NCHW input as {H*W positions, N*C planes}: box {32 positions, 32 planes}
  const uint64_t dims[2] = {static_cast<uint64_t>(a.H) * a.W, static_cast<uint64_t>(a.N) * a.C};
  const uint64_t strides[1] = {static_cast<uint64_t>(a.H) * a.W * 4};
  const uint32_t box[2] = {32, 32};
  encode_map(&mapX, false, true, I, 2, dims, strides, box, /*atom32=*/true);
}

void launch_conv_flat(const ConvFlatArgs& a, const CUtensorMap& mapX, const void* K, void* O, void* ws,
                      bool own_ws, cudaStream_t st, Marks& mk) {
  // handle-owned workspaces start zeroed: their completion counter (after the bank image) is used
  unsigned* sync = own_ws ? reinterpret_cast<unsigned*>(static_cast<char*>(ws) + a.sync_off) : nullptr;
  if ((reinterpret_cast<uintptr_t>(ws) & 15) != 0) throw Error(Code::Cuda, "conv_flat: workspace alignment");
  const size_t smem = flat_smem(a, a.stages);
  mk.mark(st);
#ifdef GENSOR_DEV_OVERRIDES
  if (a.exp & 65536) k_flat_marker<<<1, 1, 0, st>>>();  // DEV: globaltimer of the execute's start
#endif
  {
    // the conversion CTAs share SMs with the early-launched conv CTAs (PDL): give them the conv's
    // shared-memory carveout so no SM has to drain and reconfigure before a conv CTA fits
    static const bool carve = [] {
      cudaFuncSetAttribute(k_flat_filters, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      cudaFuncSetAttribute(k_flat_filters_pair, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      return true;
    }();
    (void)carve;
  }
  if (a.pair)
    k_flat_filters_pair<<<a.filt_blocks, 128, 0, st>>>(static_cast<const float*>(K), static_cast<uint8_t*>(ws), a, sync);
  else
    k_flat_filters<<<a.filt_blocks, 128, 0, st>>>(static_cast<const float*>(K), static_cast<uint8_t*>(ws), a, sync);
  check_cuda(cudaGetLastError(), "conv_flat filter launch");
  count_launch();
  const int grid = a.pair ? 2 * std::min((a.total + 1) / 2, a.sms / 2) : a.FG * std::min(a.total, a.sms / a.FG);
  auto launch = [&](auto kern) {
    set_smem_attr(kern, static_cast<int>(smem), "conv_flat smem attribute");
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(32 * (2 + 4 * kFlatEpw));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = 2;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = a.pair ? 2 : 1;
    check_cuda(cudaLaunchKernelEx(&cfg, kern, mapX, a, static_cast<const uint8_t*>(ws), static_cast<float*>(O), sync),
               "conv_flat launch");
    count_launch();
  };
  if (a.pair) {
    auto pick = [&](auto wm) {
      constexpr int WM = decltype(wm)::value;
      if (a.stages == 8)
        launch(k_conv_flat_pair<8, FlatSpecPair<3, 3, WM, 64>>);
      else
        launch(k_conv_flat_pair<6, FlatSpecPair<3, 3, WM, 64>>);
    };
    switch (a.spec) {
      case 0: pick(std::integral_constant<int, 0>{}); break;
      case 1: pick(std::integral_constant<int, 1>{}); break;
      case 2: pick(std::integral_constant<int, 2>{}); break;
      case 3: pick(std::integral_constant<int, 3>{}); break;
      default: throw Error(Code::Unsupported, "conv_flat pair: class");
    }
  } else {
    switch (a.spec < 0 ? -1 : a.spec + (a.FN == 32 ? 4 : 0)) {
      case 0: launch(k_conv_flat<4, FlatSpec<3, 3, 0, 64>>); break;
      case 1: launch(k_conv_flat<4, FlatSpec<3, 3, 1, 64>>); break;
      case 2: launch(k_conv_flat<4, FlatSpec<3, 3, 2, 64>>); break;
      case 3: launch(k_conv_flat<4, FlatSpec<3, 3, 3, 64>>); break;
      case 4: launch(k_conv_flat<6, FlatSpec<3, 3, 0, 32>>); break;
      case 5: launch(k_conv_flat<6, FlatSpec<3, 3, 1, 32>>); break;
      case 6: launch(k_conv_flat<6, FlatSpec<3, 3, 2, 32>>); break;
      case 7: launch(k_conv_flat<6, FlatSpec<3, 3, 3, 32>>); break;
      default:
        switch (a.stages) {
          case 4: launch(k_conv_flat<4, void>); break;
          case 5: launch(k_conv_flat<5, void>); break;
          case 6: launch(k_conv_flat<6, void>); break;
          default: throw Error(Code::Unsupported, "conv_flat: stage count");
        }
    }
  }
  mk.mark(st);
}

}  // namespace gb::dev
