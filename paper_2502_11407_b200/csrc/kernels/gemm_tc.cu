// Tensor-core GEMM family (tcgen05 + TMEM + TMA), instantiated from a constructed GEMM schedule:
//   C[b][m][n] = sum_k A[b][m][k] * B[b][k][n]      (reference layout, op_spec.cpp:154-158)
// One CTA computes one 128 x BN output tile; BN comes from the schedule's level-1 n tile.
//   warp 0      TMA producer: A tile (K-major, 128 B swizzled rows) and B tile (MN-major: B is
//               [K][N] row-major, loaded as 128 B N-chunks x BK rows) into a STAGES-deep ring;
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (kind::tf32 or kind::f16),
//               tcgen05.commit frees each ring slot and finally signals the epilogue;
//   warps 2..5  epilogue: tcgen05.ld 32 lanes x 16 columns -> registers -> global (fp32 or bf16).
#include <cuda_bf16.h>

#include <algorithm>
#include <cudaTypedefs.h>

#include "../host/error.hpp"
#include "common.cuh"
#include "launch.h"
#include "tc_common.cuh"

namespace gb::dev {

namespace {

using namespace tc;

template <typename T>
struct TcTraits;
template <>
struct TcTraits<float> {  // tf32 operands from fp32 memory
  static constexpr uint32_t kFormat = 2;
  static constexpr bool kF16Kind = false;
};
template <>
struct TcTraits<__nv_bfloat16> {
  static constexpr uint32_t kFormat = 1;
  static constexpr bool kF16Kind = true;
};

// 3xTF32 operand split x = hi + lo: the tensor core reads a staged fp32 word as tf32 by dropping
// its 13 low mantissa bits, so hi = trunc_tf32(x) is the staged word itself (no write-back) and
// lo = x - hi (exact in fp32, < 2^-10 |x|) is rounded to tf32 on the bit pattern (sign-magnitude:
// half an ulp added to the magnitude, then the 13 low bits cleared) and staged beside it.
// Measured: 3.7e-7 (max |error| / max |C|) at 1024^3, 4.8e-7 at K = 4096 (tools/x3_error.py);
// a round-to-nearest hi written back measured the same accuracy and 6 % more time (34.9 vs 32.8 us).
__device__ __forceinline__ float round_tf32(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

// Persistent: CTA b walks tiles b, b + grid, ... (n fastest, so consecutive CTAs share A rows in
// L2). The smem ring continues across tiles; two TMEM accumulators let the epilogue of tile i
// overlap the MMAs of tile i+1. Epilogue: tcgen05.ld 32 columns -> registers -> the warp's
// 32-row staging slice in the 128 B-swizzled layout a TMA store expects -> one TMA store per
// 128 B column block (full-line writes; OOB rows/columns clipped by the tensor map).
// CS > 1: clusters of CS CTAs along N work on CS horizontally adjacent tiles in lockstep; every
// CTA TMA-loads 1/CS of the shared A tile and multicasts it to the cluster (A's L2->SM traffic
// divided by CS), stages are released cluster-wide (multicast tcgen05.commit).
template <typename T, typename TOut, int BN, int STAGES, int CS, int SB>
__global__ void __launch_bounds__(192, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
              const __grid_constant__ CUtensorMap mapC, int M, int N, int K, int tiles_m, int tiles_n, int total,
              int a_batched) {
  constexpr int BM = 128;
  constexpr int BK = 128 / sizeof(T);           // K elements per 128 B swizzle row
  constexpr uint32_t A_BYTES = BM * 128;
  constexpr uint32_t B_BYTES = BN * 128;        // BN x BK elements
  constexpr uint32_t STAGE = A_BYTES + B_BYTES;
  constexpr int B_CHUNKS = BN * sizeof(T) / 128;  // 128 B wide N chunks of the MN-major B tile
  constexpr uint32_t ACC_COLS = BN < 32 ? 32 : BN;
  constexpr uint32_t TMEM_COLS = 2 * ACC_COLS;
  constexpr uint32_t IDESC = instr_desc(TcTraits<T>::kFormat, BM, BN, 0, 1);
  constexpr int OUT_BLOCKS = BN * sizeof(TOut) / 128;  // 128 B column blocks of one output row
  constexpr uint32_t STG_WARP = 32 * BN * sizeof(TOut);  // one epilogue warp's 32-row slice

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* staging = smem + STAGES * STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(staging + 4 * SB * STG_WARP);  // SB slices per warp
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;   // [2]
  uint64_t* acc_empty = acc_full + 2;    // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nk = (K + BK - 1) / BK;
  const int per_batch = tiles_m * tiles_n;
  // tile walk: cluster c takes tile groups g = c, c + clusters, ...; rank r of the cluster takes
  // tile (group's m, group's n * CS + r). CS = 1 is the plain persistent walk.
  const int rank = CS > 1 ? static_cast<int>(cluster_ctarank()) : 0;
  const int cid = blockIdx.x / CS, nclusters = gridDim.x / CS;
  const int groups = total / CS;
  auto tile_of = [&](int gi) { return gi * CS + rank; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CS);  // every CTA of the cluster releases each stage
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 4);  // one arrival per epilogue warp
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&mapA);
    tma_prefetch(&mapB);
    tma_prefetch(&mapC);
  }
  if (warp == 1) tmem_alloc<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  if constexpr (CS > 1) cluster_sync_relaxed();  // peers' barriers are initialised before any multicast (init fence: release.cluster)
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      int it = 0;
      for (int gi = cid; gi < groups; gi += nclusters) {
        const int t = tile_of(gi);
        const int b = t / per_batch, mt = (t % per_batch) / tiles_n, nt = t % tiles_n;
        const int m0 = mt * BM, n0 = nt * BN;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&full[s], STAGE);
          uint8_t* a_s = smem + s * STAGE;
          uint8_t* b_s = a_s + A_BYTES;
          if constexpr (CS > 1)  // this CTA's 1/CS row slice of A, to every CTA of the cluster
            tma_load_3d_mc(a_s + rank * (A_BYTES / CS), &mapA, &full[s], kb * BK, m0 + rank * (BM / CS), b * a_batched,
                           static_cast<uint16_t>((1u << CS) - 1));
          else
            tma_load_3d(a_s, &mapA, &full[s], kb * BK, m0, b * a_batched);  // 0: A shared by the batch
#pragma unroll
          for (int j = 0; j < B_CHUNKS; ++j)
            tma_load_3d(b_s + j * (BK * 128), &mapB, &full[s], n0 + j * (128 / (int)sizeof(T)), kb * BK, b);
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      int it = 0, local = 0;
      for (int gi = cid; gi < groups; gi += nclusters, ++local) {
        const int acc = local & 1;
        mbar_wait(&acc_empty[acc], ((local >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * ACC_COLS;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&full[s], (it / STAGES) & 1);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smem + s * STAGE);
          const uint32_t b_addr = a_addr + A_BYTES;
#pragma unroll
          for (int k = 0; k < 4; ++k) {  // 4 MMAs x 32 B of K (tf32 K=8, bf16 K=16)
            const uint64_t ad = smem_desc_sw128(a_addr + k * 32, 16, 1024);
            // MN-major B: bf16 -> SW128 (8-row K groups, SBO 1024); tf32 -> SW128_BASE32B (4-row, SBO 512)
            const uint64_t bd = TcTraits<T>::kF16Kind
                                    ? smem_desc_sw128(b_addr + k * (4096 / sizeof(T)), BK * 128, 1024, 2)
                                    : smem_desc_sw128(b_addr + k * (4096 / sizeof(T)), BK * 128, 512, 1);
            if constexpr (TcTraits<T>::kF16Kind)
              mma_f16(d, ad, bd, IDESC, (kb | k) != 0);
            else
              mma_tf32(d, ad, bd, IDESC, (kb | k) != 0);
          }
          if constexpr (CS > 1)
            mma_commit_mc(&empty[s], static_cast<uint16_t>((1u << CS) - 1));
          else
            mma_commit(&empty[s]);
        }
        mma_commit(&acc_full[acc]);
      }
    }
  } else {
    const int q = warp & 3;  // TMEM lane quarter this warp may access = its 32 tile rows
    // SB = 2: the warp alternates two staging slices, so tile i+1 is written while tile i's TMA
    // stores still read (short k-loops: the epilogue is the critical path)
    int local = 0;
    for (int gi = cid; gi < groups; gi += nclusters, ++local) {
      const int t = tile_of(gi);
      const int acc = local & 1;
      const int b = t / per_batch, mt = (t % per_batch) / tiles_n, nt = t % tiles_n;
      const int m0 = mt * BM, n0 = nt * BN;
      mbar_wait(&acc_full[acc], (local >> 1) & 1);
      tc_fence_after();
      uint8_t* stg = staging + (q * SB + (local % SB)) * STG_WARP;
      if (lane == 0) bulk_wait_read<SB - 1>();  // the stores that last read this slice are done
      __syncwarp();
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t r[32];
        tmem_ld32(tmem + acc * ACC_COLS + (static_cast<uint32_t>(q * 32) << 16) + c, r);
        tmem_ld_wait();
        tmem_ld_pin(r);
        if constexpr (sizeof(TOut) == 4) {  // 32 fp32 = one 128 B block, 8 chunks
          uint8_t* blk = stg + (c / 32) * (32 * 128) + lane * 128;
#pragma unroll
          for (int k = 0; k < 8; ++k)
            *reinterpret_cast<uint4*>(blk + ((k ^ (lane & 7)) << 4)) =
                make_uint4(r[4 * k], r[4 * k + 1], r[4 * k + 2], r[4 * k + 3]);
        } else {  // 32 bf16 = half a 128 B block, 4 chunks
          uint8_t* blk = stg + (c / 64) * (32 * 128) + lane * 128;
          const int k0 = (c % 64) / 8;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            uint32_t p[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(r[8 * k + 2 * v]), __uint_as_float(r[8 * k + 2 * v + 1]));
              p[v] = *reinterpret_cast<uint32_t*>(&h);
            }
            *reinterpret_cast<uint4*>(blk + (((k0 + k) ^ (lane & 7)) << 4)) = make_uint4(p[0], p[1], p[2], p[3]);
          }
        }
      }
      tc_fence_before();
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&acc_empty[acc]);  // TMEM drained into registers/smem
        if (m0 + q * 32 < M) {
#pragma unroll
          for (int j = 0; j < OUT_BLOCKS; ++j)
            if (n0 + j * (128 / (int)sizeof(TOut)) < N)
              tma_store_3d(&mapC, stg + j * (32 * 128), n0 + j * (128 / (int)sizeof(TOut)), m0 + q * 32, b);
        }
        bulk_commit();
      }
    }
    if (lane == 0) bulk_wait_read<0>();  // the staging is read; the global writes retire with the grid
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CS > 1) cluster_sync();  // no CTA leaves while peers may still signal it
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<TMEM_COLS>(tmem);
  }
}

// CTA pairs (cta_group::2): a cluster of two CTAs computes a 256 x BN tile; the leader issues
// UMMA M = 256 (its 128 rows, then the peer's), each CTA stages its own 128 rows of A and HALF of
// the tile's B columns (the UMMA splits B by columns across the pair), so per SM the B bytes
// staged and read per k-block halve. Both producers' TMA loads complete on the leader's full
// barrier; the leader's commits multicast to both CTAs' empty / accumulator-full barriers; both
// CTAs' epilogue warps release an accumulator on the leader's barrier. The epilogue is k_gemm_tc's.
template <typename T, typename TOut, int BN, int STAGES>
__global__ void __launch_bounds__(192, 1)
    k_gemm_tc_pair(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                   const __grid_constant__ CUtensorMap mapC, int M, int N, int K, int tiles_m2, int tiles_n,
                   int total, int a_batched) {
  constexpr int BM = 128;                       // rows per CTA (UMMA M = 2 * BM)
  constexpr int BK = 128 / sizeof(T);
  constexpr uint32_t A_BYTES = BM * 128;
  constexpr uint32_t B_BYTES = (BN / 2) * 128;  // this CTA's half of the B tile
  constexpr uint32_t STAGE = A_BYTES + B_BYTES;
  constexpr int B_CHUNKS = (BN / 2) * sizeof(T) / 128;
  static_assert(B_CHUNKS >= 1, "pair B half must hold whole 128 B column chunks");
  constexpr uint32_t ACC_COLS = BN;
  constexpr uint32_t TMEM_COLS = 2 * ACC_COLS;
  constexpr uint32_t IDESC = instr_desc(TcTraits<T>::kFormat, 2 * BM, BN, 0, 1);
  constexpr int OUT_BLOCKS = BN * sizeof(TOut) / 128;
  constexpr uint32_t STG_WARP = 32 * BN * sizeof(TOut);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* staging = smem + STAGES * STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(staging + 4 * STG_WARP);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nk = (K + BK - 1) / BK;
  const int per_batch = tiles_m2 * tiles_n;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 8);  // the four epilogue warps of both CTAs
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&mapA);
    tma_prefetch(&mapB);
    tma_prefetch(&mapC);
  }
  cluster_sync_relaxed();  // both CTAs' barriers initialised before any cross-CTA completion (init fence: release.cluster)
  if (warp == 1) tmem_alloc_pair<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      int it = 0;
      for (int t = pair; t < total; t += npairs) {
        const int b = t / per_batch, mt = (t % per_batch) / tiles_n, nt = t % tiles_n;
        const int m0 = mt * 2 * BM + static_cast<int>(rank) * BM, n0 = nt * BN + static_cast<int>(rank) * (BN / 2);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
          if (leader) mbar_arrive_expect_tx(&full[s], 2 * STAGE);
          uint8_t* a_s = smem + s * STAGE;
          uint8_t* b_s = a_s + A_BYTES;
          tma_load_3d_pair(a_s, &mapA, &full[s], kb * BK, m0, b * a_batched);
#pragma unroll
          for (int j = 0; j < B_CHUNKS; ++j)
            tma_load_3d_pair(b_s + j * (BK * 128), &mapB, &full[s], n0 + j * (128 / (int)sizeof(T)), kb * BK, b);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (leader && elect_one()) {
      int it = 0, local = 0;
      for (int t = pair; t < total; t += npairs, ++local) {
        const int acc = local & 1;
        mbar_wait(&acc_empty[acc], ((local >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * ACC_COLS;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&full[s], (it / STAGES) & 1);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smem + s * STAGE);
          const uint32_t b_addr = a_addr + A_BYTES;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t ad = smem_desc_sw128(a_addr + k * 32, 16, 1024);
            const uint64_t bd = TcTraits<T>::kF16Kind
                                    ? smem_desc_sw128(b_addr + k * (4096 / sizeof(T)), BK * 128, 1024, 2)
                                    : smem_desc_sw128(b_addr + k * (4096 / sizeof(T)), BK * 128, 512, 1);
            if constexpr (TcTraits<T>::kF16Kind)
              mma_f16_pair(d, ad, bd, IDESC, (kb | k) != 0);
            else
              mma_tf32_pair(d, ad, bd, IDESC, (kb | k) != 0);
          }
          mma_commit_pair(&empty[s], 3);
        }
        mma_commit_pair(&acc_full[acc], 3);
      }
    }
    __syncwarp();
  } else {
    const int q = warp & 3;
    // the MMA of tile i + 2 waits for tile i's release: the last two tiles' releases are skipped,
    // so no remote arrive can be in flight when the pair exits
    const int nlocal = total > pair ? (total - pair + npairs - 1) / npairs : 0;
    int local = 0;
    for (int t = pair; t < total; t += npairs, ++local) {
      const int acc = local & 1;
      const int b = t / per_batch, mt = (t % per_batch) / tiles_n, nt = t % tiles_n;
      const int m0 = mt * 2 * BM + static_cast<int>(rank) * BM, n0 = nt * BN;
      mbar_wait(&acc_full[acc], (local >> 1) & 1);
      tc_fence_after();
      uint8_t* stg = staging + q * STG_WARP;
      if (lane == 0) bulk_wait_read<0>();
      __syncwarp();
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t r[32];
        tmem_ld32(tmem + acc * ACC_COLS + (static_cast<uint32_t>(q * 32) << 16) + c, r);
        tmem_ld_wait();
        tmem_ld_pin(r);
        if constexpr (sizeof(TOut) == 4) {
          uint8_t* blk = stg + (c / 32) * (32 * 128) + lane * 128;
#pragma unroll
          for (int k = 0; k < 8; ++k)
            *reinterpret_cast<uint4*>(blk + ((k ^ (lane & 7)) << 4)) =
                make_uint4(r[4 * k], r[4 * k + 1], r[4 * k + 2], r[4 * k + 3]);
        } else {
          uint8_t* blk = stg + (c / 64) * (32 * 128) + lane * 128;
          const int k0 = (c % 64) / 8;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            uint32_t p[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(r[8 * k + 2 * v]), __uint_as_float(r[8 * k + 2 * v + 1]));
              p[v] = *reinterpret_cast<uint32_t*>(&h);
            }
            *reinterpret_cast<uint4*>(blk + (((k0 + k) ^ (lane & 7)) << 4)) = make_uint4(p[0], p[1], p[2], p[3]);
          }
        }
      }
      tc_fence_before();
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        if (local + 2 < nlocal) {
          if (leader) mbar_arrive(&acc_empty[acc]);
          else mbar_arrive_remote(&acc_empty[acc], 0);
        }
        if (m0 + q * 32 < M) {
#pragma unroll
          for (int j = 0; j < OUT_BLOCKS; ++j)
            if (n0 + j * (128 / (int)sizeof(TOut)) < N)
              tma_store_3d(&mapC, stg + j * (32 * 128), n0 + j * (128 / (int)sizeof(TOut)), m0 + q * 32, b);
        }
        bulk_commit();
      }
    }
    if (lane == 0) bulk_wait_read<0>();  // the staging is read; the global writes retire with the grid
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_relaxed();  // the pair's MMAs, commits and every awaited remote arrival are done
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair<TMEM_COLS>(tmem);
  }
}

// fp32-grade GEMM on the tf32 tensor cores ("3xTF32"), C = A.B with fp32 storage:
//   warp 0      TMA producer (plain FLOAT32 maps: the fp32 bits land untouched);
//   warps 2..5  converters: every staged element x -> hi = tf32(x) in place, lo = tf32(x - hi)
//               into a mirror buffer of the same swizzled layout (x - hi is exact in fp32);
//   warp 1      MMA issuer: per k-step A_lo.B_hi + A_hi.B_lo into the SMALL partial and
//               A_hi.B_hi into the BIG partial, both fresh for every 128-byte k-block;
//   warps 6..9  accumulators: after each k-block, big + small from TMEM -> fp32 registers.
// The tensor core's fp32 accumulation does not round to nearest (measured: 9e-6 normwise at
// K = 1024 when all 384 MMAs of a row accumulate in TMEM), so TMEM only ever holds one k-block
// (32 products per partial) and the k-blocks are summed in registers with IEEE adds; the
// dropped A_lo.B_lo term is < 2^-22 |a b|. Partials double-buffer in TMEM (4 x 64 columns).
template <int STAGES>
__global__ void __launch_bounds__(320, 1)
    k_gemm_x3(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
              const __grid_constant__ CUtensorMap mapC, int M, int N, int K, int tiles_m, int tiles_n, int total,
              int dbg) {
  constexpr int BM = 128, BN = 64, BK = 32;
  constexpr uint32_t A_BYTES = BM * 128, B_BYTES = BN * 128;
  constexpr uint32_t STAGE = A_BYTES + B_BYTES;     // hi half; the lo mirror follows
  constexpr uint32_t STAGE_BYTES = 2 * STAGE;
  constexpr uint32_t IDESC = instr_desc(2, BM, BN, 0, 1);
  constexpr uint32_t STG_WARP = 32 * BN * 4;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* staging = smem + STAGES * STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(staging + 4 * STG_WARP);
  uint64_t* empty = full + STAGES;
  uint64_t* split = empty + STAGES;   // [STAGES] converted (4 converter warps)
  uint64_t* pfull = split + STAGES;   // [2] partials of a k-block written (MMA commit)
  uint64_t* pempty = pfull + 2;       // [2] partials read (4 accumulator warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = (K + BK - 1) / BK;
  const int per_batch = tiles_m * tiles_n;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&split[s], 4);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&pfull[i], 1);
      mbar_init(&pempty[i], 4);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&mapA);
    tma_prefetch(&mapB);
    tma_prefetch(&mapC);
  }
  if (warp == 1) tmem_alloc<256>(tmem_slot);  // partial p: big at 128p, small at 128p + 64
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      int it = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const int b = t / per_batch, m0 = ((t % per_batch) / tiles_n) * BM, n0 = (t % tiles_n) * BN;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[s], STAGE);
          uint8_t* a_s = smem + s * STAGE_BYTES;
          tma_load_3d(a_s, &mapA, &full[s], kb * BK, m0, b);
#pragma unroll
          for (int j = 0; j < BN * 4 / 128; ++j)
            tma_load_3d(a_s + A_BYTES + j * (BK * 128), &mapB, &full[s], n0 + j * 32, kb * BK, b);
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      int it = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x)
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % STAGES, p = it & 1;
          mbar_wait(&pempty[p], ((it >> 1) & 1) ^ 1);
          mbar_wait(&split[s], (it / STAGES) & 1);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smem + s * STAGE_BYTES), b_addr = a_addr + A_BYTES;
          const uint32_t big = tmem + 128 * p, small = big + 64;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t ad = smem_desc_sw128(a_addr + k * 32, 16, 1024);
            const uint64_t bd = smem_desc_sw128(b_addr + k * 1024, BK * 128, 512, 1);
            const uint64_t ad_lo = smem_desc_sw128(a_addr + STAGE + k * 32, 16, 1024);
            const uint64_t bd_lo = smem_desc_sw128(b_addr + STAGE + k * 1024, BK * 128, 512, 1);
            if (!(dbg & 1)) {
              mma_tf32(small, ad_lo, bd, IDESC, k != 0);
              mma_tf32(small, ad, bd_lo, IDESC, 1u);
            }
            mma_tf32(big, ad, bd, IDESC, k != 0);
          }
          mma_commit(&empty[s]);
          mma_commit(&pfull[p]);
        }
    }
  } else if (warp < 6) {
    // converters (warps 2..5): split the stage once the TMA has landed it
    const int ct = threadIdx.x - 64;
    int it = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x)
      for (int kb = 0; kb < nk; ++kb, ++it) {
        const int s = it % STAGES;
        mbar_wait(&full[s], (it / STAGES) & 1);
        float4* hi = reinterpret_cast<float4*>(smem + s * STAGE_BYTES);
        float4* lo = reinterpret_cast<float4*>(smem + s * STAGE_BYTES + STAGE);
#pragma unroll 4
        for (int i = ct; i < static_cast<int>(STAGE / 16); i += 128) {
          // hi = trunc_tf32(x) is the staged word itself; only lo is stored (see round_tf32)
          const float4 v = hi[i];
          float4 l;
          l.x = round_tf32(v.x - __uint_as_float(__float_as_uint(v.x) & 0xffffe000u));
          l.y = round_tf32(v.y - __uint_as_float(__float_as_uint(v.y) & 0xffffe000u));
          l.z = round_tf32(v.z - __uint_as_float(__float_as_uint(v.z) & 0xffffe000u));
          l.w = round_tf32(v.w - __uint_as_float(__float_as_uint(v.w) & 0xffffe000u));
          if (dbg & 2) continue;  // developer: leave the stage untouched
          lo[i] = l;
        }
        fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core's reads
        __syncwarp();
        if (lane == 0) mbar_arrive(&split[s]);
      }
  } else {
    // accumulators (warps 6..9 -> TMEM lane quarters 2, 3, 0, 1): sum the k-block partials
    const int q = warp & 3;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    int it = 0, local = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++local) {
      const int b = t / per_batch, m0 = ((t % per_batch) / tiles_n) * BM, n0 = (t % tiles_n) * BN;
      float acc[BN];
#pragma unroll
      for (int j = 0; j < BN; ++j) acc[j] = 0.0f;
      for (int kb = 0; kb < nk; ++kb, ++it) {
        const int p = it & 1;
        mbar_wait(&pfull[p], (it >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          uint32_t rb[16], rs[16];
          tmem_ld16(tmem + 128 * p + lane_off + 16 * h, rb);
          tmem_ld16(tmem + 128 * p + 64 + lane_off + 16 * h, rs);
          tmem_ld_wait();
          tmem_ld_pin(rb);
          tmem_ld_pin(rs);
          if (dbg & 1)
#pragma unroll
            for (int j = 0; j < 16; ++j) rs[j] = 0u;
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[16 * h + j] += __uint_as_float(rb[j]) + __uint_as_float(rs[j]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&pempty[p]);
      }
      // store: the warp's 32 rows x 64 fp32 through a 128 B-swizzled staging slice, TMA store
      uint8_t* stg = staging + (warp - 6) * STG_WARP;
      if (lane == 0) bulk_wait_read<0>();
      __syncwarp();
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint8_t* blk = stg + c * (32 * 128) + lane * 128;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          *reinterpret_cast<float4*>(blk + ((k ^ (lane & 7)) << 4)) =
              make_float4(acc[32 * c + 4 * k], acc[32 * c + 4 * k + 1], acc[32 * c + 4 * k + 2], acc[32 * c + 4 * k + 3]);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        if (m0 + q * 32 < M) {
#pragma unroll
          for (int c = 0; c < 2; ++c)
            if (n0 + c * 32 < N) tma_store_3d(&mapC, stg + c * (32 * 128), n0 + c * 32, m0 + q * 32, b);
        }
        bulk_commit();
      }
    }
    if (lane == 0) bulk_wait_read<0>();  // the staging is read; the global writes retire with the grid
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<256>(tmem);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    check_cuda(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q), "driver entry point");
    if (!p || q != cudaDriverEntryPointSuccess) throw Error(Code::Cuda, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

template <int STAGES>
void run_x3(const GemmTcArgs& a, const GemmTcMaps& m, cudaStream_t st) {
  const size_t smem = STAGES * 2 * (128 * 128 + 64 * 128) + 4 * 32 * 64 * 4 + 1024 + 256;
  auto kern = k_gemm_x3<STAGES>;
  set_smem_attr(kern, static_cast<int>(smem), "gemm_x3 smem attribute");
  const int tiles_m = (a.M + 127) / 128, tiles_n = (a.N + 63) / 64;
  const int total = tiles_m * tiles_n * a.batch;
  const int dbg = dev_env("GENSOR_X3_DBG") ? std::atoi(dev_env("GENSOR_X3_DBG")) : 0;
  kern<<<std::min(total, a.sms), 320, smem, st>>>(m.A, m.B, m.C, a.M, a.N, a.K, tiles_m, tiles_n, total, dbg);
  check_cuda(cudaGetLastError(), "gemm_x3 launch");
  count_launch();
}

template <typename T, typename TOut, int BN, int STAGES, int CS, int SB = 1>
void run_cs(const GemmTcArgs& a, const GemmTcMaps& m, cudaStream_t st) {
  constexpr uint32_t STAGE = 128 * 128 + BN * 128;
  const size_t smem = STAGES * STAGE + SB * 4 * 32 * BN * sizeof(TOut) + 1024 + 256;
  auto kern = k_gemm_tc<T, TOut, BN, STAGES, CS, SB>;
  set_smem_attr(kern, static_cast<int>(smem), "gemm_tc smem attribute");
  const int tiles_m = (a.M + 127) / 128, tiles_n = (a.N + BN - 1) / BN;
  const int total = tiles_m * tiles_n * a.batch;
  if constexpr (CS == 1) {
    const int grid = std::min(total, a.sms);
    kern<<<grid, 192, smem, st>>>(m.A, m.B, m.C, a.M, a.N, a.K, tiles_m, tiles_n, total, a.a_shared ? 0 : 1);
    check_cuda(cudaGetLastError(), "gemm_tc launch");
  } else {
    const int grid = std::min(total, a.sms / CS * CS);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(192);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    check_cuda(cudaLaunchKernelEx(&cfg, kern, m.Am, m.B, m.C, a.M, a.N, a.K, tiles_m, tiles_n, total,
                                  a.a_shared ? 0 : 1),
               "gemm_tc cluster launch");
  }
  count_launch();
}

template <typename T, typename TOut, int BN, int STAGES>
void run_pair(const GemmTcArgs& a, const GemmTcMaps& m, cudaStream_t st) {
  constexpr uint32_t STAGE = 128 * 128 + (BN / 2) * 128;
  const size_t smem = STAGES * STAGE + 4 * 32 * BN * sizeof(TOut) + 1024 + 256;
  auto kern = k_gemm_tc_pair<T, TOut, BN, STAGES>;
  set_smem_attr(kern, static_cast<int>(smem), "gemm_tc pair smem attribute");
  const int tiles_m2 = (a.M + 255) / 256, tiles_n = (a.N + BN - 1) / BN;
  const int total = tiles_m2 * tiles_n * a.batch;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * std::min(total, a.sms / 2));
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  check_cuda(cudaLaunchKernelEx(&cfg, kern, m.A, m.B, m.C, a.M, a.N, a.K, tiles_m2, tiles_n, total,
                                a.a_shared ? 0 : 1),
             "gemm_tc pair launch");
  count_launch();
}

// Cluster multicast of A pays when the k-loop is long (A re-read from L2 for every n-tile) and
// the n-tiles split into whole clusters; CS = cluster size along N.
template <typename T, typename TOut, int BN, int STAGES>
void run(const GemmTcArgs& a, const GemmTcMaps& m, cudaStream_t st) {
  const int tiles_n = (a.N + BN - 1) / BN;
  constexpr size_t STAGE = 128 * 128 + BN * 128;
  constexpr size_t STG = 4 * 32 * BN * sizeof(TOut);
  const int nk = (a.K + (128 / (int)sizeof(T)) - 1) / (128 / (int)sizeof(T));
  if constexpr (2 * STAGE + 2 * STG + 2048 <= 227 * 1024) {
    if (nk <= 2 && a.cs == 1) {  // epilogue-bound: double-buffered staging, 2 pipeline stages
      run_cs<T, TOut, BN, 2, 1, 2>(a, m, st);
      return;
    }
  }
  if constexpr ((BN / 2) * sizeof(T) >= 128) {
    if (a.pair) {
      constexpr size_t PSTAGE = 128 * 128 + (BN / 2) * 128;
      constexpr int FIT = static_cast<int>((227 * 1024 - 2048 - STG) / PSTAGE);
      constexpr int PS = FIT >= 8 ? 8 : FIT >= 6 ? 6 : 4;
      static_assert(FIT >= 4, "gemm_tc pair stages do not fit shared memory");
      run_pair<T, TOut, BN, PS>(a, m, st);
      return;
    }
  }
  if (a.cs == 4 && tiles_n % 4 == 0)
    run_cs<T, TOut, BN, STAGES, 4>(a, m, st);
  else if (a.cs >= 2 && tiles_n % 2 == 0)
    run_cs<T, TOut, BN, STAGES, 2>(a, m, st);
  else
    run_cs<T, TOut, BN, STAGES, 1>(a, m, st);
}

// Pipeline depth: the plan's stage count (from the schedule), capped by what fits next to the
// epilogue staging (227 KB opt-in) and by the k-loop length.
template <typename T, typename TOut, int BN>
void run_bn(const GemmTcArgs& a, const GemmTcMaps& m, cudaStream_t st) {
  constexpr size_t STAGE = 128 * 128 + BN * 128;
  constexpr size_t STG = 4 * 32 * BN * sizeof(TOut);
  constexpr int MAXS = static_cast<int>((227 * 1024 - 2048 - STG) / STAGE);
  static_assert(MAXS >= 2, "gemm_tc tile does not fit shared memory");
  const int stages = std::min(MAXS, gemm_tc_stages(a));
  if (stages >= 8)
    run<T, TOut, BN, 8>(a, m, st);
  else if (stages >= 6)
    run<T, TOut, BN, 6>(a, m, st);
  else if (stages >= 4)
    run<T, TOut, BN, 4>(a, m, st);
  else if (stages >= 3)
    run<T, TOut, BN, 3>(a, m, st);
  else
    run<T, TOut, BN, 2>(a, m, st);
}

}  // namespace

void encode_map_swizzle(CUtensorMap* map, bool bf16, bool tf32, const void* ptr, int rank, const uint64_t* dims,
                        const uint64_t* strides_bytes, const uint32_t* box, CUtensorMapSwizzle swizzle) {
  uint32_t elem_strides[5] = {1, 1, 1, 1, 1};
  CUtensorMapDataType dt = bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                : (tf32 ? CU_TENSOR_MAP_DATA_TYPE_TFLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32);
  CUresult r = encode_fn()(map, dt, rank, const_cast<void*>(ptr), dims, strides_bytes, box, elem_strides,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(Code::Cuda, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
}

void encode_map(CUtensorMap* map, bool bf16, bool tf32, const void* ptr, int rank, const uint64_t* dims,
                const uint64_t* strides_bytes, const uint32_t* box, bool atom32) {
  encode_map_swizzle(map, bf16, tf32, ptr, rank, dims, strides_bytes, box,
                     atom32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B);
}

bool gemm_tc_supported(int M, int N, int K, int elem_bytes) {
  return M >= 1 && N >= 1 && K >= 1 && (static_cast<int64_t>(K) * elem_bytes) % 16 == 0 &&
         (static_cast<int64_t>(N) * elem_bytes) % 16 == 0;
}

int gemm_tc_max_stages(int BN, bool bf16, bool x3) {
  const size_t stage = (128 * 128 + static_cast<size_t>(BN) * 128) * (x3 ? 2 : 1);
  const size_t stg = 4 * 32 * static_cast<size_t>(BN) * (bf16 ? 2 : 4);
  return static_cast<int>((227 * 1024 - 2048 - stg) / stage);
}

int gemm_tc_stages(const GemmTcArgs& a) { return std::max(2, std::min(a.stages, 8)); }

void gemm_tc_maps(const GemmTcArgs& a, const void* A, const void* B, void* C, GemmTcMaps& m) {
  const int es = a.bf16 ? 2 : 4;
  const uint32_t bk = 128 / es;
  const uint64_t da[3] = {static_cast<uint64_t>(a.K), static_cast<uint64_t>(a.M),
                          static_cast<uint64_t>(a.a_shared ? 1 : a.batch)};
  const uint64_t sa[2] = {static_cast<uint64_t>(a.K) * es, static_cast<uint64_t>(a.K) * a.M * es};
  const uint32_t ba[3] = {bk, 128, 1};
  // tf32 maps round fp32 to tf32 in flight (TFLOAT32 data type); the 3xTF32 split needs the
  // untouched fp32 bits in shared memory, so its maps load plain FLOAT32
  const bool tf32 = !a.bf16 && !a.x3;
  encode_map(&m.A, a.bf16, tf32, A, 3, da, sa, ba);
  if (a.cs > 1) {  // multicast slices: 128/cs rows per CTA of the cluster
    const uint32_t bam[3] = {bk, static_cast<uint32_t>(128 / a.cs), 1};
    encode_map(&m.Am, a.bf16, tf32, A, 3, da, sa, bam);
  }
  const uint64_t db[3] = {static_cast<uint64_t>(a.N), static_cast<uint64_t>(a.K), static_cast<uint64_t>(a.batch)};
  const uint64_t sb[2] = {static_cast<uint64_t>(a.N) * es, static_cast<uint64_t>(a.N) * a.K * es};
  const uint32_t bb[3] = {bk, bk, 1};  // 128 B of N x BK rows of K
  encode_map(&m.B, a.bf16, tf32, B, 3, db, sb, bb, /*atom32=*/!a.bf16);
  // output map: 128 B column blocks x 32 rows (one epilogue warp's slice)
  const uint64_t dc[3] = {static_cast<uint64_t>(a.N), static_cast<uint64_t>(a.M), static_cast<uint64_t>(a.batch)};
  const uint64_t sc[2] = {static_cast<uint64_t>(a.N) * es, static_cast<uint64_t>(a.N) * a.M * es};
  const uint32_t bc[3] = {static_cast<uint32_t>(128 / es), 32, 1};
  encode_map(&m.C, a.bf16, false, C, 3, dc, sc, bc);
}

void launch_gemm_tc(const GemmTcArgs& a, const GemmTcMaps& m, cudaStream_t st) {
  if (a.x3) {  // fp32-grade 3xTF32: BN = 64 (two operand copies per stage), plain persistent grid
    constexpr int MAXS = static_cast<int>((227 * 1024 - 2048 - 4 * 32 * 64 * 4) / (2 * (128 * 128 + 64 * 128)));
    static_assert(MAXS >= 3, "3xTF32 stages do not fit shared memory");
    if (gemm_tc_stages(a) >= 4 && MAXS >= 4)
      run_x3<(MAXS >= 4 ? 4 : 3)>(a, m, st);
    else
      run_x3<3>(a, m, st);
    return;
  }
  if (a.bf16) {
    switch (a.BN) {
      case 64: run_bn<__nv_bfloat16, __nv_bfloat16, 64>(a, m, st); break;
      case 128: run_bn<__nv_bfloat16, __nv_bfloat16, 128>(a, m, st); break;
      default: run_bn<__nv_bfloat16, __nv_bfloat16, 256>(a, m, st); break;
    }
  } else {
    switch (a.BN) {
      case 64: run_bn<float, float, 64>(a, m, st); break;
      default: run_bn<float, float, 128>(a, m, st); break;
    }
  }
}

}  // namespace gb::dev
