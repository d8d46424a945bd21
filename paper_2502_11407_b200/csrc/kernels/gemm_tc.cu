// Tensor-core GEMM family (tcgen05 + TMEM + TMA), instantiated from a constructed GEMM schedule:
//   C[b][m][n] = sum_k A[b][m][k] * B[b][k][n]      (reference layout, op_spec.cpp:154-158)
// One CTA computes one 128 x BN output tile; BN comes from the schedule's level-1 n tile.
//   warp 0      TMA producer: A tile (K-major, 128 B swizzled rows) and B tile (MN-major: B is
//               [K][N] row-major, loaded as 128 B N-chunks x BK rows) into a STAGES-deep ring;
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (kind::tf32 or kind::f16),
//               tcgen05.commit frees each ring slot and finally signals the epilogue;
//   warps 2..5  epilogue: tcgen05.ld 32 lanes x 16 columns -> registers -> global (fp32 or bf16).
#include <cuda_bf16.h>
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

template <typename T, typename TOut, int BN, int STAGES>
__global__ void __launch_bounds__(192, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, TOut* __restrict__ C,
              int M, int N, int K) {
  constexpr int BM = 128;
  constexpr int BK = 128 / sizeof(T);           // K elements per 128 B swizzle row
  constexpr uint32_t A_BYTES = BM * 128;
  constexpr uint32_t B_BYTES = BN * 128;        // BN x BK elements
  constexpr uint32_t STAGE = A_BYTES + B_BYTES;
  constexpr int B_CHUNKS = BN * sizeof(T) / 128;  // 128 B wide N chunks of the MN-major B tile
  constexpr uint32_t TMEM_COLS = BN < 32 ? 32 : BN;
  constexpr uint32_t IDESC = instr_desc(TcTraits<T>::kFormat, BM, BN, 0, 1);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * BN;
  const int m0 = blockIdx.y * BM;
  const int b = blockIdx.z;
  const int nk = (K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&mapA);
    tma_prefetch(&mapB);
  }
  if (warp == 1) tmem_alloc<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        const uint32_t ph = (kb / STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], STAGE);
        uint8_t* a_s = smem + s * STAGE;
        uint8_t* b_s = a_s + A_BYTES;
        tma_load_3d(a_s, &mapA, &full[s], kb * BK, m0, b);
#pragma unroll
        for (int j = 0; j < B_CHUNKS; ++j)
          tma_load_3d(b_s + j * (BK * 128), &mapB, &full[s], n0 + j * (128 / (int)sizeof(T)), kb * BK, b);
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        const uint32_t ph = (kb / STAGES) & 1;
        mbar_wait(&full[s], ph);
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
            mma_f16(tmem, ad, bd, IDESC, (kb | k) != 0);
          else
            mma_tf32(tmem, ad, bd, IDESC, (kb | k) != 0);
        }
        mma_commit(&empty[s]);
      }
      mma_commit(tmem_full);
    }
  } else {
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int row = m0 + q * 32 + lane;
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    TOut* crow = C + (static_cast<int64_t>(b) * M + row) * N;
#pragma unroll 1
    for (int c = 0; c < BN; c += 16) {
      uint32_t r[16];
      tmem_ld16(tmem + (static_cast<uint32_t>(q * 32) << 16) + c, r);
      tmem_ld_wait();
      const int n = n0 + c;
      if (row >= M || n >= N) continue;
      if constexpr (sizeof(TOut) == 4) {
        if (n + 16 <= N && (N & 3) == 0) {
          float4* dst = reinterpret_cast<float4*>(crow + n);
#pragma unroll
          for (int v = 0; v < 4; ++v)
            dst[v] = make_float4(__uint_as_float(r[4 * v]), __uint_as_float(r[4 * v + 1]), __uint_as_float(r[4 * v + 2]),
                                 __uint_as_float(r[4 * v + 3]));
        } else {
          for (int v = 0; v < 16 && n + v < N; ++v) crow[n + v] = __uint_as_float(r[v]);
        }
      } else {
        if (n + 16 <= N && (N & 7) == 0) {
          uint32_t p[8];
#pragma unroll
          for (int v = 0; v < 8; ++v) {
            __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(r[2 * v]), __uint_as_float(r[2 * v + 1]));
            p[v] = *reinterpret_cast<uint32_t*>(&h);
          }
          uint4* dst = reinterpret_cast<uint4*>(crow + n);
          dst[0] = make_uint4(p[0], p[1], p[2], p[3]);
          dst[1] = make_uint4(p[4], p[5], p[6], p[7]);
        } else {
          for (int v = 0; v < 16 && n + v < N; ++v) crow[n + v] = __float2bfloat16_rn(__uint_as_float(r[v]));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<TMEM_COLS>(tmem);
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

template <typename T, typename TOut, int BN, int STAGES>
void run(const GemmTcArgs& a, cudaStream_t st) {
  constexpr int BK = 128 / sizeof(T);
  constexpr uint32_t STAGE = 128 * 128 + BN * 128;
  const size_t smem = STAGES * STAGE + 1024 + 256;
  auto kern = k_gemm_tc<T, TOut, BN, STAGES>;
  check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
             "gemm_tc smem attribute");
  dim3 grid((a.N + BN - 1) / BN, (a.M + 127) / 128, a.batch);
  kern<<<grid, 192, smem, st>>>(a.mapA, a.mapB, static_cast<TOut*>(a.C), a.M, a.N, a.K);
  check_cuda(cudaGetLastError(), "gemm_tc launch");
  count_launch();
  (void)BK;
}

template <typename T, typename TOut, int BN>
void run_bn(const GemmTcArgs& a, cudaStream_t st) {
  constexpr uint32_t STAGE = 128 * 128 + BN * 128;
  constexpr int MAXS = static_cast<int>((200 * 1024) / STAGE);
  const int nk = (a.K + (128 / (int)sizeof(T)) - 1) / (128 / (int)sizeof(T));
  if (nk <= 1)
    run<T, TOut, BN, 1>(a, st);
  else if (nk <= 2 || MAXS < 4)
    run<T, TOut, BN, 2>(a, st);
  else if (MAXS < 6)
    run<T, TOut, BN, 4>(a, st);
  else
    run<T, TOut, BN, 6>(a, st);
}

}  // namespace

void encode_map(CUtensorMap* map, bool bf16, bool tf32, const void* ptr, int rank, const uint64_t* dims,
                const uint64_t* strides_bytes, const uint32_t* box, bool atom32) {
  uint32_t elem_strides[5] = {1, 1, 1, 1, 1};
  CUtensorMapDataType dt = bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                : (tf32 ? CU_TENSOR_MAP_DATA_TYPE_TFLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32);
  CUresult r = encode_fn()(map, dt, rank, const_cast<void*>(ptr), dims, strides_bytes, box, elem_strides,
                           CU_TENSOR_MAP_INTERLEAVE_NONE,
                           atom32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(Code::Cuda, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
}

bool gemm_tc_supported(int M, int N, int K, int elem_bytes) {
  return M >= 1 && N >= 1 && K >= 1 && (static_cast<int64_t>(K) * elem_bytes) % 16 == 0 &&
         (static_cast<int64_t>(N) * elem_bytes) % 16 == 0;
}

void launch_gemm_tc(GemmTcArgs& a, const void* A, const void* B, void* C, cudaStream_t st) {
  const int es = a.bf16 ? 2 : 4;
  const uint32_t bk = 128 / es;
  if (A != a.last_A || B != a.last_B) {
    const uint64_t da[3] = {static_cast<uint64_t>(a.K), static_cast<uint64_t>(a.M), static_cast<uint64_t>(a.batch)};
    const uint64_t sa[2] = {static_cast<uint64_t>(a.K) * es, static_cast<uint64_t>(a.K) * a.M * es};
    const uint32_t ba[3] = {bk, 128, 1};
    encode_map(&a.mapA, a.bf16, !a.bf16, A, 3, da, sa, ba);
    const uint64_t db[3] = {static_cast<uint64_t>(a.N), static_cast<uint64_t>(a.K), static_cast<uint64_t>(a.batch)};
    const uint64_t sb[2] = {static_cast<uint64_t>(a.N) * es, static_cast<uint64_t>(a.N) * a.K * es};
    const uint32_t bb[3] = {bk, bk, 1};  // 128 B of N x BK rows of K
    encode_map(&a.mapB, a.bf16, !a.bf16, B, 3, db, sb, bb, /*atom32=*/!a.bf16);
    a.last_A = A;
    a.last_B = B;
  }
  a.C = C;
  if (a.bf16) {
    switch (a.BN) {
      case 64: run_bn<__nv_bfloat16, __nv_bfloat16, 64>(a, st); break;
      case 128: run_bn<__nv_bfloat16, __nv_bfloat16, 128>(a, st); break;
      default: run_bn<__nv_bfloat16, __nv_bfloat16, 256>(a, st); break;
    }
  } else {
    switch (a.BN) {
      case 64: run_bn<float, float, 64>(a, st); break;
      case 128: run_bn<float, float, 128>(a, st); break;
      default: run_bn<float, float, 256>(a, st); break;
    }
  }
}

}  // namespace gb::dev
