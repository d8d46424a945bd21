// Standalone tcgen05/TMA probe (developer tool, not part of the product library).
//   nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O2 -I include -o tools/tc_probe tools/tc_probe.cu
// Runs single-CTA experiments and compares against CPU results:
//   1. TMA SW128 load of a 128x32 fp32 tile: dump raw smem (checks the swizzle mapping)
//   2. tf32 MMA M=128 N=64, A K-major, B K-major
//   3. tf32 MMA M=128 N=64, A K-major, B MN-major
//   4. bf16 MMA M=128 N=64, A K-major, B MN-major
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2502_11407_b200/csrc/kernels/tc_common.cuh"

using namespace gb::dev::tc;

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e = (x);                                                             \
    if (e != cudaSuccess) {                                                          \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

static CUtensorMap map2d(void* ptr, CUtensorMapDataType dt, int es, uint64_t inner, uint64_t outer, uint32_t bi,
                         uint32_t bo, CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
  CUtensorMap m;
  uint64_t dims[2] = {inner, outer};
  uint64_t strides[1] = {inner * es};
  uint32_t box[2] = {bi, bo};
  uint32_t el[2] = {1, 1};
  CUresult r = enc()(&m, dt, 2, ptr, dims, strides, box, el, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("encode failed %d\n", int(r));
  return m;
}

__global__ void k_tma_dump(const __grid_constant__ CUtensorMap m, float* out, int bytes) {
  extern __shared__ uint8_t raw[];
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, bytes);
    tma_load_2d(s, &m, &bar, 0, 0);
  }
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < bytes / 4; i += blockDim.x) out[i] = reinterpret_cast<float*>(s)[i];
}

// A: 128 x K32 (4 B) or 128 x K64 (2 B) K-major tile; B: N64 tile, K-major or MN-major.
template <bool BF16, bool B_MN>
__global__ void k_mma(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb, float* D,
                      uint32_t sbo_b, uint32_t lbo_b, uint32_t layout_b) {
  extern __shared__ uint8_t raw[];
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar, done;
  __shared__ uint32_t slot;
  constexpr int ES = BF16 ? 2 : 4;
  constexpr int BK = 128 / ES;
  uint8_t* sa = s;
  uint8_t* sb = s + 128 * 128;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<64>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, 128 * 128 + 64 * 128);
    tma_load_2d(sa, &ma, &bar, 0, 0);
    if (B_MN) {
      for (int j = 0; j < 64 * ES / 128; ++j) tma_load_2d(sb + j * BK * 128, &mb, &bar, j * BK, 0);
    } else {
      tma_load_2d(sb, &mb, &bar, 0, 0);
    }
  }
  if (warp == 0) {
    mbar_wait(&bar, 0);
    tc_fence_after();
    if (elect_one()) {
      constexpr uint32_t idesc = instr_desc(BF16 ? 1 : 2, 128, 64, 0, B_MN ? 1 : 0);
      for (int k = 0; k < 4; ++k) {
        uint64_t ad = smem_desc_sw128(smem_u32(sa) + k * 32, 16, 1024);
        uint64_t bd = B_MN ? smem_desc_sw128(smem_u32(sb) + k * (4096 / ES), lbo_b, sbo_b)
                           : smem_desc_sw128(smem_u32(sb) + k * 32, 16, 1024);
        if (B_MN && layout_b != 2) bd = (bd & ~(7ull << 61)) | (uint64_t(layout_b) << 61);
        if (BF16)
          mma_f16(tmem, ad, bd, idesc, k > 0);
        else
          mma_tf32(tmem, ad, bd, idesc, k > 0);
      }
      mma_commit(&done);
    }
    __syncwarp();
  }
  mbar_wait(&done, 0);
  tc_fence_after();
  if (warp < 4) {
    for (int c = 0; c < 64; c += 16) {
      uint32_t r[16];
      tmem_ld16(tmem + ((warp * 32) << 16) + c, r);
      tmem_ld_wait();
      for (int v = 0; v < 16; ++v) D[(warp * 32 + threadIdx.x % 32) * 64 + c + v] = __uint_as_float(r[v]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<64>(tmem);
  }
}

template <bool BF16, bool B_MN>
static int run_mma(const char* name, uint32_t sbo_b, uint32_t lbo_b, uint32_t layout_b = 2) {
  constexpr int ES = BF16 ? 2 : 4;
  constexpr int BK = 128 / ES;
  std::vector<float> A(128 * BK), B(BK * 64);
  for (auto& x : A) x = float(rand() % 5 - 2);
  for (auto& x : B) x = float(rand() % 5 - 2);
  // A[m][k] row-major (K-major). B logical [k][n]: K-major storage Bt[n][k]; MN-major storage B[k][n].
  std::vector<uint16_t> Ah(A.size()), Bh(B.size());
  std::vector<float> Bst(B.size());
  for (int k = 0; k < BK; ++k)
    for (int n = 0; n < 64; ++n) Bst[B_MN ? k * 64 + n : n * BK + k] = B[k * 64 + n];
  void *dA, *dB;
  float* dD;
  CK(cudaMalloc(&dA, A.size() * 4));
  CK(cudaMalloc(&dB, B.size() * 4));
  CK(cudaMalloc(&dD, 128 * 64 * 4));
  CK(cudaMemset(dD, 0xff, 128 * 64 * 4));
  if (BF16) {
    std::vector<__nv_bfloat16> a16(A.size()), b16(B.size());
    for (size_t i = 0; i < A.size(); ++i) a16[i] = __float2bfloat16(A[i]);
    for (size_t i = 0; i < B.size(); ++i) b16[i] = __float2bfloat16(Bst[i]);
    CK(cudaMemcpy(dA, a16.data(), A.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, b16.data(), B.size() * 2, cudaMemcpyHostToDevice));
  } else {
    CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, Bst.data(), B.size() * 4, cudaMemcpyHostToDevice));
  }
  CUtensorMapDataType dt = BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_TFLOAT32;
  CUtensorMap ma = map2d(dA, dt, ES, BK, 128, BK, 128);
  CUtensorMap mb = B_MN ? map2d(dB, dt, ES, 64, BK, BK, BK,
                                layout_b == 1 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B)
                        : map2d(dB, dt, ES, BK, 64, BK, 64);
  auto kern = k_mma<BF16, B_MN>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
  kern<<<1, 128, 64 * 1024>>>(ma, mb, dD, sbo_b, lbo_b, layout_b);
  CK(cudaDeviceSynchronize());
  std::vector<float> D(128 * 64);
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 64; ++n) {
      float ref = 0;
      for (int k = 0; k < BK; ++k) ref += A[m * BK + k] * B[k * 64 + n];
      if (D[m * 64 + n] != ref) {
        if (bad < 5) printf("  %s mismatch m=%d n=%d got %g want %g\n", name, m, n, D[m * 64 + n], ref);
        ++bad;
      }
    }
  printf("%s (sbo %u lbo %u layout %u): %s (%d bad)\n", name, sbo_b, lbo_b, layout_b, bad ? "FAIL" : "PASS", bad);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
  return bad;
}

int main() {
  // 1. swizzle dump
  {
    std::vector<float> h(128 * 32);
    for (int i = 0; i < 128 * 32; ++i) h[i] = float(i);
    float *d, *o;
    CK(cudaMalloc(&d, h.size() * 4));
    CK(cudaMalloc(&o, h.size() * 4));
    CK(cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
    CUtensorMap m = map2d(d, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, 32, 128, 32, 128);
    CK(cudaFuncSetAttribute(k_tma_dump, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024));
    k_tma_dump<<<1, 128, 40 * 1024>>>(m, o, 128 * 32 * 4);
    CK(cudaDeviceSynchronize());
    std::vector<float> r(h.size());
    CK(cudaMemcpy(r.data(), o, r.size() * 4, cudaMemcpyDeviceToHost));
    printf("TMA SW128 dump rows 0..2 (16B chunks as first element index):\n");
    for (int row = 0; row < 3; ++row) {
      printf("  row %d:", row);
      for (int ch = 0; ch < 8; ++ch) printf(" %g", r[row * 32 + ch * 4]);
      printf("\n");
    }
    int ok = 1;
    for (int row = 0; row < 128; ++row)
      for (int ch = 0; ch < 8; ++ch)
        for (int e = 0; e < 4; ++e)
          ok &= r[row * 32 + ((ch ^ (row & 7)) * 4) + e] == h[row * 32 + ch * 4 + e];
    printf("swizzle = chunk ^ (row %% 8): %s\n", ok ? "PASS" : "FAIL");
  }
  int bad = 0;
  bad += run_mma<false, false>("tf32 A-K B-K", 1024, 16);
  bad += run_mma<false, true>("tf32 A-K B-MN", 1024, 4096);
  bad += run_mma<false, true>("tf32 A-K B-MN swapped", 4096, 1024);
  bad += run_mma<false, true>("tf32 A-K B-MN base32b", 512, 4096, 1);
  bad += run_mma<false, true>("tf32 A-K B-MN base32b swapped", 4096, 512, 1);
  bad += run_mma<true, false>("bf16 A-K B-K", 1024, 16);
  bad += run_mma<true, true>("bf16 A-K B-MN", 1024, 8192);
  bad += run_mma<true, true>("bf16 A-K B-MN swapped", 8192, 1024);
  printf("done (%d bad)\n", bad);
  return 0;
}
