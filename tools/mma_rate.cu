// Developer microbenchmark (not part of the product library): tcgen05.mma issue rate per SM and
// TMA load latency, measured with clock64 inside one CTA per SM.
//   nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O2 -o tools/mma_rate tools/mma_rate.cu -lcuda
// Prints cycles per MMA for kind::tf32 / kind::f16(bf16), M=128, N in {64,128,256}, K-major
// SW128 operands (smem contents irrelevant), and the round trip of one TMA 2-D box load.
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>

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

template <bool BF16, int N, bool BMN = false>
__global__ void k_rate(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  constexpr uint32_t IDESC = instr_desc(BF16 ? 1 : 2, 128, N, 0, BMN ? 1 : 0);
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<256>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 32) {
    const uint32_t a = smem_u32(smem), b = a + 16384;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t ad = smem_desc_sw128(a + k * 32, 16, 1024);
        const uint64_t bd = BMN ? (BF16 ? smem_desc_sw128(b + k * 2048, 4096, 1024, 2)
                                         : smem_desc_sw128(b + k * 1024, 4096, 512, 1))
                                : smem_desc_sw128(b + k * 32, 16, 1024);
        if (BF16)
          mma_f16(tmem, ad, bd, IDESC, 1u);
        else
          mma_tf32(tmem, ad, bd, IDESC, 1u);
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<256>(tmem);
  }
}


// The conv_tc issue pattern: 4 rotating 20 KB A stages, each feeding 3 filter-row shifts (+2 KB)
// x 4 k-steps against a resident 72 KB B bank (distinct operands every MMA).
template <int N, bool MNA>
__global__ void k_rate_conv(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  constexpr uint32_t IDESC = instr_desc(2, 128, N, MNA ? 1 : 0, 0);
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<256>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 32) {
    const uint32_t a = smem_u32(smem), b = a + 4 * 24576;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t as = a + (i & 3) * 24576;
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          mma_tf32(tmem, MNA ? smem_desc_sw128(as + r * 4096 + k * 1024, 4096, 512, 1)
                             : smem_desc_sw128(as + r * 2048 + k * 32, 16, 1024),
                   smem_desc_sw128(b + r * (N * 128) + k * 32, 16, 1024), IDESC, 1u);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<256>(tmem);
  }
}

// Round trip of `k` MMAs + tcgen05.commit -> mbarrier wait, repeated.
__global__ void k_commit_rtt(long long* out, int k, int reps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  constexpr uint32_t IDESC = instr_desc(2, 128, 64, 0, 0);
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<64>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 32) {
    const uint32_t a = smem_u32(smem), b = a + 16384;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      for (int i = 0; i < k; ++i)
        mma_tf32(tmem, smem_desc_sw128(a, 16, 1024), smem_desc_sw128(b, 16, 1024), IDESC, 1u);
      mma_commit(&bar);
      mbar_wait(&bar, r & 1);
    }
    out[blockIdx.x] = (clock64() - t0) / reps;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<64>(tmem);
  }
}

__global__ void k_tma_latency(const __grid_constant__ CUtensorMap map, long long* out, int reps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
    long long best = 1LL << 60, sum = 0;
    for (int r = 0; r < reps; ++r) {
      long long t0 = clock64();
      mbar_arrive_expect_tx(&bar, 16384);
      tma_load_2d(smem, &map, &bar, 0, (blockIdx.x * reps + r) * 128 % 8192);
      mbar_wait(&bar, r & 1);
      long long d = clock64() - t0;
      best = d < best ? d : best;
      sum += d;
    }
    out[2 * blockIdx.x] = best;
    out[2 * blockIdx.x + 1] = sum / reps;
  }
}

template <bool BF16, int N, bool BMN = false>
void rate(long long* d, int sms, const char* name) {
  const int iters = 512;
  CK(cudaFuncSetAttribute(k_rate<BF16, N, BMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  k_rate<BF16, N, BMN><<<sms, 64, 65536>>>(d, iters);
  CK(cudaDeviceSynchronize());
  long long h[256];
  CK(cudaMemcpy(h, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost));
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  const double per = avg / (iters * 4.0);
  const double macs = 128.0 * N * (BF16 ? 16 : 8);
  printf("%s M=128 N=%d: %.1f cycles/MMA, %.0f MAC/clk/SM\n", name, N, per, macs / per);
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  long long* d;
  CK(cudaMalloc(&d, 4096 * sizeof(long long)));
  rate<false, 64>(d, sms, "tf32");
  rate<false, 128>(d, sms, "tf32");
  rate<false, 256>(d, sms, "tf32");
  rate<true, 64>(d, sms, "bf16");
  rate<true, 128>(d, sms, "bf16");
  rate<true, 256>(d, sms, "bf16");
  rate<false, 64, true>(d, sms, "tf32 B MN-major");
  rate<false, 128, true>(d, sms, "tf32 B MN-major");
  rate<true, 64, true>(d, sms, "bf16 B MN-major");
  rate<true, 256, true>(d, sms, "bf16 B MN-major");
  auto conv_rate = [&](auto kern, int n, const char* name) {
    const int iters = 256;
    const int smem = 4 * 24576 + 3 * n * 128;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<sms, 64, smem>>>(d, iters);
    CK(cudaDeviceSynchronize());
    long long h[256];
    CK(cudaMemcpy(h, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost));
    double avg = 0;
    for (int i = 0; i < sms; ++i) avg += h[i];
    printf("tf32 N=%d conv pattern, %s, distinct operands: %.1f cycles/MMA\n", n, name, avg / sms / (iters * 12.0));
  };
  conv_rate(k_rate_conv<64, false>, 64, "A K-major");
  conv_rate(k_rate_conv<64, true>, 64, "A MN-major");
  conv_rate(k_rate_conv<96, true>, 96, "A MN-major");
  conv_rate(k_rate_conv<128, true>, 128, "A MN-major");
  conv_rate(k_rate_conv<192, true>, 192, "A MN-major");
  conv_rate(k_rate_conv<192, false>, 192, "A K-major");
  conv_rate(k_rate_conv<256, true>, 256, "A MN-major");
  for (int k : {0, 1, 4, 12}) {
    CK(cudaFuncSetAttribute(k_commit_rtt, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    k_commit_rtt<<<sms, 64, 65536>>>(d, k, 64);
    CK(cudaDeviceSynchronize());
    long long h[256];
    CK(cudaMemcpy(h, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost));
    double avg = 0;
    for (int i = 0; i < sms; ++i) avg += h[i];
    printf("%d x tf32 MMA(N=64) + commit + wait round trip: %.0f cycles\n", k, avg / sms);
  }
  // TMA latency: 128 rows x 128 B box of an 8192 x 32 fp32 matrix (L2-resident after first touch)
  float* g;
  CK(cudaMalloc(&g, 8192 * 32 * 4));
  CK(cudaMemset(g, 0, 8192 * 32 * 4));
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  CUtensorMap m;
  uint64_t dims[2] = {32, 8192}, strides[1] = {128};
  uint32_t box[2] = {32, 128}, es[2] = {1, 1};
  enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  for (int grid : {1, sms}) {
    CK(cudaFuncSetAttribute(k_tma_latency, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768));
    k_tma_latency<<<grid, 32, 32768>>>(m, d, 64);
    CK(cudaDeviceSynchronize());
    long long h[512];
    CK(cudaMemcpy(h, d, sizeof(long long) * 2 * grid, cudaMemcpyDeviceToHost));
    double best = 0, avg = 0;
    for (int i = 0; i < grid; ++i) best += h[2 * i], avg += h[2 * i + 1];
    printf("TMA 16 KB box round trip (grid %d): best %.0f, mean %.0f cycles\n", grid, best / grid, avg / grid);
  }
  return 0;
}
