// Developer microbenchmark (not part of the product library): the conv_flat MMA issue pattern in
// isolation (one CTA per SM, MMAs only, smem contents irrelevant), to separate tensor-pipe cost
// from pipeline effects.
//   nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O2 -o tools/flat_rate tools/flat_rate.cu
// Variants: 0 = conv_flat's op table (N 192/64/64/64/192 then 192/128/64/192 per k-step, D blocks
// b*64, 4 rotating 16 KB MN-major A stages, 147 KB K-major bank); 1 = every MMA N=192 at D=0;
// 2 = variant 1 with a fixed A stage; 3 = variant 1 with B rows fixed; 4 = variant 1 with the
// 24 KB-stage / r*4096 A addressing of tools/mma_rate.cu; 5 = variant 0 with A K-major.
#include <cstdio>
#include <cstdlib>

#include "../paper_2502_11407_b200/csrc/kernels/tc_common.cuh"

using namespace gb::dev::tc;

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e = (x);                                                         \
    if (e != cudaSuccess) {                                                      \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));           \
      exit(1);                                                                   \
    }                                                                            \
  } while (0)

struct Op {
  int dcol, n, brow;
};
__constant__ Op c_ops[2][4][3];
__constant__ int c_nop[2][4];

__global__ void k_flat_rate(long long* out, int tiles, int variant) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 32) {
    const uint32_t bank = smem_u32(smem), ring = bank + 147456;
    const uint32_t blk = 73728;
    long long t0 = clock64();
    int it = 0;
    for (int t = 0; t < tiles; ++t) {
      const uint32_t d = tmem + (t & 1) * 256;
      for (int ck = 0; ck < 2; ++ck) {
        const int pass = ck == 0 ? 0 : 1;
        for (int g = 0; g < 4; ++g, ++it) {
          const int st = variant == 2 ? 0 : (it & 3);
          uint32_t a_addr = ring + st * 16384;
          if (variant == 4) a_addr = ring + (it & 1) * 24576 + (g & 1) * 4096;
          for (int o = 0; o < c_nop[pass][g]; ++o) {
            const Op op = c_ops[pass][g][o];
            const bool fixed = variant >= 1 && variant <= 4;
            const uint32_t n = fixed ? 192 : op.n;
            const uint32_t dc = fixed ? d : d + op.dcol;
            const uint32_t b_addr = bank + ck * blk + (variant == 3 ? 0 : op.brow * 128);
            const bool kmaj = variant == 5;
            const uint32_t idesc = instr_desc(2, 128, n, kmaj ? 0 : 1, 0);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t ad = kmaj ? smem_desc_sw128(a_addr + kk * 32, 16, 1024)
                                       : smem_desc_sw128(a_addr + kk * 1024, 4096, 512, 1);
              mma_tf32(dc, ad, smem_desc_sw128(b_addr + kk * 32, 16, 1024), idesc, 1u);
            }
          }
        }
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// variant 6: the same op table as compile-time constants (fully unrolled issue)
template <int DCOL, int N, int BROW>
__device__ __forceinline__ void op4(uint32_t d, uint32_t a_addr, uint32_t b_base) {
  constexpr uint32_t idesc = instr_desc(2, 128, N, 1, 0);
#pragma unroll
  for (int kk = 0; kk < 4; ++kk)
    mma_tf32(d + DCOL, smem_desc_sw128(a_addr + kk * 1024, 4096, 512, 1),
             smem_desc_sw128(b_base + BROW * 128 + kk * 32, 16, 1024), idesc, 1u);
}

__global__ void k_flat_static(long long* out, int tiles) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 32) {
    const uint32_t bank = smem_u32(smem), ring = bank + 147456;
    long long t0 = clock64();
    for (int t = 0; t < tiles; ++t) {
      const uint32_t d = tmem + (t & 1) * 256;
      op4<0, 192, 0>(d, ring, bank);
      op4<128, 64, 192>(d, ring + 16384, bank);
      op4<192, 64, 256>(d, ring + 16384, bank);
      op4<0, 64, 320>(d, ring + 32768, bank);
      op4<0, 192, 384>(d, ring + 49152, bank);
      op4<0, 192, 0>(d, ring, bank + 73728);
      op4<128, 128, 192>(d, ring + 16384, bank + 73728);
      op4<0, 64, 320>(d, ring + 32768, bank + 73728);
      op4<0, 192, 384>(d, ring + 49152, bank + 73728);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  // conv_flat's table for 3x3 over a 58-wide plane (FN = 64): pass 0 = chunk 0, pass 1 = chunk 1
  Op ops[2][4][3] = {{{{0, 192, 0}}, {{128, 64, 192}, {192, 64, 256}}, {{0, 64, 320}}, {{0, 192, 384}}},
                     {{{0, 192, 0}}, {{128, 128, 192}}, {{0, 64, 320}}, {{0, 192, 384}}}};
  int nop[2][4] = {{1, 2, 1, 1}, {1, 1, 1, 1}};
  CK(cudaMemcpyToSymbol(c_ops, ops, sizeof ops));
  CK(cudaMemcpyToSymbol(c_nop, nop, sizeof nop));
  long long* d;
  CK(cudaMalloc(&d, 4096 * sizeof(long long)));
  const int smem = 147456 + 65536 + 1024;
  CK(cudaFuncSetAttribute(k_flat_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int tiles = 64;
  const char* names[] = {"op table", "all N=192 D=0", "N=192, fixed A stage", "N=192, fixed B rows",
                         "N=192, mma_rate A addressing", "op table, A K-major"};
  for (int v = 0; v < 6; ++v) {
    k_flat_rate<<<sms, 64, smem>>>(d, tiles, v);
    CK(cudaDeviceSynchronize());
    long long h[256];
    CK(cudaMemcpy(h, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost));
    double avg = 0;
    for (int i = 0; i < sms; ++i) avg += h[i];
    avg /= sms;
    printf("variant %d (%s): %.0f cycles per tile (36 MMAs: %.1f per MMA)\n", v, names[v], avg / tiles,
           avg / tiles / 36.0);
  }
  CK(cudaFuncSetAttribute(k_flat_static, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k_flat_static<<<sms, 64, smem>>>(d, tiles);
  CK(cudaDeviceSynchronize());
  {
    long long h[256];
    CK(cudaMemcpy(h, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost));
    double avg = 0;
    for (int i = 0; i < sms; ++i) avg += h[i];
    avg /= sms;
    printf("variant 6 (op table, compile-time unrolled): %.0f cycles per tile\n", avg / tiles);
  }
  return 0;
}
