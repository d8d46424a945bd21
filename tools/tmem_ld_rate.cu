// Developer probe (not part of the library): TMEM -> register read throughput per SM with 16 warps
// (4 per lane quarter, as conv_flat's epilogue) for tcgen05.ld shapes 32x32b.x16 / .x32 / .x64
// and 16x256b.x4 (same bytes per instruction pair).
//   nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tmem_ld_rate tools/tmem_ld_rate.cu
#include <cstdio>
#include "../paper_2502_11407_b200/csrc/kernels/tc_common.cuh"
using namespace gb::dev::tc;

template <int SHAPE>
__global__ void k_rate(long long* out, unsigned* sink, int iters) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot + (static_cast<uint32_t>((warp & 3) * 32) << 16);
  uint32_t acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const uint32_t col = ((it * 4 + (warp >> 2)) * 64) & 255;
    if constexpr (SHAPE == 0) {  // 4 x 32x32b.x16 = 8 KB per warp
      uint32_t r[4][16];
#pragma unroll
      for (int b = 0; b < 4; ++b) tmem_ld16(tmem + col + b * 16, r[b]);
      tmem_ld_wait();
#pragma unroll
      for (int b = 0; b < 4; ++b) tmem_ld_pin(r[b]);
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int i = 0; i < 16; ++i) acc += r[b][i];
    } else if constexpr (SHAPE == 1) {  // 2 x 32x32b.x32
      uint32_t r[2][32];
#pragma unroll
      for (int b = 0; b < 2; ++b) tmem_ld32(tmem + col + b * 32, r[b]);
      tmem_ld_wait();
#pragma unroll
      for (int b = 0; b < 2; ++b) tmem_ld_pin(r[b]);
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int i = 0; i < 32; ++i) acc += r[b][i];
    } else {  // 16x256b.x8: 16 lanes x 256 bit x 8 = 32 regs per thread... two of them = 8 KB per warp
      uint32_t r[2][32];
#pragma unroll
      for (int h = 0; h < 2; ++h)
        asm volatile(
            "tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
            "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[h][0]), "=r"(r[h][1]), "=r"(r[h][2]), "=r"(r[h][3]), "=r"(r[h][4]), "=r"(r[h][5]), "=r"(r[h][6]),
              "=r"(r[h][7]), "=r"(r[h][8]), "=r"(r[h][9]), "=r"(r[h][10]), "=r"(r[h][11]), "=r"(r[h][12]),
              "=r"(r[h][13]), "=r"(r[h][14]), "=r"(r[h][15]), "=r"(r[h][16]), "=r"(r[h][17]), "=r"(r[h][18]),
              "=r"(r[h][19]), "=r"(r[h][20]), "=r"(r[h][21]), "=r"(r[h][22]), "=r"(r[h][23]), "=r"(r[h][24]),
              "=r"(r[h][25]), "=r"(r[h][26]), "=r"(r[h][27]), "=r"(r[h][28]), "=r"(r[h][29]), "=r"(r[h][30]),
              "=r"(r[h][31])
            : "r"(tmem + col + h * 64 + (h ? (16u << 16) : 0u)));
      tmem_ld_wait();
#pragma unroll
      for (int h = 0; h < 2; ++h) tmem_ld_pin(r[h]);
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int i = 0; i < 32; ++i) acc += r[h][i];
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(slot);
  }
}

int main() {
  long long* d; unsigned* s;
  cudaMalloc(&d, 148 * 8); cudaMalloc(&s, 148 * 512 * 4);
  const int iters = 256;
  const char* names[] = {"4 x 32x32b.x16", "2 x 32x32b.x32", "2 x 16x256b.x8"};
  for (int v = 0; v < 3; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      if (v == 0) k_rate<0><<<148, 512>>>(d, s, iters);
      if (v == 1) k_rate<1><<<148, 512>>>(d, s, iters);
      if (v == 2) k_rate<2><<<148, 512>>>(d, s, iters);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("%s: %s\n", names[v], cudaGetErrorString(e)); return 1; }
    }
    long long h[148];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
    const double bytes = 16.0 * 8192 * iters;  // 16 warps x 8 KB per iteration
    printf("%s: %.0f cycles, %.1f B/clk/SM (%.0f cycles per 128 KB tile)\n", names[v], avg, bytes / avg, 131072.0 / (bytes / avg));
  }
  return 0;
}
