// Developer microbenchmark: per-launch device time of an (almost) empty kernel vs its dynamic
// shared-memory size, block size and TMEM allocation (events around 100 back-to-back launches).
//   nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O2 -o tools/launch_cost tools/launch_cost.cu
#include <cstdio>
#include <cstdint>
#include "../paper_2502_11407_b200/csrc/kernels/tc_common.cuh"
using namespace gb::dev::tc;
__global__ void k_empty(int* p) { if (threadIdx.x == 0 && blockIdx.x == 100000) p[0] = 1; }
__global__ void k_smem(int* p) {
  extern __shared__ int s[];
  if (threadIdx.x == 0) s[0] = 1;
  __syncthreads();
  if (threadIdx.x == 0 && s[0] == 2) p[0] = 1;
}
__global__ void k_tmem(int* p) {
  __shared__ uint32_t slot;
  if (threadIdx.x < 32) tmem_alloc<256>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc<256>(slot);
  if (threadIdx.x == 0 && slot == 12345) p[0] = 1;
}
template <typename F>
float time_it(F launch) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 10; ++i) launch();
  cudaEventRecord(a);
  for (int i = 0; i < 100; ++i) launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms * 1000.f / 100.f;
}
int main() {
  int* p; cudaMalloc(&p, 4);
  printf("empty 148x192: %.2f us\n", time_it([&] { k_empty<<<148, 192>>>(p); }));
  for (int kb : {0, 48, 100, 200, 227}) {
    cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, kb * 1024);
    printf("smem %3d KB 148x192: %.2f us\n", kb, time_it([&] { k_smem<<<148, 192, kb * 1024>>>(p); }));
  }
  printf("tmem alloc 148x192: %.2f us\n", time_it([&] { k_tmem<<<148, 192>>>(p); }));
  cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  printf("smem 227 KB 148x416: %.2f us\n", time_it([&] { k_smem<<<148, 416, 227 * 1024>>>(p); }));
  return 0;
}
