// Developer probe (not part of the library): semantics and cost of tcgen05.shift on sm_100a.
//   nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tmem_shift_probe tools/tmem_shift_probe.cu
// Each of 4 warps stores value lane*1000 + column into TMEM columns 0..255 of its lane quarter,
// one thread issues tcgen05.shift.cta_group::1.down at column `c0`, a commit waits for it, and the
// block reads back; prints which (lane, column) values moved.
#include <cstdio>
#include "../paper_2502_11407_b200/csrc/kernels/tc_common.cuh"
using namespace gb::dev::tc;

__global__ void k_probe(unsigned* out, int c0, int nshift, long long* cyc) {
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<256>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const int row = warp * 32 + lane;
  for (int cb = 0; cb < 256; cb += 16) {
    uint32_t v[16];
    for (int i = 0; i < 16; ++i) v[i] = row * 1000 + cb + i;
    tmem_st16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + cb, v);
  }
  tmem_st_wait();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    long long t0 = clock64();
    for (int k = 0; k < nshift; ++k)  // nshift > 2: spread over columns (throughput)
      asm volatile("tcgen05.shift.cta_group::1.down [%0];" ::"r"(tmem + (nshift > 2 ? (k * 8) % 256 : c0)) : "memory");
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    cyc[0] = clock64() - t0;
  }
  __syncthreads();
  tc_fence_after();
  for (int cb = 0; cb < 256; cb += 16) {
    uint32_t v[16];
    tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + cb, v);
    tmem_ld_wait();
    for (int i = 0; i < 16; ++i) out[row * 256 + cb + i] = v[i];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<256>(tmem); }
}

int main() {
  unsigned* d; long long* c;
  cudaMalloc(&d, 128 * 256 * 4); cudaMalloc(&c, 8);
  static unsigned h[128 * 256];
  for (int c0 : {0, 32, 64}) for (int ns : {1, 2}) {
    k_probe<<<1, 128>>>(d, c0, ns, c);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("c0 %d: %s\n", c0, cudaGetErrorString(e)); return 1; }
    long long cy; cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    int lo = 999, hi = -1, changed = 0;
    for (int r = 0; r < 128; ++r) for (int col = 0; col < 256; ++col) {
      unsigned v = h[r * 256 + col];
      if (v != unsigned(r * 1000 + col)) { ++changed; lo = col < lo ? col : lo; hi = col > hi ? col : hi; }
    }
    printf("c0 %d nshift %d: %lld cycles, %d changed cells, columns %d..%d\n", c0, ns, cy, changed, lo, hi);
    for (int r : {0, 1, 2, 31, 32, 33, 126, 127}) printf("  row %3d col c0..c0+1: %u %u  col c0+7..8: %u %u\n", r,
        h[r * 256 + c0], h[r * 256 + c0 + 1], h[r * 256 + c0 + 7], h[r * 256 + c0 + 8]);
  }
  for (int ns : {0, 1, 8, 16, 48, 96, 192}) {
    long long best = 1ll << 60;
    for (int rep = 0; rep < 5; ++rep) {
      k_probe<<<1, 128>>>(d, 0, ns, c);
      cudaDeviceSynchronize();
      long long cy; cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
      best = cy < best ? cy : best;
    }
    printf("throughput: %d shifts + commit: %lld cycles\n", ns, best);
  }
  return 0;
}
