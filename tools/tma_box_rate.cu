// Developer probe (not part of the library): TMA throughput of conv_flat's A staging — four 2D
// boxes {32 positions, 32 planes} with the 128 B swizzle (32 B atoms), as the kernel stages one
// tap group — against one 3D box {4 positions, 32 planes, 61 position groups} without swizzle
// (the core-matrix layout a shared stage for all tap groups would need).
//   nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tma_box_rate tools/tma_box_rate.cu -lcuda
#include <cuda.h>
#include <cstdio>
#include "../paper_2502_11407_b200/csrc/kernels/tc_common.cuh"
using namespace gb::dev::tc;

__global__ void k_boxes(const __grid_constant__ CUtensorMap m2, const __grid_constant__ CUtensorMap m3, int mode,
                        int iters, int planes, long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar[4];
  const int S = mode == 0 ? 2 : 4;  // chunks in flight: ~128 KB of staging either way
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int sidx = 0; sidx < S; ++sidx) {
        const int plane = ((blockIdx.x + it * S + sidx) % (planes / 32)) * 32;
        const int x0 = (((it * S + sidx) * 7) % 20) * 124;
        if (mode == 0) {  // 4 tap groups x 4 boxes of 4 KB = 64 KB
          mbar_arrive_expect_tx(&bar[sidx], 65536);
          for (int g = 0; g < 4; ++g)
            for (int m = 0; m < 4; ++m)
              tma_load_2d(smem + sidx * 65536 + g * 16384 + m * 4096, &m2, &bar[sidx], x0 + g * 56 + 32 * m, plane);
        } else {          // one 61-group box = 31232 B
          mbar_arrive_expect_tx(&bar[sidx], 61 * 512);
          asm volatile(
              "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                  smem_u32(smem + sidx * 32768)),
              "l"(&m3), "r"(0), "r"(plane), "r"(x0 / 4), "r"(smem_u32(&bar[sidx]))
              : "memory");
        }
      }
      for (int sidx = 0; sidx < S; ++sidx) mbar_wait(&bar[sidx], it & 1);
    }
    out[blockIdx.x] = (clock64() - t0) / S;  // per chunk
  }
}

int main() {
  const int N = 16, C = 64, H = 58, W = 58;
  float* x;
  cudaMalloc(&x, sizeof(float) * N * C * H * W);
  cudaMemset(x, 0, sizeof(float) * N * C * H * W);
  CUtensorMap m2, m3;
  {
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(H * W), static_cast<cuuint64_t>(N * C)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(H * W * 4)};
    cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&m2, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, x, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("m2 encode %d\n", r); return 1; }
  }
  {
    // {4 positions (16 B), planes, position groups}: group stride 16 B
    cuuint64_t dims[3] = {4, static_cast<cuuint64_t>(N * C), static_cast<cuuint64_t>(H * W / 4)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(H * W * 4), 16};
    cuuint32_t box[3] = {4, 32, 61}, es[3] = {1, 1, 1};
    CUresult r = cuTensorMapEncodeTiled(&m3, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, x, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("m3 encode %d\n", r); return 1; }
  }
  long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(k_boxes, cudaFuncAttributeMaxDynamicSharedMemorySize, 132 * 1024);
  const int iters = 200;
  const char* names[] = {"4 groups x 4 SW128 boxes (64 KB)", "one 3D core-matrix box (31 KB)"};
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 2; ++rep) k_boxes<<<148, 32, 132 * 1024>>>(m2, m3, mode, iters, N * C, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: %s\n", names[mode], cudaGetErrorString(e)); return 1; }
    long long h[148];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148 * iters;
    printf("%s: %.0f cycles per chunk (one CTA per SM, ~128 KB in flight)\n", names[mode], avg);
  }
  return 0;
}
