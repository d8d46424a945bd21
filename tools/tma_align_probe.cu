// Developer probe: is a TMA tiled load legal when the box starts at a dim-0 coordinate whose byte
// offset is not a 16 B multiple (per swizzle mode)? One case per process.
//   nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tma_align_probe tools/tma_align_probe.cu -lcuda
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include "../paper_2502_11407_b200/csrc/kernels/tc_common.cuh"
using namespace gb::dev::tc;
__global__ void k(const __grid_constant__ CUtensorMap m, int c0, float* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
    mbar_arrive_expect_tx(&bar, 32 * 32 * 4);
    tma_load_2d(smem, &m, &bar, c0, 0);
    mbar_wait(&bar, 0);
    out[0] = reinterpret_cast<float*>(smem)[0];
  }
}
int main(int argc, char** argv) {
  const int sw = atoi(argv[1]), c0 = atoi(argv[2]);
  float* g; cudaMalloc(&g, 1 << 22);
  float* o; cudaMalloc(&o, 4);
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  CUtensorMap m;
  uint64_t dims[2] = {4096, 64}, strides[1] = {4096 * 4};
  uint32_t box[2] = {32, 32}, es[2] = {1, 1};
  CUtensorMapSwizzle s = sw == 0 ? CU_TENSOR_MAP_SWIZZLE_NONE : sw == 1 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, s,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
  k<<<1, 32, 8192>>>(m, c0, o);
  cudaError_t e = cudaDeviceSynchronize();
  printf("swizzle %d coord %d (byte offset %d): encode %d, run %s\n", sw, c0, c0 * 4, int(r), cudaGetErrorString(e));
  return 0;
}
