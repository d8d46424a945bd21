// Kernel plans: plain-old-data launch descriptors shared by the host lowering (g++) and the
// sm_100a kernels (nvcc). A plan is the lowered form of one complete schedule state — the
// B200 counterpart of the SPEC's LoopProgram.
#pragma once

#include <stdint.h>

namespace gb {

// State-driven SIMT plan: one CTA per level-1 spatial tile, one thread "slot" per level-L
// thread tile, virtual threads as strided slices inside the thread tile, reduce axes walked in
// the interpreter's order (level-1 chunks staged in shared memory, then deeper levels, then
// scalar loops), guarded iterations skipped.
struct GenericPlan {
  int32_t nsp, nred;           // spatial / reduce axis counts
  int32_t sp[4], red[3];       // op axis index of each spatial / reduce slot
  int64_t ext[8];              // true extent per op axis
  int32_t B[4], T[4], V[4];    // spatial: block tile, thread tile, vthreads (powers of two)
  int32_t tiles[4];            // CTAs along each spatial slot: ceil(extent / B)
  int32_t slots;               // thread tiles per CTA = prod B/T
  int32_t acc;                 // outputs per thread tile = prod T
  int32_t acc_chunks;          // acc / ACC (kernel template width)
  int32_t rounds;              // ceil(slots / blockDim)
  // reduce walk: level-1 chunk digits, then inner digits (levels 2..L, then scalar)
  int32_t outer_radix[3];      // padded / T1 per reduce slot
  int32_t chunk_tile[3];       // T1 per reduce slot
  int32_t n_chunks;            // prod outer_radix
  int32_t n_inner;             // inner digit count
  int32_t inner_slot[12];      // reduce slot of each inner digit (slowest first)
  int32_t inner_radix[12];
  int32_t inner_mul[12];
  int32_t chunk_len;           // prod T1 over reduce slots
  // tensors: 0 = in0, 1 = in1 (if any), 2 = out; affine element coefficients per op axis
  int32_t n_in;
  int64_t coef[3][8];
  int64_t batch_stride[3];
  // shared-memory staging of input boxes (staged = 0: read inputs from global/L2 directly)
  int32_t staged;
  int32_t sm_nd[2];
  int32_t sm_axis[2][4], sm_win[2][4];
  int32_t sm_range[2][4];      // box extent per tensor dim (coordinate range, not distinct count)
  int64_t sm_gdim[2][4];       // true tensor dims (bounds)
  int64_t sm_gstride[2][4];    // global element strides of tensor dims
  int32_t sm_elems[2];
  int32_t sm_base[2];          // element offset of each box in shared memory
  int64_t scoef[2][8];         // shared-memory coefficient per op axis (relative index)
  int64_t stride;              // window stride
  int32_t divisor;             // avgpool: F*F (true window), 0 otherwise
  int32_t block;               // threads per CTA
  int32_t smem_bytes;
  // register-tiled fast paths of the same plan (same tiles, vthreads and reduce order):
  // 0 = the general walk, 1 = gemm (spatial m, n; reduce k), 2 = gemv (spatial m; reduce n)
  int32_t fast;
  int32_t fast_pad;            // gemm: row padding (floats) of the staged k-major A box
};

}  // namespace gb
