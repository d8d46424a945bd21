/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the reference's execute step.
 *
 * The reference's executor (src/lowering.cpp: lower / interpret / reference_compute, listed in
 * proj/src/CMakeLists.txt:10) is ABSENT from the snapshot; this file restates it from its spec:
 *   reference_compute  SPEC.md:488-498  naive Table III formulas, alpha=1 beta=0, avgpool / F^2
 *   interpret(lower(s)) SPEC.md:470-487 tiled loop nest, guards skip padded iterations,
 *                                       double accumulation
 * with the tensor layouts of the reference's access maps (op_spec.cpp:150-193) on the TRUE
 * domain (tensor_dims(t,false), op_spec.cpp:227-243; tensor_offset, op_spec.cpp:251-262).
 * Pinned by the SPEC's execute known-answer examples (tests/test_oracle.py).
 * Extension ops (dwconv2d, softmax, batched gemm) have no reference counterpart: parity for
 * them is UNPINNED by the reference and rests on this restatement alone.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference legs may call it.
 */
#ifndef GENSOR_ORACLE_H
#define GENSOR_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORACLE_GEMM = 0, ORACLE_GEMV = 1, ORACLE_CONV2D = 2, ORACLE_AVGPOOL2D = 3, ORACLE_DWCONV2D = 4,
       ORACLE_SOFTMAX = 5 };

typedef struct oracle_op {
  int32_t kind;
  int32_t pad_;
  int64_t M, K, N;                /* gemm: A[M][K] B[K][N] C[M][N]; gemv/softmax: [M][N] */
  int64_t n, c, h, w, f, r, s;    /* conv/pool/dw: I[n][c][h][w], K[f][c][r][s] / [c][r][s]; pool F = r = s */
  int64_t stride;
  int64_t batch;                  /* gemm only: independent repetitions, contiguous */
} oracle_op;

/* Naive formula, lexicographic reduce order, double accumulation. Returns 0 or -1 (bad op). */
int oracle_reference_compute(const oracle_op* op, const float* in0, const float* in1, double* out, int threads);

/* Interpreter of the schedule's loop nest. tiles: naxes x levels, row-major [axis][level-1]
 * (level 1 = outermost cache level); vthreads: per axis (1 on reduce axes). Axis order is the
 * reference's (gemm m,n,k; gemv m,n; conv n,f,h,w,c,r,s; pool n,c,h,w,i,j; dw n,c,h,w,r,s). */
int oracle_interpret(const oracle_op* op, int levels, const int64_t* tiles, const int64_t* vthreads,
                     const float* in0, const float* in1, double* out, int threads);

/* Number of output elements (per batch * batch). */
int64_t oracle_out_elems(const oracle_op* op);

#ifdef __cplusplus
}
#endif

#endif
