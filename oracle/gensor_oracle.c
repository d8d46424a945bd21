/* TEST INFRASTRUCTURE ONLY — see gensor_oracle.h for what this restates and why. */
#include "gensor_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define MAXA 8

/* Iteration domain + affine tensor offsets written out per kind from the Table III formulas
 * and the reference's access maps (op_spec.cpp:150-193); windowed coords are o*stride + w. */
typedef struct {
  int naxes;
  int64_t ext[MAXA];
  int reduce[MAXA];
  int nin;
  int64_t coef[3][MAXA]; /* in0, in1, out element coefficient per axis */
  int64_t size[3];       /* elements per batch of in0, in1, out */
  int64_t divisor;       /* avgpool: F*F on the true window */
} domain;

static int64_t out_extent(int64_t in, int64_t win, int64_t stride) { return (in - win) / stride + 1; }

static int make_domain(const oracle_op* op, domain* d) {
  memset(d, 0, sizeof *d);
  int64_t S = op->stride > 0 ? op->stride : 1;
  switch (op->kind) {
    case ORACLE_GEMM: { /* axes m n k: C[m][n] = sum_k A[m][k] B[k][n] */
      int64_t M = op->M, K = op->K, N = op->N;
      d->naxes = 3;
      d->ext[0] = M; d->ext[1] = N; d->ext[2] = K; d->reduce[2] = 1;
      d->nin = 2;
      d->coef[0][0] = K; d->coef[0][2] = 1;      /* A[m][k] */
      d->coef[1][2] = N; d->coef[1][1] = 1;      /* B[k][n] */
      d->coef[2][0] = N; d->coef[2][1] = 1;      /* C[m][n] */
      d->size[0] = M * K; d->size[1] = K * N; d->size[2] = M * N;
      return 0;
    }
    case ORACLE_GEMV: { /* axes m n: y[m] = sum_n A[m][n] x[n] */
      d->naxes = 2;
      d->ext[0] = op->M; d->ext[1] = op->N; d->reduce[1] = 1;
      d->nin = 2;
      d->coef[0][0] = op->N; d->coef[0][1] = 1;
      d->coef[1][1] = 1;
      d->coef[2][0] = 1;
      d->size[0] = op->M * op->N; d->size[1] = op->N; d->size[2] = op->M;
      return 0;
    }
    case ORACLE_CONV2D: { /* axes n f h w c r s: O[n][f][h][w] = sum I[n][c][hS+r][wS+s] K[f][c][r][s] */
      int64_t C = op->c, H = op->h, W = op->w, F = op->f, R = op->r, Sk = op->s;
      int64_t OH = out_extent(H, R, S), OW = out_extent(W, Sk, S);
      if (OH < 1 || OW < 1) return -1;
      d->naxes = 7;
      d->ext[0] = op->n; d->ext[1] = F; d->ext[2] = OH; d->ext[3] = OW;
      d->ext[4] = C; d->ext[5] = R; d->ext[6] = Sk;
      d->reduce[4] = d->reduce[5] = d->reduce[6] = 1;
      d->nin = 2;
      d->coef[0][0] = C * H * W; d->coef[0][4] = H * W; d->coef[0][2] = S * W; d->coef[0][5] = W;
      d->coef[0][3] = S; d->coef[0][6] = 1;
      d->coef[1][1] = C * R * Sk; d->coef[1][4] = R * Sk; d->coef[1][5] = Sk; d->coef[1][6] = 1;
      d->coef[2][0] = F * OH * OW; d->coef[2][1] = OH * OW; d->coef[2][2] = OW; d->coef[2][3] = 1;
      d->size[0] = op->n * C * H * W; d->size[1] = F * C * R * Sk; d->size[2] = op->n * F * OH * OW;
      return 0;
    }
    case ORACLE_AVGPOOL2D:
    case ORACLE_DWCONV2D: { /* axes n c h w i j (pool) / r s (dw) */
      int64_t C = op->c, H = op->h, W = op->w, R = op->r, Sk = op->s;
      int64_t OH = out_extent(H, R, S), OW = out_extent(W, Sk, S);
      if (OH < 1 || OW < 1) return -1;
      d->naxes = 6;
      d->ext[0] = op->n; d->ext[1] = C; d->ext[2] = OH; d->ext[3] = OW; d->ext[4] = R; d->ext[5] = Sk;
      d->reduce[4] = d->reduce[5] = 1;
      d->coef[0][0] = C * H * W; d->coef[0][1] = H * W; d->coef[0][2] = S * W; d->coef[0][4] = W;
      d->coef[0][3] = S; d->coef[0][5] = 1;
      d->coef[2][0] = C * OH * OW; d->coef[2][1] = OH * OW; d->coef[2][2] = OW; d->coef[2][3] = 1;
      d->size[0] = op->n * C * H * W; d->size[2] = op->n * C * OH * OW;
      if (op->kind == ORACLE_AVGPOOL2D) {
        d->nin = 1;
        d->divisor = R * Sk;
      } else {
        d->nin = 2;
        d->coef[1][1] = R * Sk; d->coef[1][4] = Sk; d->coef[1][5] = 1;
        d->size[1] = C * R * Sk;
      }
      return 0;
    }
    default:
      return -1;
  }
}

int64_t oracle_out_elems(const oracle_op* op) {
  if (op->kind == ORACLE_SOFTMAX) return op->M * op->N;
  domain d;
  if (make_domain(op, &d)) return -1;
  return d.size[2] * (op->kind == ORACLE_GEMM && op->batch > 1 ? op->batch : 1);
}

static void softmax_rows(const oracle_op* op, const float* x, double* out, int threads) {
  int64_t M = op->M, N = op->N;
  (void)threads;
#pragma omp parallel for num_threads(threads > 0 ? threads : 1) schedule(static)
  for (int64_t m = 0; m < M; ++m) {
    const float* row = x + m * N;
    double mx = -INFINITY, sum = 0.0;
    for (int64_t n = 0; n < N; ++n) mx = row[n] > mx ? row[n] : mx;
    for (int64_t n = 0; n < N; ++n) sum += exp((double)row[n] - mx);
    for (int64_t n = 0; n < N; ++n) out[m * N + n] = exp((double)row[n] - mx) / sum;
  }
}

/* ---- reference_compute: naive formula, lexicographic reduce order ---------------------- */
int oracle_reference_compute(const oracle_op* op, const float* in0, const float* in1, double* out, int threads) {
  if (op->kind == ORACLE_SOFTMAX) {
    softmax_rows(op, in0, out, threads);
    return 0;
  }
  domain d;
  if (make_domain(op, &d)) return -1;
  int64_t batch = op->kind == ORACLE_GEMM && op->batch > 1 ? op->batch : 1;
  int nsp = 0, nred = 0, sp[MAXA], rd[MAXA];
  for (int a = 0; a < d.naxes; ++a) {
    if (d.reduce[a]) rd[nred++] = a;
    else sp[nsp++] = a;
  }
  int64_t nout = 1, nr = 1;
  for (int i = 0; i < nsp; ++i) nout *= d.ext[sp[i]];
  for (int i = 0; i < nred; ++i) nr *= d.ext[rd[i]];
  (void)threads;
  for (int64_t b = 0; b < batch; ++b) {
    const float* x0 = in0 + b * d.size[0];
    const float* x1 = d.nin == 2 ? in1 + b * d.size[1] : NULL;
    double* y = out + b * d.size[2];
#pragma omp parallel for num_threads(threads > 0 ? threads : 1) schedule(static)
    for (int64_t o = 0; o < nout; ++o) {
      int64_t idx[MAXA] = {0};
      int64_t t = o;
      for (int i = nsp - 1; i >= 0; --i) {
        idx[sp[i]] = t % d.ext[sp[i]];
        t /= d.ext[sp[i]];
      }
      double acc = 0.0;
      for (int64_t q = 0; q < nr; ++q) {
        int64_t u = q;
        for (int i = nred - 1; i >= 0; --i) {
          idx[rd[i]] = u % d.ext[rd[i]];
          u /= d.ext[rd[i]];
        }
        int64_t o0 = 0, o1 = 0;
        for (int a = 0; a < d.naxes; ++a) {
          o0 += idx[a] * d.coef[0][a];
          o1 += idx[a] * d.coef[1][a];
        }
        double v = (double)x0[o0];
        if (x1) v *= (double)x1[o1];
        acc += v;
      }
      int64_t oo = 0;
      for (int a = 0; a < d.naxes; ++a) oo += idx[a] * d.coef[2][a];
      y[oo] = d.divisor ? acc / (double)d.divisor : acc;
    }
  }
  return 0;
}

/* ---- interpret(lower(state)) ------------------------------------------------------------
 * Loop nest (code level numbering: level 1 = outermost cache level):
 *   for level l = 1..L:  level-l tile loops, spatial axes then reduce axes,
 *                        radix T_{l-1}/T_l (T_0 = padded extent), step T_l
 *   vthread loops (spatial): radix V, step T_{L-1}/V
 *   scalar loops, spatial then reduce: radix T_L (spatial: T_L/V), step 1
 * At level L a spatial axis's tile loop steps T_L/V, so a thread tile is V strided slices of
 * T_L/V elements across its parent tile (the virtual-thread layout). Guards skip every
 * iteration with an index past the true extent. Per output element the reduce iterations are
 * visited level by level, which fixes the double accumulation order the parity kernel follows.
 */
typedef struct {
  int axis;
  int64_t radix;
  int64_t step;
} loop_t;

int oracle_interpret(const oracle_op* op, int L, const int64_t* tiles, const int64_t* vts, const float* in0,
                     const float* in1, double* out, int threads) {
  if (op->kind == ORACLE_SOFTMAX) {
    softmax_rows(op, in0, out, threads);
    return 0;
  }
  domain d;
  if (make_domain(op, &d) || L < 0 || L > 8) return -1;
  int64_t padded[MAXA];
  for (int a = 0; a < d.naxes; ++a) {
    padded[a] = 1;
    while (padded[a] < d.ext[a]) padded[a] <<= 1;
  }
#define TILE(a, l) ((l) == 0 ? padded[a] : tiles[(a) * L + (l) - 1])
  loop_t loops[64];
  int nl = 0;
  for (int l = 1; l <= L; ++l)
    for (int pass = 0; pass < 2; ++pass)
      for (int a = 0; a < d.naxes; ++a) {
        if (d.reduce[a] != pass) continue;
        int64_t v = (!d.reduce[a] && l == L && vts) ? vts[a] : 1;
        loops[nl].axis = a;
        loops[nl].radix = TILE(a, l - 1) / TILE(a, l);
        loops[nl].step = TILE(a, l) / v;
        ++nl;
      }
  for (int a = 0; a < d.naxes; ++a) {
    int64_t v = (!d.reduce[a] && vts && L > 0) ? vts[a] : 1;
    if (v <= 1) continue;
    loops[nl].axis = a;
    loops[nl].radix = v;
    loops[nl].step = TILE(a, L - 1) / v;
    ++nl;
  }
  for (int pass = 0; pass < 2; ++pass)
    for (int a = 0; a < d.naxes; ++a) {
      if (d.reduce[a] != pass) continue;
      int64_t v = (!d.reduce[a] && vts && L > 0) ? vts[a] : 1;
      loops[nl].axis = a;
      loops[nl].radix = TILE(a, L) / v;
      loops[nl].step = 1;
      ++nl;
    }
#undef TILE
  /* outermost parallel region: the level-1 spatial tile loops (disjoint outputs) */
  int npar = 0;
  int64_t par_total = 1;
  if (L >= 1)
    while (npar < nl && !d.reduce[loops[npar].axis] && npar < d.naxes) {
      par_total *= loops[npar].radix;
      ++npar;
    }
  int64_t batch = op->kind == ORACLE_GEMM && op->batch > 1 ? op->batch : 1;
  int64_t nout_b = d.size[2];
  for (int64_t i = 0; i < nout_b * batch; ++i) out[i] = 0.0;

  for (int64_t b = 0; b < batch; ++b) {
    const float* x0 = in0 + b * d.size[0];
    const float* x1 = d.nin == 2 ? in1 + b * d.size[1] : NULL;
    double* y = out + b * d.size[2];
    (void)threads;
#pragma omp parallel for num_threads(threads > 0 ? threads : 1) schedule(dynamic, 1)
    for (int64_t pi = 0; pi < par_total; ++pi) {
      int64_t idx[MAXA] = {0};
      int64_t dig[64] = {0};
      int64_t t = pi;
      for (int q = npar - 1; q >= 0; --q) {
        dig[q] = t % loops[q].radix;
        t /= loops[q].radix;
        idx[loops[q].axis] += dig[q] * loops[q].step;
      }
      int inner = nl - npar;
      if (inner == 0) continue;
      for (;;) {
        int ok = 1;
        for (int a = 0; a < d.naxes; ++a) ok &= idx[a] < d.ext[a];
        if (ok) {
          int64_t o0 = 0, o1 = 0, oo = 0;
          for (int a = 0; a < d.naxes; ++a) {
            o0 += idx[a] * d.coef[0][a];
            o1 += idx[a] * d.coef[1][a];
            oo += idx[a] * d.coef[2][a];
          }
          double v = (double)x0[o0];
          if (x1) v *= (double)x1[o1];
          y[oo] += v;
        }
        int q = nl - 1;
        for (; q >= npar; --q) {
          idx[loops[q].axis] += loops[q].step;
          if (++dig[q] < loops[q].radix) break;
          idx[loops[q].axis] -= loops[q].radix * loops[q].step;
          dig[q] = 0;
        }
        if (q < npar) break;
      }
    }
    if (d.divisor)
      for (int64_t i = 0; i < nout_b; ++i) y[i] = y[i] / (double)d.divisor;
  }
  return 0;
}
