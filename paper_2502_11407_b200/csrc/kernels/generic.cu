// State-driven SIMT kernel: executes ANY complete schedule of a contraction-form operator
// (gemm, gemv, conv2d, avgpool2d, dwconv2d; batched gemm via grid.y) exactly as the schedule
// tiles it. This is the execute step the reference's (absent) interpreter performs on the CPU
// (SPEC.md:479-487), moved onto the GPU:
//   * one CTA per level-1 spatial tile; one thread slot per level-L thread tile;
//   * virtual threads = strided slices of the thread tile;
//   * each level-1 reduce chunk's input boxes staged in shared memory, then the deeper reduce
//     digits walked in the interpreter's order, guarded (padding) iterations skipped.
// Acc = double gives the parity variant: products of fp32/bf16 inputs are exact in double and
// the additions happen in the interpreter's order, so outputs equal the oracle's interpret()
// bit for bit. Acc = float is the fp32 FFMA variant.
#include "../host/error.hpp"
#include "common.cuh"
#include "launch.h"
#include "plan.h"

namespace gb::dev {

namespace {

template <typename In, typename Out, typename Acc, int ACC>
__global__ void __launch_bounds__(256) k_generic(const GenericPlan p, const In* __restrict__ in0,
                                                  const In* __restrict__ in1, Out* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  In* sm = reinterpret_cast<In*>(smem_raw);
  const int64_t b = blockIdx.y;
  in0 += b * p.batch_stride[0];
  if (p.n_in == 2) in1 += b * p.batch_stride[1];
  out += b * p.batch_stride[2];

  int64_t org[8];
#pragma unroll
  for (int a = 0; a < 8; ++a) org[a] = 0;
  {
    int64_t c = blockIdx.x;
    for (int i = p.nsp - 1; i >= 0; --i) {
      org[p.sp[i]] = (c % p.tiles[i]) * p.B[i];
      c /= p.tiles[i];
    }
  }

  for (int round = 0; round < p.rounds; ++round) {
    const int slot = round * p.block + threadIdx.x;
    const bool active = slot < p.slots;
    int th[4] = {0, 0, 0, 0};
    {
      int c = active ? slot : 0;
      for (int i = p.nsp - 1; i >= 0; --i) {
        const int n = p.B[i] / p.T[i];
        th[i] = c % n;
        c /= n;
      }
    }
    for (int ch = 0; ch < p.acc_chunks; ++ch) {
      int64_t o0[ACC], o1[ACC], og[ACC];
      bool ok[ACC];
#pragma unroll
      for (int j = 0; j < ACC; ++j) {
        int e = ch * ACC + j;
        int64_t g0 = 0, g1 = 0, go = 0;
        bool inb = active;
        for (int i = p.nsp - 1; i >= 0; --i) {
          const int Ti = p.T[i];
          const int ei = e % Ti;
          e /= Ti;
          const int per = Ti / p.V[i];
          const int rel = (ei / per) * (p.B[i] / p.V[i]) + th[i] * per + (ei % per);
          const int a = p.sp[i];
          const int64_t ab = org[a] + rel;
          inb = inb && ab < p.ext[a];
          if (p.staged) {
            g0 += rel * p.scoef[0][a];
            g1 += rel * p.scoef[1][a];
          } else {
            g0 += ab * p.coef[0][a];
            g1 += ab * p.coef[1][a];
          }
          go += ab * p.coef[2][a];
        }
        o0[j] = g0;
        o1[j] = g1;
        og[j] = go;
        ok[j] = inb;
      }
      Acc acc[ACC];
#pragma unroll
      for (int j = 0; j < ACC; ++j) acc[j] = Acc(0);

      for (int c = 0; c < p.n_chunks; ++c) {
        int64_t ro[3] = {0, 0, 0};
        {
          int x = c;
          for (int q = p.nred - 1; q >= 0; --q) {
            ro[q] = static_cast<int64_t>(x % p.outer_radix[q]) * p.chunk_tile[q];
            x /= p.outer_radix[q];
          }
        }
        if (p.staged) {
          for (int q = 0; q < p.nred; ++q) org[p.red[q]] = ro[q];
          __syncthreads();  // previous chunk fully consumed
          for (int t = 0; t < p.n_in; ++t) {
            const In* src = t == 0 ? in0 : in1;
            int64_t bo[4];
            for (int d = 0; d < p.sm_nd[t]; ++d) {
              const int w = p.sm_win[t][d];
              bo[d] = w < 0 ? org[p.sm_axis[t][d]] : org[p.sm_axis[t][d]] * p.stride + org[w];
            }
            In* dst = sm + p.sm_base[t];
            for (int e = threadIdx.x; e < p.sm_elems[t]; e += blockDim.x) {
              int x = e;
              int64_t ga = 0;
              bool inb = true;
              for (int d = p.sm_nd[t] - 1; d >= 0; --d) {
                const int rel = x % p.sm_range[t][d];
                x /= p.sm_range[t][d];
                const int64_t coord = bo[d] + rel;
                inb = inb && coord < p.sm_gdim[t][d];
                ga += coord * p.sm_gstride[t][d];
              }
              dst[e] = inb ? src[ga] : In(0.0f);
            }
          }
          __syncthreads();
        }
        const In* s0 = p.staged ? sm + p.sm_base[0] : in0;
        const In* s1 = p.staged ? sm + p.sm_base[1] : in1;
        for (int i = 0; i < p.chunk_len; ++i) {
          int rr[3] = {0, 0, 0};
          {
            int x = i;
            for (int d = p.n_inner - 1; d >= 0; --d) {
              const int r = x % p.inner_radix[d];
              x /= p.inner_radix[d];
              rr[p.inner_slot[d]] += r * p.inner_mul[d];
            }
          }
          bool guard = false;
          int64_t r0 = 0, r1 = 0;
          for (int q = 0; q < p.nred; ++q) {
            const int a = p.red[q];
            const int64_t ab = ro[q] + rr[q];
            guard = guard || ab >= p.ext[a];
            if (p.staged) {
              r0 += rr[q] * p.scoef[0][a];
              r1 += rr[q] * p.scoef[1][a];
            } else {
              r0 += ab * p.coef[0][a];
              r1 += ab * p.coef[1][a];
            }
          }
          if (guard) continue;  // padded iteration: skipped, as the interpreter does
#pragma unroll
          for (int j = 0; j < ACC; ++j) {
            if (!ok[j]) continue;
            Acc v = static_cast<Acc>(to_f32(s0[o0[j] + r0]));
            if (p.n_in == 2) v *= static_cast<Acc>(to_f32(s1[o1[j] + r1]));
            acc[j] += v;
          }
        }
      }
#pragma unroll
      for (int j = 0; j < ACC; ++j) {
        if (!ok[j]) continue;
        Acc v = acc[j];
        if (p.divisor) v = v / static_cast<Acc>(p.divisor);
        out[og[j]] = from_f32<Out>(static_cast<float>(v));
      }
    }
  }
}

template <typename In, typename Out, typename Acc>
void dispatch(const GenericPlan& p, int width, const void* in0, const void* in1, void* out, int batch,
              cudaStream_t st) {
  int64_t grid = 1;
  for (int i = 0; i < p.nsp; ++i) grid *= p.tiles[i];
  dim3 g(static_cast<unsigned>(grid), static_cast<unsigned>(batch));
  auto go = [&](auto kern) {
    if (p.smem_bytes > 48 * 1024)
      check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, p.smem_bytes),
                 "generic smem attribute");
    kern<<<g, p.block, p.smem_bytes, st>>>(p, static_cast<const In*>(in0), static_cast<const In*>(in1),
                                          static_cast<Out*>(out));
    check_cuda(cudaGetLastError(), "generic launch");
    count_launch();
  };
  switch (width) {
    case 1: go(k_generic<In, Out, Acc, 1>); break;
    case 2: go(k_generic<In, Out, Acc, 2>); break;
    case 4: go(k_generic<In, Out, Acc, 4>); break;
    case 8: go(k_generic<In, Out, Acc, 8>); break;
    case 16: go(k_generic<In, Out, Acc, 16>); break;
    case 32: go(k_generic<In, Out, Acc, 32>); break;
    default: throw Error(Code::Unsupported, "generic accumulator width " + std::to_string(width));
  }
}

}  // namespace

int generic_max_width(bool f64) { return f64 ? 16 : 32; }

void launch_generic(const GenericPlan& p, bool f64, bool bf16, const void* in0, const void* in1, void* out,
                    int batch, cudaStream_t st) {
  const int width = p.acc / p.acc_chunks;
  if (bf16) {
    if (f64)
      dispatch<__nv_bfloat16, __nv_bfloat16, double>(p, width, in0, in1, out, batch, st);
    else
      dispatch<__nv_bfloat16, __nv_bfloat16, float>(p, width, in0, in1, out, batch, st);
  } else {
    if (f64)
      dispatch<float, float, double>(p, width, in0, in1, out, batch, st);
    else
      dispatch<float, float, float>(p, width, in0, in1, out, batch, st);
  }
}

}  // namespace gb::dev
