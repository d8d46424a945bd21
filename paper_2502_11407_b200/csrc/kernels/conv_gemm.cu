// General tensor-core implicit-GEMM conv2d (any stride, window, channel and filter count),
// instantiated from a constructed conv2d schedule:
//   O[n][f][oh][ow] = sum_{c,r,s} I[n][c][oh*S+r][ow*S+s] * K[f][c][r][s]   (op_spec.cpp:177-181)
// GEMM view: M = output positions (n, oh, ow) flattened, N = f, K = (r, s, c).
// Reads the NCHW input IN PLACE — no NHWC copy (for a network the copy would cost two extra
// activation round trips per layer):
//   * A (positions x channels) is staged MN-major: for a fixed channel the 32 positions of a warp
//     are (mostly) consecutive addresses of one NCHW plane, so producer warps issue coalesced
//     32-bit loads and conflict-free 32-bit shared stores into the tf32 MN-major 128 B swizzle
//     (32 B granules XOR k%4, 4-row K groups 512 B apart, 32-position chunks 4 KB apart);
//   * B is W'[r][s][f][c] (K-major rows, converted by a small pre-pass launch that the conv grid
//     overlaps through programmatic dependent launch), TMA-loaded per k-block;
//   * persistent CTAs, BN-wide filter tiles, tcgen05.mma kind::tf32 into two TMEM accumulators,
//     4 epilogue warps storing NCHW rows (32 consecutive positions per f: 128 B).
#include <cuda_bf16.h>

#include "../host/error.hpp"
#include "common.cuh"
#include "launch.h"
#include "tc_common.cuh"

namespace gb::dev {

namespace {

using namespace tc;

constexpr int kGGroups = 4;                    // producer groups: group g fills k-blocks kb = g (mod 4)
constexpr int kGProducerWarps = 4 * kGGroups;  // 4 warps (one 32-position MN chunk each) per group
constexpr int kGThreads = 32 * (kGProducerWarps + 1 + 4);

__device__ __forceinline__ void sts32(uint32_t addr, float v) {
  asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}

template <int BN, int STAGES>
__global__ void __launch_bounds__(kGThreads, 1)
    k_conv_gemm(const float* __restrict__ I, const __grid_constant__ CUtensorMap mapW, float* __restrict__ O, int N,
                int C, int H, int W, int F, int R, int S, int stride, int OH, int OW, int tiles_m, int tiles_n,
                int total, int packed) {
  constexpr int BM = 128, BK = 32;                 // tf32: 32 channels = 128 B per K row
  constexpr uint32_t A_BYTES = BM * BK * 4;        // 4 MN chunks x 4 KB
  constexpr uint32_t B_BYTES = BN * 128;
  constexpr uint32_t STAGE = A_BYTES + B_BYTES;
  constexpr uint32_t TMEM_COLS = 2 * BN;
  constexpr uint32_t IDESC = instr_desc(2, BM, BN, /*a_mn_major=*/1, /*b_mn_major=*/0);
  constexpr int kMma = kGProducerWarps;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* staging = smem + STAGES * STAGE;  // 4 epilogue warps x 32 x 32 fp32
  uint64_t* full = reinterpret_cast<uint64_t*>(staging + 4 * 32 * 32 * 4);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;  // [2]
  uint64_t* acc_empty = acc_full + 2;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // k-blocks: general mode (r, s, 32-channel chunk); packed mode (few channels, C*S <= 64): per
  // filter row r the (s, c) pairs form one K axis k = s*C + c, cut into 32-wide blocks
  const int nck = packed ? (S * C + BK - 1) / BK : (C + BK - 1) / BK;
  const int nk = packed ? R * nck : R * S * nck;
  const int64_t P = static_cast<int64_t>(N) * OH * OW;
  const int64_t plane = static_cast<int64_t>(H) * W;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 128 + 1);  // one producer group + the B tensor-map arrival
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 4);
    }
    fence_barrier_init();
  }
  if (warp == kMma) tmem_alloc<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < kGProducerWarps) {
    // producer warp (group g, index pw): MN chunk pw (positions 32*pw .. 32*pw+31 of the tile),
    // all 32 channels of the k-block; lane = position. Group 0 additionally issues the B TMA.
    const int grp = warp >> 2, pw = warp & 3;
    // the B-issuing lanes read W', which the preceding pre-pass launch writes (programmatic
    // dependent launch: this grid may start before it completes)
    if (pw == 0 && lane == 0) asm volatile("griddepcontrol.wait;" ::: "memory");
    int it = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      const int mt = t / tiles_n, nt = t % tiles_n;
      const int64_t p = static_cast<int64_t>(mt) * BM + pw * 32 + lane;
      const bool pv = p < P;
      const int64_t pp = pv ? p : 0;
      const int n = static_cast<int>(pp / (static_cast<int64_t>(OH) * OW));
      const int rem = static_cast<int>(pp - static_cast<int64_t>(n) * OH * OW);
      const int oh = rem / OW, ow = rem - oh * OW;
      const float* base = I + static_cast<int64_t>(n) * C * plane + static_cast<int64_t>(oh) * stride * W +
                          static_cast<int64_t>(ow) * stride;
      // k-block kb -> (r, s, channel chunk) [general] or (r, (s,c) chunk) [packed]
      auto load_kb = [&](int kb, float (&v)[BK]) {
        if (!packed) {
          const int ck = kb % nck, rs = kb / nck, r = rs / S, s = rs - r * S;
          const float* src = base + static_cast<int64_t>(r) * W + s + static_cast<int64_t>(ck) * BK * plane;
#pragma unroll
          for (int k = 0; k < BK; ++k)
            v[k] = (pv && ck * BK + k < C) ? __ldg(src + static_cast<int64_t>(k) * plane) : 0.0f;
        } else {
          const int ck = kb % nck, r = kb / nck;
          const float* src = base + static_cast<int64_t>(r) * W;
#pragma unroll
          for (int k = 0; k < BK; ++k) {
            const int kk = ck * BK + k;  // uniform across the warp
            const int sk = kk / C, c = kk - sk * C;
            v[k] = (pv && sk < S) ? __ldg(src + static_cast<int64_t>(c) * plane + sk) : 0.0f;
          }
        }
      };
      // this group's k-blocks of the tile: global k-block counter it + kb = grp (mod kGGroups)
      const int kb0 = ((grp - it) % kGGroups + kGGroups) % kGGroups;
      for (int kb = kb0; kb < nk; kb += kGGroups) {
        const int k_it = it + kb;
        const int st = k_it % STAGES;
        mbar_wait(&empty[st], ((k_it / STAGES) & 1) ^ 1);
        uint8_t* a_s = smem + st * STAGE;
        if (pw == 0 && lane == 0) {  // B: BN filters x 32 K of W' (an extra arrival)
          const int ck = kb % nck;
          mbar_arrive_expect_tx(&full[st], B_BYTES);
          tma_load_3d(a_s + A_BYTES, &mapW, &full[st], ck * BK, nt * BN, kb / nck);
        }
        float v[BK];
        load_kb(kb, v);
        // MN-major tf32 layout: chunk pw (4 KB) | K row k: (k/4)*512 + (k%4)*128 | granule
        // (lane/8) ^ (k%4), word lane%8
        const uint32_t chunk = smem_u32(a_s) + pw * 4096 + (lane & 7) * 4;
#pragma unroll
        for (int k = 0; k < BK; ++k)
          sts32(chunk + (k >> 2) * 512 + (k & 3) * 128 + ((((lane >> 3) ^ (k & 3)) & 3) << 5), v[k]);
        fence_proxy_async_smem();
        mbar_arrive(&full[st]);
      }
      it += nk;
    }
  } else if (warp == kMma) {
    if (elect_one()) {
      asm volatile("griddepcontrol.wait;" ::: "memory");  // W' comes from the pre-pass launch
      tma_prefetch(&mapW);
      int it = 0, local = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++local) {
        const int acc = local & 1;
        mbar_wait(&acc_empty[acc], ((local >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * BN;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int st = it % STAGES;
          mbar_wait(&full[st], (it / STAGES) & 1);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smem + st * STAGE);
          const uint32_t b_addr = a_addr + A_BYTES;
#pragma unroll
          for (int k = 0; k < 4; ++k) {  // 4 MMAs x K=8
            const uint64_t ad = smem_desc_sw128(a_addr + k * 1024, 4096, 512, 1);
            const uint64_t bd = smem_desc_sw128(b_addr + k * 32, 16, 1024);
            mma_tf32(d, ad, bd, IDESC, (kb | k) != 0);
          }
          mma_commit(&empty[st]);
        }
        mma_commit(&acc_full[acc]);
      }
    }
  } else {
    // Epilogue: TMEM lanes (positions) x 32 filters -> the warp's staging rows [f][32 positions]
    // (conflict-free 4 B stores) -> each lane re-reads 16 B = 4 consecutive positions of one
    // filter and stores them with one 16 B streaming store: a warp instruction writes 4 filter
    // rows x 128 B instead of 1 x 128 B. Positions must not straddle an image within a group
    // of 4 (OH*OW % 4 == 0); otherwise per-element stores.
    const int q = warp & 3;  // TMEM lane quarter = tile rows (positions) 32q .. 32q+31
    const int64_t ohw = static_cast<int64_t>(OH) * OW;
    float* stg = reinterpret_cast<float*>(staging) + q * (32 * 32);
    const uint32_t stg_s = smem_u32(stg);
    const bool vec = (ohw & 3) == 0;
    int local = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++local) {
      const int acc = local & 1;
      const int mt = t / tiles_n, nt = t % tiles_n;
      const int64_t pw0 = static_cast<int64_t>(mt) * BM + q * 32;  // first position of this warp
      const int64_t p = pw0 + lane;
      mbar_wait(&acc_full[acc], (local >> 1) & 1);
      tc_fence_after();
      // vector-store geometry: lane -> (filter row lane/8 of 4, positions 4*(lane%8) .. +3)
      const int64_t pv4 = pw0 + 4 * (lane & 7);
      const int n4 = static_cast<int>(pv4 / ohw);
      const int64_t pr4 = pv4 - n4 * ohw;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t r[32];
        tmem_ld32(tmem + acc * BN + (static_cast<uint32_t>(q * 32) << 16) + c, r);
        tmem_ld_wait();
        tmem_ld_pin(r);
        const int f0 = nt * BN + c;
        if (vec) {
          __syncwarp();  // previous chunk's re-reads are done
#pragma unroll
          for (int v = 0; v < 32; ++v) sts32(stg_s + (v * 32 + lane) * 4, __uint_as_float(r[v]));
          __syncwarp();
#pragma unroll
          for (int g = 0; g < 8; ++g) {
            const int fl = g * 4 + (lane >> 3);
            const float4 val = *reinterpret_cast<const float4*>(stg + fl * 32 + 4 * (lane & 7));
            if (pv4 < P && f0 + fl < F)
              __stcs(reinterpret_cast<float4*>(O + (static_cast<int64_t>(n4) * F + f0 + fl) * ohw + pr4), val);
          }
        } else if (p < P) {
          const int n = static_cast<int>(p / ohw);
          float* obase = O + (static_cast<int64_t>(n) * F) * ohw + (p - n * ohw);
#pragma unroll
          for (int v = 0; v < 32; ++v)
            if (f0 + v < F) __stcs(obase + static_cast<int64_t>(f0 + v) * ohw, __uint_as_float(r[v]));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMma) {
    tc_fence_after();
    tmem_dealloc<TMEM_COLS>(tmem);
  }
}

// K[f][c][r][s] -> W'[r][s][f][c] (K-major B rows for the TMA); primary grid of the PDL pair.
// Rows are padded to Cp = C rounded up to 4 channels (16 B, the TMA stride unit), pad = 0.
// Packed mode (Cp = S*C rounded up to 4): W'[r][f][s*C + c].
__global__ void __launch_bounds__(256) k_filters_rsfc(const float* __restrict__ K, float* __restrict__ Wt, int F,
                                                      int C, int Cp, int RS, int S, int packed) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (packed) {
    const int R = RS / S;
    const int64_t tot = static_cast<int64_t>(R) * F * Cp;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < tot;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
      const int kk = static_cast<int>(e % Cp);  // e = (r*F + f)*Cp + kk
      const int64_t rf = e / Cp;
      const int f = static_cast<int>(rf % F), r = static_cast<int>(rf / F);
      const int sk = kk / C, c = kk - sk * C;
      Wt[e] = sk < S ? __ldg(K + ((static_cast<int64_t>(f) * C + c) * R + r) * S + sk) : 0.0f;
    }
    return;
  }
  const int64_t total = static_cast<int64_t>(F) * Cp * RS;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int rs = static_cast<int>(e % RS);  // e = (f*Cp + c)*RS + rs
    const int64_t fc = e / RS;
    const int c = static_cast<int>(fc % Cp), f = static_cast<int>(fc / Cp);
    Wt[(static_cast<int64_t>(rs) * F + f) * Cp + c] = c < C ? __ldg(K + (static_cast<int64_t>(f) * C + c) * RS + rs) : 0.0f;
  }
}

template <int BN>
constexpr int conv_gemm_stages() {
  constexpr size_t STAGE = 128 * 128 + BN * 128;
  return static_cast<int>((227 * 1024 - 2048 - 16384) / STAGE) >= 4 ? 4 : 3;
}

template <int BN>
void run_gemm_conv(const ConvGemmArgs& a, const CUtensorMap& mapW, const float* I, const float* K, float* O, void* ws,
                   cudaStream_t st, Marks& mk) {
  constexpr size_t STAGE = 128 * 128 + BN * 128;
  constexpr int STAGES = conv_gemm_stages<BN>();
  const int Cp = a.packed ? (a.S * a.C + 3) / 4 * 4 : (a.C + 3) / 4 * 4;
  const int planes = a.packed ? a.R : a.R * a.S;
  const int64_t P = static_cast<int64_t>(a.N) * a.OH * a.OW;
  const int tiles_m = static_cast<int>((P + 127) / 128), tiles_n = (a.F + BN - 1) / BN;
  const int total = tiles_m * tiles_n;
  const int grid = std::min(total, a.sms);
  mk.mark(st);
  const int64_t wt = static_cast<int64_t>(a.F) * Cp * planes;
  k_filters_rsfc<<<static_cast<unsigned>(std::min<int64_t>(4 * a.sms, (wt + 255) / 256)), 256, 0, st>>>(
      K, static_cast<float*>(ws), a.F, a.C, Cp, a.R * a.S, a.S, a.packed);
  check_cuda(cudaGetLastError(), "filters_rsfc launch");
  count_launch();
  auto kern = k_conv_gemm<BN, STAGES>;
  const size_t smem = STAGES * STAGE + 16384 + 1024 + 256;
  set_smem_attr(kern, static_cast<int>(smem), "conv_gemm smem attribute");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kGThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  check_cuda(cudaLaunchKernelEx(&cfg, kern, I, mapW, O, a.N, a.C, a.H, a.W, a.F, a.R, a.S, a.stride, a.OH, a.OW,
                                tiles_m, tiles_n, total, a.packed),
             "conv_gemm launch");
  count_launch();
  mk.mark(st);
}

}  // namespace

void conv_gemm_map(const ConvGemmArgs& a, void* ws, CUtensorMap& mapW) {
  const int Cp = a.packed ? (a.S * a.C + 3) / 4 * 4 : (a.C + 3) / 4 * 4;
  const int planes = a.packed ? a.R : a.R * a.S;
  const uint64_t dw[3] = {static_cast<uint64_t>(Cp), static_cast<uint64_t>(a.F), static_cast<uint64_t>(planes)};
  const uint64_t sw[2] = {static_cast<uint64_t>(Cp) * 4, static_cast<uint64_t>(Cp) * a.F * 4};
  const uint32_t bw[3] = {32, static_cast<uint32_t>(a.BN), 1};
  encode_map(&mapW, false, true, ws, 3, dw, sw, bw);
}

void launch_conv_gemm(const ConvGemmArgs& a, const CUtensorMap& mapW, const void* I, const void* K, void* O, void* ws,
                      cudaStream_t st, Marks& mk) {
  const float* i = static_cast<const float*>(I);
  const float* k = static_cast<const float*>(K);
  float* o = static_cast<float*>(O);
  switch (a.BN) {
    case 64: run_gemm_conv<64>(a, mapW, i, k, o, ws, st, mk); break;
    case 128: run_gemm_conv<128>(a, mapW, i, k, o, ws, st, mk); break;
    default: run_gemm_conv<256>(a, mapW, i, k, o, ws, st, mk); break;
  }
}

}  // namespace gb::dev
