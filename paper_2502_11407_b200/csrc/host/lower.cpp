#include "lower.hpp"

#include <algorithm>
#include <cstring>
#include <sstream>

#include "error.hpp"

namespace gb {

namespace {
inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
}  // namespace

// Mapping:
//   grid.x   = prod over spatial axes of ceil(extent / T1)     (guarded tail tiles kept, fully
//              out-of-range tiles never launched); grid.y = batch
//   slots    = prod over spatial axes of T1 / T_L              (thread tiles per CTA)
//   acc      = prod over spatial axes of T_L                   (outputs per thread tile)
//   vthreads = T_L split into V strided slices, slice stride T1 / V (TVM virtual threads)
//   reduce   = level-1 chunks (padded / T1 per axis, lexicographic) staged in shared memory,
//              then the level-2..L digits, then the scalar digits — the interpreter's
//              reduce order, so fp64 accumulation reproduces interpret() bit for bit.
GenericPlan lower_generic(const OpDesc& op, const Sched& s, int acc_width, int elem_bytes, int64_t smem_limit) {
  if (!s.complete()) throw Error(Code::IncompleteState, "lowering needs a complete schedule");
  GenericPlan p;
  std::memset(&p, 0, sizeof p);
  if (op.kind == Kind::Softmax) throw Error(Code::Unsupported, "softmax has no contraction form; use the stream variant");
  const int L = s.L;
  p.nsp = 0;
  p.nred = 0;
  for (int a = 0; a < op.naxes; ++a) {
    p.ext[a] = op.ax[a].extent;
    if (op.ax[a].reduce) {
      if (p.nred == 3) throw Error(Code::Unsupported, "more than 3 reduce axes");
      p.red[p.nred++] = a;
    } else {
      if (p.nsp == 4) throw Error(Code::Unsupported, "more than 4 spatial axes");
      p.sp[p.nsp++] = a;
    }
  }

  // spatial tiling
  int64_t grid = 1, slots = 1, acc = 1;
  for (int i = 0; i < p.nsp; ++i) {
    const int a = p.sp[i];
    const int64_t b = L ? s.tile(op, a, 1) : 1;
    const int64_t t = L ? s.tile(op, a, L) : 1;
    const int64_t v = L ? s.vt(a) : 1;
    p.B[i] = static_cast<int32_t>(b);
    p.T[i] = static_cast<int32_t>(t);
    p.V[i] = static_cast<int32_t>(v);
    p.tiles[i] = static_cast<int32_t>(cdiv(op.ax[a].extent, b));
    grid *= p.tiles[i];
    slots *= b / t;
    acc *= t;
  }
  if (grid > (1LL << 31) - 1) throw Error(Code::Unsupported, "grid too large");
  p.slots = static_cast<int32_t>(slots);
  p.acc = static_cast<int32_t>(acc);
  const int width = static_cast<int>(std::min<int64_t>(acc, acc_width));
  p.acc_chunks = static_cast<int32_t>(acc / width);
  p.block = static_cast<int32_t>(std::min<int64_t>(256, std::max<int64_t>(32, cdiv(slots, 32) * 32)));
  p.rounds = static_cast<int32_t>(cdiv(slots, p.block));

  // reduce walk
  p.n_chunks = 1;
  p.chunk_len = 1;
  p.n_inner = 0;
  for (int q = 0; q < p.nred; ++q) {
    const int a = p.red[q];
    const int64_t t1 = L ? s.tile(op, a, 1) : op.ax[a].padded;
    p.chunk_tile[q] = static_cast<int32_t>(t1);
    p.outer_radix[q] = static_cast<int32_t>(op.ax[a].padded / t1);
    p.n_chunks *= p.outer_radix[q];
    p.chunk_len *= static_cast<int32_t>(t1);
  }
  auto digit = [&](int q, int64_t radix, int64_t mul) {
    if (radix <= 1) return;
    if (p.n_inner == 12) throw Error(Code::Unsupported, "reduce loop nest too deep");
    p.inner_slot[p.n_inner] = q;
    p.inner_radix[p.n_inner] = static_cast<int32_t>(radix);
    p.inner_mul[p.n_inner] = static_cast<int32_t>(mul);
    ++p.n_inner;
  };
  for (int l = 2; l <= L; ++l)
    for (int q = 0; q < p.nred; ++q) {
      const int a = p.red[q];
      digit(q, s.tile(op, a, l - 1) / s.tile(op, a, l), s.tile(op, a, l));
    }
  for (int q = 0; q < p.nred; ++q) {
    const int a = p.red[q];
    digit(q, L ? s.tile(op, a, L) : op.ax[a].padded, 1);
  }

  // tensors
  p.n_in = op.input_count();
  for (int t = 0; t < op.ntensors; ++t) {
    const int slot = op.t[t].output ? 2 : t;
    int64_t c[kMaxAxes];
    op.affine_coefs(t, c);
    for (int a = 0; a < 8; ++a) p.coef[slot][a] = a < op.naxes ? c[a] : 0;
    p.batch_stride[slot] = op.tensor_elems(t, false);
  }
  p.stride = op.stride;
  p.divisor = op.kind == Kind::AvgPool2d ? static_cast<int32_t>(op.param("F") * op.param("F")) : 0;

  // shared-memory boxes: per input dim, the coordinate range one (CTA tile, reduce chunk) covers
  auto range_of = [&](int a) -> int64_t {
    for (int i = 0; i < p.nsp; ++i)
      if (p.sp[i] == a) return p.B[i];
    for (int q = 0; q < p.nred; ++q)
      if (p.red[q] == a) return p.chunk_tile[q];
    return 1;
  };
  int64_t total = 0;
  for (int t = 0; t < p.n_in; ++t) {
    const TensorDesc& td = op.t[t];
    int64_t dims[kMaxDims];
    op.tensor_dims(t, false, dims);
    p.sm_nd[t] = td.ndims;
    int64_t gstr = 1;
    for (int d = td.ndims - 1; d >= 0; --d) {
      p.sm_gstride[t][d] = gstr;
      gstr *= dims[d];
    }
    int64_t elems = 1;
    for (int d = 0; d < td.ndims; ++d) {
      const DimMap& m = td.dim[d];
      p.sm_axis[t][d] = m.axis;
      p.sm_win[t][d] = m.win;
      p.sm_gdim[t][d] = dims[d];
      const int64_t r = m.win < 0 ? range_of(m.axis) : (range_of(m.axis) - 1) * op.stride + range_of(m.win);
      p.sm_range[t][d] = static_cast<int32_t>(std::min<int64_t>(r, 1LL << 30));
      elems *= r;
    }
    int64_t sstr = 1;
    for (int a = 0; a < 8; ++a) p.scoef[t][a] = 0;
    for (int d = td.ndims - 1; d >= 0; --d) {
      const DimMap& m = td.dim[d];
      if (m.win < 0) {
        p.scoef[t][m.axis] += sstr;
      } else {
        p.scoef[t][m.axis] += sstr * op.stride;
        p.scoef[t][m.win] += sstr;
      }
      sstr *= p.sm_range[t][d];
    }
    p.sm_base[t] = static_cast<int32_t>(std::min<int64_t>(total, 1LL << 30));
    p.sm_elems[t] = static_cast<int32_t>(std::min<int64_t>(elems, 1LL << 30));
    total += elems;
  }
  p.staged = total * elem_bytes <= smem_limit ? 1 : 0;
  p.smem_bytes = p.staged ? static_cast<int32_t>(total * elem_bytes) : 0;
  return p;
}

std::string plan_json(const GenericPlan& p) {
  std::ostringstream os;
  int64_t grid = 1;
  for (int i = 0; i < p.nsp; ++i) grid *= p.tiles[i];
  os << "{\"family\":\"generic\",\"grid\":" << grid << ",\"block\":" << p.block << ",\"slots\":" << p.slots
     << ",\"acc\":" << p.acc << ",\"acc_chunks\":" << p.acc_chunks << ",\"rounds\":" << p.rounds
     << ",\"n_chunks\":" << p.n_chunks << ",\"chunk_len\":" << p.chunk_len << ",\"staged\":" << p.staged
     << ",\"smem_bytes\":" << p.smem_bytes
     << ",\"fast\":\"" << (p.fast == 1 ? "gemm" : p.fast == 2 ? "gemv" : p.fast == 3 ? "gemv_tma" : "none") << "\",\"block_tile\":[";
  for (int i = 0; i < p.nsp; ++i) os << (i ? "," : "") << p.B[i];
  os << "],\"thread_tile\":[";
  for (int i = 0; i < p.nsp; ++i) os << (i ? "," : "") << p.T[i];
  os << "],\"vthreads\":[";
  for (int i = 0; i < p.nsp; ++i) os << (i ? "," : "") << p.V[i];
  os << "]}";
  return os.str();
}

}  // namespace gb
