#include "op.hpp"

#include <algorithm>
#include <cstring>
#include <sstream>

#include "error.hpp"

namespace gb {

const char* kind_name(Kind k) {
  switch (k) {
    case Kind::Gemm: return "gemm";
    case Kind::Gemv: return "gemv";
    case Kind::Conv2d: return "conv2d";
    case Kind::AvgPool2d: return "avgpool2d";
    case Kind::DwConv2d: return "dwconv2d";
    case Kind::Softmax: return "softmax";
  }
  return "?";
}

bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }

int64_t next_pow2(int64_t v) {
  int64_t p = 1;
  while (p < v) p <<= 1;
  return p;
}

namespace {

// Parameter codes: one char per reference parameter name; OH/OW use 'h'/'w'.
char code_of(const char* name) {
  if (std::strcmp(name, "OH") == 0) return 'h';
  if (std::strcmp(name, "OW") == 0) return 'w';
  return name[0];
}

int64_t need_int(const json::Value& doc, const char* key) {
  const json::Value* v = doc.find(key);
  if (!v) throw Error(Code::MissingParam, std::string("missing parameter '") + key + "'");
  if (!v->is_int()) throw Error(Code::MissingParam, std::string("parameter '") + key + "' must be an integer");
  return v->i;
}

int64_t need_extent(const json::Value& doc, const char* key) {
  int64_t v = need_int(doc, key);
  if (v < 1) throw Error(Code::NonPositiveExtent, std::string("'") + key + "' = " + std::to_string(v));
  return v;
}

std::array<int64_t, 4> need_quad(const json::Value& doc, const char* key) {
  const json::Value* v = doc.find(key);
  if (!v || !v->is_array() || v->arr.size() != 4)
    throw Error(Code::MissingParam, std::string("'") + key + "' must be a 4-element array");
  std::array<int64_t, 4> out{};
  for (size_t i = 0; i < 4; ++i) {
    int64_t x = v->arr[i].as_int();
    if (x < 1) throw Error(Code::NonPositiveExtent, std::string("'") + key + "' entry " + std::to_string(x));
    out[i] = x;
  }
  return out;
}

// (in - window) / stride + 1 (op_spec.cpp:55-60).
int64_t out_extent(int64_t in, int64_t window, int64_t stride, const char* what) {
  int64_t o = (in - window) / stride + 1;
  if (in < window || o < 1) throw Error(Code::NonPositiveExtent, std::string(what) + " output extent would be < 1");
  return o;
}

// |{o*stride + w : o < to, w < tw}|: windows overlap only when stride < tw (op_spec.cpp:64-66).
inline int64_t span(int64_t to, int64_t tw, int64_t stride) { return tw + (to - 1) * std::min(stride, tw); }

}  // namespace

void OpDesc::set(char code, int64_t v) {
  for (int i = 0; i < nparams_; ++i)
    if (params_[static_cast<size_t>(i)].first == code) {
      params_[static_cast<size_t>(i)].second = v;
      return;
    }
  params_[static_cast<size_t>(nparams_++)] = {code, v};
}

int64_t OpDesc::get(char code) const {
  for (int i = 0; i < nparams_; ++i)
    if (params_[static_cast<size_t>(i)].first == code) return params_[static_cast<size_t>(i)].second;
  throw Error(Code::MissingParam, std::string("no parameter '") + code + "'");
}

int64_t OpDesc::param(const char* name) const { return get(code_of(name)); }

OpDesc OpDesc::parse_text(const std::string& text) { return parse(json::parse(text)); }

OpDesc OpDesc::parse(const json::Value& doc) {
  const json::Value* kv = doc.find("kind");
  if (!kv) throw Error(Code::MissingParam, "missing parameter 'kind'");
  const std::string& kind = kv->as_string();

  OpDesc op;
  if (doc.has("dtype_bytes")) op.dtype_bytes = static_cast<int>(need_extent(doc, "dtype_bytes"));

  // Conv/pool accept either I/K arrays with "S" as the stride, or flat keys with "stride"
  // (op_spec.cpp:90-122) — note "S" means the stride in the array form and the kernel width
  // in the flat form, exactly as the reference reads it.
  auto windowed = [&](bool has_kernel_tensor, bool depthwise) {
    if (doc.has("I")) {
      auto in = need_quad(doc, "I");
      op.set('N', in[0]);
      op.set('C', in[1]);
      op.set('H', in[2]);
      op.set('W', in[3]);
      if (has_kernel_tensor) {
        auto kn = need_quad(doc, "K");
        if (depthwise) {
          if (kn[0] != in[1] || kn[1] != 1)
            throw Error(Code::ConfigError, "dwconv2d kernel must be [C,1,R,S] with C = input channels");
        } else {
          op.set('F', kn[0]);
          if (kn[1] != in[1]) throw Error(Code::ConfigError, "conv2d kernel channels do not match input channels");
        }
        op.set('R', kn[2]);
        op.set('S', kn[3]);
      } else {
        op.set('F', need_extent(doc, "F"));
      }
      op.stride = doc.has("S") ? need_extent(doc, "S") : 1;
    } else {
      const char* conv_keys[] = {"N", "C", "H", "W", "F", "R", "S"};
      const char* dw_keys[] = {"N", "C", "H", "W", "R", "S"};
      const char* pool_keys[] = {"N", "C", "H", "W", "F"};
      if (!has_kernel_tensor)
        for (const char* k : pool_keys) op.set(code_of(k), need_extent(doc, k));
      else if (depthwise)
        for (const char* k : dw_keys) op.set(code_of(k), need_extent(doc, k));
      else
        for (const char* k : conv_keys) op.set(code_of(k), need_extent(doc, k));
      op.stride = doc.has("stride") ? need_extent(doc, "stride") : 1;
    }
  };

  if (kind == "gemm") {
    op.kind = Kind::Gemm;
    op.set('M', need_extent(doc, "M"));
    op.set('K', need_extent(doc, "K"));
    op.set('N', need_extent(doc, "N"));
    if (doc.has("batch")) op.batch = need_extent(doc, "batch");
  } else if (kind == "gemv") {
    op.kind = Kind::Gemv;
    op.set('M', need_extent(doc, "M"));
    op.set('N', need_extent(doc, "N"));
  } else if (kind == "conv2d") {
    op.kind = Kind::Conv2d;
    windowed(true, false);
    op.set('h', out_extent(op.get('H'), op.get('R'), op.stride, "conv2d"));
    op.set('w', out_extent(op.get('W'), op.get('S'), op.stride, "conv2d"));
  } else if (kind == "avgpool2d") {
    op.kind = Kind::AvgPool2d;
    windowed(false, false);
    op.set('h', out_extent(op.get('H'), op.get('F'), op.stride, "avgpool2d"));
    op.set('w', out_extent(op.get('W'), op.get('F'), op.stride, "avgpool2d"));
  } else if (kind == "dwconv2d") {
    op.kind = Kind::DwConv2d;
    windowed(true, true);
    op.set('h', out_extent(op.get('H'), op.get('R'), op.stride, "dwconv2d"));
    op.set('w', out_extent(op.get('W'), op.get('S'), op.stride, "dwconv2d"));
  } else if (kind == "softmax") {
    op.kind = Kind::Softmax;
    op.set('M', need_extent(doc, "M"));
    op.set('N', need_extent(doc, "N"));
  } else {
    throw Error(Code::UnknownKind, "unsupported op kind '" + kind + "'");
  }
  op.build();
  return op;
}

void OpDesc::build() {
  naxes = 0;
  auto axis = [&](const char* name, int64_t extent, bool reduce) {
    AxisDesc& a = ax[naxes++];
    std::strncpy(a.name, name, 3);
    a.extent = extent;
    a.padded = next_pow2(extent);
    a.reduce = reduce;
  };
  auto tensor = [&](int idx, const char* name, bool output, std::initializer_list<DimMap> dims) {
    TensorDesc& td = t[idx];
    std::strncpy(td.name, name, 3);
    td.output = output;
    td.ndims = 0;
    for (const DimMap& d : dims) td.dim[td.ndims++] = d;
  };
  switch (kind) {
    case Kind::Gemm:
      axis("m", get('M'), false);
      axis("n", get('N'), false);
      axis("k", get('K'), true);
      ntensors = 3;
      tensor(0, "A", false, {{0, -1}, {2, -1}});
      tensor(1, "B", false, {{2, -1}, {1, -1}});
      tensor(2, "C", true, {{0, -1}, {1, -1}});
      break;
    case Kind::Gemv:
      axis("m", get('M'), false);
      axis("n", get('N'), true);
      ntensors = 3;
      tensor(0, "A", false, {{0, -1}, {1, -1}});
      tensor(1, "x", false, {{1, -1}});
      tensor(2, "y", true, {{0, -1}});
      break;
    case Kind::Conv2d:
      axis("n", get('N'), false);
      axis("f", get('F'), false);
      axis("h", get('h'), false);
      axis("w", get('w'), false);
      axis("c", get('C'), true);
      axis("r", get('R'), true);
      axis("s", get('S'), true);
      ntensors = 3;
      tensor(0, "I", false, {{0, -1}, {4, -1}, {2, 5}, {3, 6}});
      tensor(1, "K", false, {{1, -1}, {4, -1}, {5, -1}, {6, -1}});
      tensor(2, "O", true, {{0, -1}, {1, -1}, {2, -1}, {3, -1}});
      break;
    case Kind::AvgPool2d:
      axis("n", get('N'), false);
      axis("c", get('C'), false);
      axis("h", get('h'), false);
      axis("w", get('w'), false);
      axis("i", get('F'), true);
      axis("j", get('F'), true);
      ntensors = 2;
      tensor(0, "I", false, {{0, -1}, {1, -1}, {2, 4}, {3, 5}});
      tensor(1, "O", true, {{0, -1}, {1, -1}, {2, -1}, {3, -1}});
      break;
    case Kind::DwConv2d:
      axis("n", get('N'), false);
      axis("c", get('C'), false);
      axis("h", get('h'), false);
      axis("w", get('w'), false);
      axis("r", get('R'), true);
      axis("s", get('S'), true);
      ntensors = 3;
      tensor(0, "I", false, {{0, -1}, {1, -1}, {2, 4}, {3, 5}});
      tensor(1, "K", false, {{1, -1}, {4, -1}, {5, -1}});
      tensor(2, "O", true, {{0, -1}, {1, -1}, {2, -1}, {3, -1}});
      break;
    case Kind::Softmax:
      axis("m", get('M'), false);
      axis("n", get('N'), true);
      ntensors = 2;
      tensor(0, "X", false, {{0, -1}, {1, -1}});
      tensor(1, "O", true, {{0, -1}, {1, -1}});
      break;
  }
}

int OpDesc::axis_index(const std::string& name) const {
  for (int i = 0; i < naxes; ++i)
    if (name == ax[i].name) return i;
  throw Error(Code::AxisNotFound, "no axis '" + name + "' in " + label());
}

void OpDesc::tile_elems(const int64_t* tile, int64_t* out) const {
  for (int ti = 0; ti < ntensors; ++ti) {
    const TensorDesc& td = t[ti];
    int64_t n = 1;
    for (int d = 0; d < td.ndims; ++d) {
      const DimMap& m = td.dim[d];
      n *= m.win < 0 ? tile[m.axis] : span(tile[m.axis], tile[m.win], stride);
    }
    out[ti] = n;
  }
}

int OpDesc::tensor_dims(int ti, bool padded, int64_t* dims) const {
  const TensorDesc& td = t[ti];
  for (int d = 0; d < td.ndims; ++d) {
    const DimMap& m = td.dim[d];
    const AxisDesc& a = ax[m.axis];
    if (m.win < 0)
      dims[d] = padded ? a.padded : a.extent;
    else if (padded)
      dims[d] = span(a.padded, ax[m.win].padded, stride);
    else
      dims[d] = a.name[0] == 'h' ? get('H') : get('W');  // true input extent (op_spec.cpp:237-240)
  }
  return td.ndims;
}

int64_t OpDesc::tensor_elems(int ti, bool padded) const {
  int64_t dims[kMaxDims];
  int n = tensor_dims(ti, padded, dims);
  int64_t e = 1;
  for (int d = 0; d < n; ++d) e *= dims[d];
  return e;
}

void OpDesc::affine_coefs(int ti, int64_t* coef) const {
  int64_t dims[kMaxDims];
  int n = tensor_dims(ti, false, dims);
  for (int a = 0; a < kMaxAxes; ++a) coef[a] = 0;
  int64_t s = 1;
  for (int d = n - 1; d >= 0; --d) {
    const DimMap& m = t[ti].dim[d];
    if (m.win < 0) {
      coef[m.axis] += s;
    } else {
      coef[m.axis] += s * stride;
      coef[m.win] += s;
    }
    s *= dims[d];
  }
}

int64_t OpDesc::flops_padded() const {
  int64_t iters = 1;
  for (int a = 0; a < naxes; ++a) iters *= ax[a].padded;
  switch (kind) {
    case Kind::Gemm:
    case Kind::Gemv:
    case Kind::Conv2d:
    case Kind::DwConv2d:
      return 2 * iters;
    case Kind::AvgPool2d:
      return iters;
    case Kind::Softmax:
      return 5 * iters;
  }
  return iters;
}

double OpDesc::flops_true() const {
  double iters = 1;
  for (int a = 0; a < naxes; ++a) iters *= static_cast<double>(ax[a].extent);
  iters *= static_cast<double>(batch);
  switch (kind) {
    case Kind::AvgPool2d: return iters;
    case Kind::Softmax: return 5 * iters;
    default: return 2 * iters;
  }
}

double OpDesc::bytes_true() const {
  double b = 0;
  for (int ti = 0; ti < ntensors; ++ti) b += static_cast<double>(tensor_elems(ti, false));
  return b * dtype_bytes * static_cast<double>(batch);
}

int OpDesc::input_count() const { return ntensors - 1; }
int OpDesc::output_index() const { return ntensors - 1; }

std::string OpDesc::to_json() const {
  std::ostringstream os;
  os << "{\"kind\":\"" << kind_name(kind) << "\"";
  switch (kind) {
    case Kind::Gemm:
      os << ",\"M\":" << get('M') << ",\"K\":" << get('K') << ",\"N\":" << get('N');
      if (batch != 1) os << ",\"batch\":" << batch;
      break;
    case Kind::Gemv:
    case Kind::Softmax:
      os << ",\"M\":" << get('M') << ",\"N\":" << get('N');
      break;
    case Kind::Conv2d:
      os << ",\"I\":[" << get('N') << "," << get('C') << "," << get('H') << "," << get('W') << "],\"K\":["
         << get('F') << "," << get('C') << "," << get('R') << "," << get('S') << "],\"S\":" << stride;
      break;
    case Kind::DwConv2d:
      os << ",\"I\":[" << get('N') << "," << get('C') << "," << get('H') << "," << get('W') << "],\"K\":["
         << get('C') << ",1," << get('R') << "," << get('S') << "],\"S\":" << stride;
      break;
    case Kind::AvgPool2d:
      os << ",\"I\":[" << get('N') << "," << get('C') << "," << get('H') << "," << get('W') << "],\"F\":" << get('F')
         << ",\"S\":" << stride;
      break;
  }
  os << ",\"dtype_bytes\":" << dtype_bytes << "}";
  return os.str();
}

std::string OpDesc::label() const {
  std::ostringstream os;
  os << kind_name(kind) << "(";
  for (int a = 0; a < naxes; ++a) os << (a ? "," : "") << ax[a].name << "=" << ax[a].extent;
  os << ")";
  return os.str();
}

bool OpDesc::operator==(const OpDesc& o) const {
  if (kind != o.kind || dtype_bytes != o.dtype_bytes || stride != o.stride || batch != o.batch || naxes != o.naxes)
    return false;
  for (int a = 0; a < naxes; ++a)
    if (ax[a].extent != o.ax[a].extent) return false;
  return true;
}

}  // namespace gb
