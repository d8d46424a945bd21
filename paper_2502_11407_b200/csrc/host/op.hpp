// Operator description: the iteration domain of one tensor operator and its tensor access maps.
//
// Mirrors the reference's TensorOpSpec (include/gensor/op_spec.hpp:48-116, src/op_spec.cpp:70-287)
// with a flat, allocation-free layout so the construction engine's inner loops (candidate
// enumeration, greedy completion) never touch the heap:
//   * up to kMaxAxes loop axes, each with its true extent and the next-power-of-two scheduling
//     extent ("padded", op_spec.cpp:145);
//   * up to 3 tensors, each dim mapping one axis or an (output axis, window axis) pair for
//     strided-window dims (op_spec.cpp:150-193);
//   * every tensor's true-domain element offset is an affine function of the axis indices
//     (op_spec.cpp:251-262 with windowed coord = o*stride + w), exported per tensor as
//     per-axis coefficients — the layout contract the kernels and the oracle share.
// Reference kinds: gemm, gemv, conv2d, avgpool2d. Extensions for the B200 suite (no reference
// counterpart, parity unpinned by the reference): dwconv2d, softmax, and a "batch" count on gemm
// (independent GEMMs scheduled once and executed batch times).
#pragma once

#include <array>
#include <cstdint>
#include <string>

#include "json.hpp"

namespace gb {

constexpr int kMaxAxes = 8;
constexpr int kMaxLevels = 8;
constexpr int kMaxTensors = 3;
constexpr int kMaxDims = 4;

enum class Kind : uint8_t { Gemm, Gemv, Conv2d, AvgPool2d, DwConv2d, Softmax };

const char* kind_name(Kind k);
int64_t next_pow2(int64_t v);
bool is_pow2(int64_t v);

struct AxisDesc {
  char name[4] = {0, 0, 0, 0};
  int64_t extent = 1;
  int64_t padded = 1;
  bool reduce = false;
};

struct DimMap {
  int8_t axis = -1;
  int8_t win = -1;  // window axis for strided-window dims, -1 otherwise
};

struct TensorDesc {
  char name[4] = {0, 0, 0, 0};
  bool output = false;
  int8_t ndims = 0;
  DimMap dim[kMaxDims];
};

class OpDesc {
 public:
  static OpDesc parse(const json::Value& doc);
  static OpDesc parse_text(const std::string& text);

  Kind kind = Kind::Gemm;
  int dtype_bytes = 4;
  int64_t stride = 1;
  int64_t batch = 1;  // extension: independent repetitions of the whole domain (gemm only)
  int naxes = 0;
  AxisDesc ax[kMaxAxes];
  int ntensors = 0;
  TensorDesc t[kMaxTensors];

  // Named integer parameters (M,K,N / N,C,H,W,F,R,S,OH,OW), in the reference's sense.
  int64_t param(const char* name) const;

  int axis_index(const std::string& name) const;  // throws AxisNotFound

  // Distinct elements of each tensor touched by one tile (closed form, op_spec.cpp:210-225).
  void tile_elems(const int64_t* tile, int64_t* out) const;

  // Concrete dims of tensor `ti` on the true or padded domain (op_spec.cpp:227-243).
  int tensor_dims(int ti, bool padded, int64_t* dims) const;
  int64_t tensor_elems(int ti, bool padded) const;

  // True-domain affine layout: offset = sum_a idx[a] * coef[a] (elements).
  void affine_coefs(int ti, int64_t* coef) const;

  int64_t flops_padded() const;  // cost-model work on the padded domain (op_spec.cpp:275-287)
  double flops_true() const;     // algorithmic work on true extents (roofline numerator)
  double bytes_true() const;     // compulsory bytes: every input read once, output written once

  int input_count() const;
  int output_index() const;

  std::string to_json() const;
  std::string label() const;
  bool operator==(const OpDesc& o) const;

 private:
  // Parameter storage: fixed small table, insertion order irrelevant.
  std::array<std::pair<char, int64_t>, 12> params_{};  // keyed by a 1-char code, see op.cpp
  int nparams_ = 0;
  void set(char code, int64_t v);
  int64_t get(char code) const;
  void build();
};

}  // namespace gb
