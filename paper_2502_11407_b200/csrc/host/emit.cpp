// emit_source: a complete schedule -> deterministic, portable C source of its tiled loop nest
// (the SPEC's `emit_source(prog)`, and the `emit` CLI subcommand, SPEC.md:
// 519-520; the reference ships neither). The loop program is the SPEC's `lower` (SPEC.md:470-
// 478) in the order the execute families honour: level-1 tile loops outermost (spatial axes
// first, then reduce axes, each in axis order), down to the level-L loops, then the virtual-
// thread slice loops (strided across the level-(L-1) tile), then the scalar loops. Loops whose
// trip count is 1 are omitted; scalar loops with trip count <= 16 are marked unrolled. A guard
// is emitted iff some axis was padded, naming each padded axis exactly once. Accumulation is in
// double, the interpreter's convention.
#include "emit.hpp"

#include <sstream>
#include <vector>

namespace gb {
namespace {

struct Loop {
  int axis;
  int64_t radix;
  int64_t step;
  std::string var;
  bool scalar;
};

std::string indent(int depth) { return std::string(static_cast<size_t>(2 * depth), ' '); }

std::string affine(const OpDesc& op, const int64_t* coef) {
  std::ostringstream os;
  bool any = false;
  for (int a = 0; a < op.naxes; ++a) {
    if (!coef[a]) continue;
    os << (any ? " + " : "") << op.ax[a].name;
    if (coef[a] != 1) os << " * " << coef[a];
    any = true;
  }
  if (!any) os << "0";
  return os.str();
}

std::vector<Loop> loop_program(const OpDesc& op, const Sched& s) {
  std::vector<Loop> loops;
  const int L = s.L;
  auto vt = [&](int a) -> int64_t { return !op.ax[a].reduce && L > 0 ? s.vt(a) : 1; };
  for (int l = 1; l <= L; ++l)
    for (int pass = 0; pass < 2; ++pass)
      for (int a = 0; a < op.naxes; ++a) {
        if (static_cast<int>(op.ax[a].reduce) != pass) continue;
        const int64_t v = l == L ? vt(a) : 1;
        loops.push_back({a, s.tile(op, a, l - 1) / s.tile(op, a, l), s.tile(op, a, l) / v,
                         std::string(op.ax[a].name) + "_" + std::to_string(l), false});
      }
  for (int a = 0; a < op.naxes; ++a)
    if (vt(a) > 1)
      loops.push_back({a, vt(a), s.tile(op, a, L - 1) / vt(a), std::string(op.ax[a].name) + "_v", false});
  for (int pass = 0; pass < 2; ++pass)
    for (int a = 0; a < op.naxes; ++a) {
      if (static_cast<int>(op.ax[a].reduce) != pass) continue;
      loops.push_back({a, s.tile(op, a, L) / vt(a), 1, std::string(op.ax[a].name) + "_s", true});
    }
  std::vector<Loop> kept;
  for (auto& lp : loops)
    if (lp.radix > 1) kept.push_back(lp);
  return kept;
}

}  // namespace

std::string emit_source(const OpDesc& op, const Sched& s, const std::string& trace) {
  std::ostringstream os;
  const int nin = op.input_count();
  const int out = op.output_index();
  os << "/* gensor-b200 emit_source: " << op.label() << "\n"
     << " * schedule: " << s.repr(op) << "\n";
  if (!trace.empty()) os << " * trace: " << trace << "\n";
  os << " * loops: level-1 tiles (outermost) .. level-" << s.L
     << " tiles, vthread slices, scalar loops (unrolled when <= 16)\n"
     << " * accumulation: double (SPEC interpreter convention); inputs/outputs true-domain row-major\n"
     << " */\n#include <math.h>\n#include <stdint.h>\n\n";
  os << "void gensor_" << kind_name(op.kind) << "(";
  for (int ti = 0; ti < nin; ++ti) os << "const float* restrict " << op.t[ti].name << ", ";
  os << "double* restrict " << op.t[out].name << ") {\n";

  if (op.kind == Kind::Softmax) {
    const int64_t M = op.ax[0].extent, N = op.ax[1].extent;
    const char* X = op.t[0].name;
    const char* Y = op.t[out].name;
    os << "  for (int64_t m = 0; m < " << M << "; ++m) {\n"
       << "    double mx = -INFINITY, sum = 0.0;\n"
       << "    for (int64_t n = 0; n < " << N << "; ++n) mx = " << X << "[m * " << N << " + n] > mx ? " << X
       << "[m * " << N << " + n] : mx;\n"
       << "    for (int64_t n = 0; n < " << N << "; ++n) sum += exp((double)" << X << "[m * " << N
       << " + n] - mx);\n"
       << "    for (int64_t n = 0; n < " << N << "; ++n) " << Y << "[m * " << N << " + n] = exp((double)" << X
       << "[m * " << N << " + n] - mx) / sum;\n"
       << "  }\n}\n";
    return os.str();
  }

  const int64_t nout = op.tensor_elems(out, false);
  int depth = 1;
  if (op.batch > 1) {
    os << indent(depth) << "for (int64_t b = 0; b < " << op.batch << "; ++b) {\n";
    ++depth;
    for (int ti = 0; ti <= nin; ++ti) {
      const int64_t n = op.tensor_elems(ti, false);
      os << indent(depth) << (ti < nin ? "const float* " : "double* ") << op.t[ti].name << "_b = "
         << op.t[ti].name << " + b * " << n << ";\n";
    }
  }
  const std::string sfx = op.batch > 1 ? "_b" : "";
  os << indent(depth) << "for (int64_t e = 0; e < " << nout << "; ++e) " << op.t[out].name << sfx
     << "[e] = 0.0;\n";

  const std::vector<Loop> loops = loop_program(op, s);
  const int body_base = depth;
  for (const Loop& lp : loops) {
    os << indent(depth) << "for (int64_t " << lp.var << " = 0; " << lp.var << " < " << lp.radix << "; ++" << lp.var
       << ")";
    if (lp.scalar && lp.radix <= 16) os << "  /* unrolled */";
    os << "\n";
    ++depth;
  }
  os << indent(depth) << "{\n";
  ++depth;
  for (int a = 0; a < op.naxes; ++a) {
    os << indent(depth) << "const int64_t " << op.ax[a].name << " = ";
    bool any = false;
    for (const Loop& lp : loops) {
      if (lp.axis != a) continue;
      os << (any ? " + " : "") << lp.var;
      if (lp.step != 1) os << " * " << lp.step;
      any = true;
    }
    if (!any) os << "0";
    os << ";\n";
  }
  std::ostringstream guard;
  bool guarded = false;
  for (int a = 0; a < op.naxes; ++a) {
    if (op.ax[a].padded == op.ax[a].extent) continue;
    guard << (guarded ? " && " : "") << op.ax[a].name << " < " << op.ax[a].extent;
    guarded = true;
  }
  std::ostringstream stmt;
  int64_t coef[kMaxAxes];
  op.affine_coefs(out, coef);
  stmt << op.t[out].name << sfx << "[" << affine(op, coef) << "] += ";
  for (int ti = 0; ti < nin; ++ti) {
    op.affine_coefs(ti, coef);
    stmt << (ti ? " * " : "") << "(double)" << op.t[ti].name << sfx << "[" << affine(op, coef) << "]";
  }
  stmt << ";\n";
  if (guarded) {
    os << indent(depth) << "if (" << guard.str() << ")  /* guard: padded axes */\n" << indent(depth + 1) << stmt.str();
  } else {
    os << indent(depth) << stmt.str();
  }
  --depth;
  os << indent(depth) << "}\n";
  depth = body_base;
  if (op.kind == Kind::AvgPool2d) {
    const int64_t F = op.param("F");
    os << indent(depth) << "for (int64_t e = 0; e < " << nout << "; ++e) " << op.t[out].name << sfx << "[e] /= "
       << F * F << ".0;  /* true window F*F */\n";
  }
  if (op.batch > 1) os << indent(1) << "}\n";
  os << "}\n";
  return os.str();
}

}  // namespace gb
