#include "sched.hpp"

#include <sstream>

#include "error.hpp"

namespace gb {

const char* act_kind_name(ActKind k) {
  switch (k) {
    case ActKind::Tile: return "tile";
    case ActKind::InvTile: return "inv_tile";
    case ActKind::SetVThread: return "set_vthread";
    case ActKind::Cache: return "cache";
  }
  return "?";
}

std::string action_str(const Action& a, const OpDesc& op) {
  std::string s = act_kind_name(a.kind);
  if (a.kind != ActKind::Cache) {
    std::string ax = (a.axis >= 0 && a.axis < op.naxes) ? op.ax[a.axis].name : std::to_string(a.axis);
    s += "(" + ax + "," + std::to_string(a.factor) + ")";
  }
  return s;
}

Sched Sched::initial(const OpDesc& op, int levels) {
  if (levels < 0 || levels > kMaxLevels)
    throw Error(Code::LevelOutOfRange, "schedulable levels " + std::to_string(levels));
  Sched s;
  s.L = levels;
  s.cur = 0;
  for (int a = 0; a < op.naxes; ++a) {
    for (int l = 0; l < levels; ++l) s.tiles[a][l] = op.ax[a].padded;
    s.vts[a] = 1;
  }
  return s;
}

bool Sched::legal(const OpDesc& op, const Action& act) const {
  if (act.kind == ActKind::Cache) return cur < L;
  if (act.axis < 0 || act.axis >= op.naxes) return false;
  const int a = act.axis;
  if (act.kind == ActKind::SetVThread) {
    // spatial only, power of two, not a no-op, no wider than the innermost tile (etir.cpp:74-78)
    return !op.ax[a].reduce && is_pow2(act.factor) && act.factor != vts[a] && act.factor <= tile(op, a, L);
  }
  if (cur >= L || act.factor < 2 || !is_pow2(act.factor)) return false;
  const int64_t t = tile(op, a, cur + 1);
  if (act.kind == ActKind::Tile) return t % act.factor == 0 && t / act.factor >= vts[a];
  return t * act.factor <= tile(op, a, cur);  // stay inside the next outer tile
}

void Sched::apply_unchecked(const OpDesc& op, const Action& act) {
  switch (act.kind) {
    case ActKind::Cache:
      ++cur;
      break;
    case ActKind::SetVThread:
      vts[act.axis] = act.factor;
      break;
    case ActKind::Tile:
    case ActKind::InvTile: {
      const int64_t t = tile(op, act.axis, cur + 1);
      const int64_t nt = act.kind == ActKind::Tile ? t / act.factor : t * act.factor;
      for (int l = cur + 1; l <= L; ++l) tiles[act.axis][l - 1] = nt;
      break;
    }
  }
}

Sched Sched::apply(const OpDesc& op, const Action& act) const {
  if (act.kind != ActKind::Cache && (act.axis < 0 || act.axis >= op.naxes))
    throw Error(Code::AxisNotFound, "axis index " + std::to_string(act.axis));
  if (!legal(op, act)) throw Error(Code::IllegalAction, action_str(act, op) + " in " + repr(op));
  Sched n = *this;
  n.apply_unchecked(op, act);
  return n;
}

bool Sched::same(const Sched& o, int naxes) const {
  if (L != o.L || cur != o.cur) return false;
  for (int a = 0; a < naxes; ++a) {
    if (vts[a] != o.vts[a]) return false;
    for (int l = 0; l < L; ++l)
      if (tiles[a][l] != o.tiles[a][l]) return false;
  }
  return true;
}

std::string Sched::repr(const OpDesc& op) const {
  std::ostringstream os;
  os << "L" << cur;
  for (int a = 0; a < op.naxes; ++a) {
    os << " " << op.ax[a].name << "=[";
    for (int l = 1; l <= L; ++l) os << (l > 1 ? "," : "") << tile(op, a, l);
    os << "]";
    if (!op.ax[a].reduce) os << "v" << vts[a];
  }
  return os.str();
}

std::string Sched::to_json(const OpDesc& op) const {
  std::ostringstream os;
  os << "{\"level\":" << cur << ",\"tiles\":[";
  for (int a = 0; a < op.naxes; ++a) {
    os << (a ? "," : "") << "[";
    for (int l = 1; l <= L; ++l) os << (l > 1 ? "," : "") << tile(op, a, l);
    os << "]";
  }
  os << "],\"vthreads\":[";
  for (int a = 0; a < op.naxes; ++a) os << (a ? "," : "") << vts[a];
  os << "],\"repr\":\"" << repr(op) << "\"}";
  return os.str();
}

}  // namespace gb
