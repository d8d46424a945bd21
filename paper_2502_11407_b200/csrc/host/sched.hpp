// Schedule state (the paper's ETIR) and the four scheduling actions.
//
// Semantics follow the reference's ETIRState (include/gensor/etir.hpp:41-80, src/etir.cpp):
//   tile(a, l)  level l in [1, L] (code numbering: 1 = outermost cache level = CTA tile,
//               L = innermost = thread tile); tile(a, 0) is the padded extent;
//   vt(a)       virtual-thread stride on spatial axes (1 on reduce axes);
//   cur         current memory level; Tile/InvTile edit level cur+1 and every deeper level
//               follows the edited tile until Cache commits it (etir.cpp:106-107).
// The state is a fixed-size POD so candidate evaluation copies ~600 bytes instead of
// allocating nested vectors; the op it belongs to is passed alongside, never stored.
#pragma once

#include <cstdint>
#include <string>

#include "op.hpp"

namespace gb {

enum class ActKind : uint8_t { Tile = 0, InvTile = 1, SetVThread = 2, Cache = 3 };

const char* act_kind_name(ActKind k);

// Lexicographic order (kind, axis, factor) is the reference's tie-break order (etir.hpp:27).
struct Action {
  ActKind kind = ActKind::Cache;
  int axis = -1;
  int64_t factor = 0;
  friend bool operator==(const Action& a, const Action& b) {
    return a.kind == b.kind && a.axis == b.axis && a.factor == b.factor;
  }
  friend bool operator<(const Action& a, const Action& b) {
    if (a.kind != b.kind) return a.kind < b.kind;
    if (a.axis != b.axis) return a.axis < b.axis;
    return a.factor < b.factor;
  }
};

std::string action_str(const Action& a, const OpDesc& op);

struct Sched {
  int L = 0;    // schedulable levels
  int cur = 0;  // current memory level
  int64_t tiles[kMaxAxes][kMaxLevels] = {};  // tiles[a][l-1]
  int64_t vts[kMaxAxes] = {};

  static Sched initial(const OpDesc& op, int levels);

  bool complete() const { return cur == L; }
  int edit_level() const { return cur + 1; }
  int64_t tile(const OpDesc& op, int a, int level) const {
    return level == 0 ? op.ax[a].padded : tiles[a][level - 1];
  }
  int64_t vt(int a) const { return vts[a]; }
  void tiles_at(const OpDesc& op, int level, int64_t* out) const {
    for (int a = 0; a < op.naxes; ++a) out[a] = tile(op, a, level);
  }

  bool legal(const OpDesc& op, const Action& act) const;
  Sched apply(const OpDesc& op, const Action& act) const;       // throws IllegalAction / AxisNotFound
  void apply_unchecked(const OpDesc& op, const Action& act);     // caller guarantees legality

  bool same(const Sched& o, int naxes) const;
  std::string repr(const OpDesc& op) const;  // "L1 m=[16,8]v2 n=[8,8]v1 k=[64,64]" (etir.cpp:129-139)
  std::string to_json(const OpDesc& op) const;
};

}  // namespace gb
