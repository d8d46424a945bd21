// Construction-chain analysis (markov.hpp). Semantics follow the reference's markov-verify
// module (markov.cpp:40-364) so the differential tests against oracle/_ref can
// compare state for state; the implementation is this library's own (Tarjan SCCs over a CSR
// level graph, string-keyed state interning).
#include "markov.hpp"

#include <algorithm>
#include <cmath>
#include <deque>
#include <numeric>
#include <sstream>
#include <unordered_map>

#include "cost.hpp"
#include "error.hpp"
#include "json.hpp"

namespace gb {

int Chain::max_level() const {
  int m = 0;
  for (int l : level) m = std::max(m, l);
  return m;
}

namespace {

std::string state_key(const Sched& s, int naxes) {
  std::string k;
  k.reserve(static_cast<size_t>(8 * (1 + naxes * (s.L + 1))));
  auto put = [&](int64_t v) { k.append(reinterpret_cast<const char*>(&v), sizeof v); };
  put(s.cur);
  for (int a = 0; a < naxes; ++a) {
    put(s.vts[a]);
    for (int l = 0; l < s.L; ++l) put(s.tiles[a][l]);
  }
  return k;
}

// Upper bound on the space (for the SpaceTooLarge message): per axis, log2(padded)+1 tile
// choices per level, times the vthread options on spatial axes, times the level count.
double space_bound(const OpDesc& op, int L, size_t nvopts) {
  double b = L + 1;
  for (int a = 0; a < op.naxes; ++a) {
    const double choices = std::log2(static_cast<double>(op.ax[a].padded)) + 1;
    b *= std::pow(choices, L);
    if (!op.ax[a].reduce) b *= static_cast<double>(nvopts);
  }
  return b;
}

// The within-level subgraph in CSR form over local ids (ascending global id).
struct LevelGraph {
  std::vector<int> nodes;               // local -> global
  std::vector<int> start, to;           // CSR, edges in row order
  std::vector<char> art;
  int n() const { return static_cast<int>(nodes.size()); }
};

LevelGraph level_graph(const Chain& c, int level) {
  LevelGraph g;
  std::vector<int> local(static_cast<size_t>(c.size()), -1);
  for (int i = 0; i < c.size(); ++i)
    if (c.level[static_cast<size_t>(i)] == level) {
      local[static_cast<size_t>(i)] = g.n();
      g.nodes.push_back(i);
    }
  g.start.push_back(0);
  for (int u : g.nodes) {
    for (const ChainEdge& e : c.rows[static_cast<size_t>(u)]) {
      const int v = local[static_cast<size_t>(e.to)];
      if (v < 0) continue;
      g.to.push_back(v);
      g.art.push_back(e.artificial ? 1 : 0);
    }
    g.start.push_back(static_cast<int>(g.to.size()));
  }
  return g;
}

// Iterative Tarjan: component id per local node, returns the component count.
int tarjan(const LevelGraph& g, std::vector<int>& comp) {
  const int n = g.n();
  std::vector<int> index(static_cast<size_t>(n), -1), low(static_cast<size_t>(n), 0), stack;
  std::vector<char> on(static_cast<size_t>(n), 0);
  comp.assign(static_cast<size_t>(n), -1);
  int counter = 0, ncomp = 0;
  std::vector<std::pair<int, int>> call;  // (node, next edge)
  for (int s = 0; s < n; ++s) {
    if (index[static_cast<size_t>(s)] >= 0) continue;
    call.push_back({s, g.start[static_cast<size_t>(s)]});
    index[static_cast<size_t>(s)] = low[static_cast<size_t>(s)] = counter++;
    stack.push_back(s);
    on[static_cast<size_t>(s)] = 1;
    while (!call.empty()) {
      auto& [u, ei] = call.back();
      if (ei < g.start[static_cast<size_t>(u) + 1]) {
        const int v = g.to[static_cast<size_t>(ei++)];
        if (index[static_cast<size_t>(v)] < 0) {
          index[static_cast<size_t>(v)] = low[static_cast<size_t>(v)] = counter++;
          stack.push_back(v);
          on[static_cast<size_t>(v)] = 1;
          call.push_back({v, g.start[static_cast<size_t>(v)]});
        } else if (on[static_cast<size_t>(v)]) {
          low[static_cast<size_t>(u)] = std::min(low[static_cast<size_t>(u)], index[static_cast<size_t>(v)]);
        }
        continue;
      }
      const int done = u;
      call.pop_back();
      if (!call.empty()) {
        const int parent = call.back().first;
        low[static_cast<size_t>(parent)] = std::min(low[static_cast<size_t>(parent)], low[static_cast<size_t>(done)]);
      }
      if (low[static_cast<size_t>(done)] == index[static_cast<size_t>(done)]) {
        for (;;) {
          const int w = stack.back();
          stack.pop_back();
          on[static_cast<size_t>(w)] = 0;
          comp[static_cast<size_t>(w)] = ncomp;
          if (w == done) break;
        }
        ++ncomp;
      }
    }
  }
  return ncomp;
}

struct Pieces {  // weakly connected pieces (union-find with path halving)
  std::vector<int> p;
  explicit Pieces(int n) : p(static_cast<size_t>(n)) { std::iota(p.begin(), p.end(), 0); }
  int find(int x) {
    while (p[static_cast<size_t>(x)] != x) x = p[static_cast<size_t>(x)] = p[static_cast<size_t>(p[static_cast<size_t>(x)])];
    return x;
  }
  void join(int a, int b) { p[static_cast<size_t>(find(a))] = find(b); }
};

}  // namespace

Chain enumerate_chain(const OpDesc& op, const HwModel& hw, const ChainCaps& caps) {
  EngineCfg cfg;
  cfg.vthread_options = caps.vthread_options;
  cfg.max_tile_factor = caps.max_tile_factor;
  cfg.enable_inv_tile = caps.enable_inv_tile;
  cfg.mode = caps.mode;
  cfg.validate();
  Chain c;
  std::unordered_map<std::string, int> ids;
  std::deque<int> queue;
  auto intern = [&](const Sched& s) {
    auto [it, fresh] = ids.emplace(state_key(s, op.naxes), c.size());
    if (!fresh) return it->second;
    if (c.size() >= caps.max_states) {
      std::ostringstream os;
      os << "more than " << caps.max_states << " states (bound estimate "
         << space_bound(op, s.L, caps.vthread_options.size()) << ")";
      throw Error(Code::SpaceTooLarge, os.str());
    }
    c.states.push_back(s);
    c.rows.emplace_back();
    c.level.push_back(s.cur);
    c.complete.push_back(s.complete() ? 1 : 0);
    c.absorbing.push_back(0);
    queue.push_back(it->second);
    return it->second;
  };
  intern(Sched::initial(op, hw.schedulable_levels()));
  std::vector<Candidate> cands;
  while (!queue.empty()) {
    const int id = queue.front();
    queue.pop_front();
    const Sched s = c.states[static_cast<size_t>(id)];
    if (!candidates(op, hw, s, cfg, caps.fixed_iteration, cands)) {
      c.absorbing[static_cast<size_t>(id)] = 1;
      c.rows[static_cast<size_t>(id)].push_back({id, 1.0, Action{}, true});
      continue;
    }
    for (const Candidate& cd : cands) {
      if (cd.probability <= 0.0) continue;
      const int to = intern(s.apply(op, cd.action));
      c.rows[static_cast<size_t>(id)].push_back({to, cd.probability, cd.action, false});
    }
  }
  c.terminal.assign(c.states.size(), 0.0);
  double best = 0.0;
  for (size_t i = 0; i < c.states.size(); ++i) {
    if (!c.complete[i]) continue;
    c.terminal[i] = 1.0 / cost_of(op, hw, c.states[i], caps.mode).est_seconds;
    best = std::max(best, c.terminal[i]);
  }
  if (best > 0.0)
    for (double& v : c.terminal) v /= best;
  return c;
}

std::vector<bool> irreducible_per_level(const Chain& c, std::vector<int>* scc_counts) {
  const int levels = c.max_level() + 1;
  std::vector<bool> out(static_cast<size_t>(levels), true);
  if (scc_counts) scc_counts->assign(static_cast<size_t>(levels), 0);
  for (int l = 0; l < levels; ++l) {
    const LevelGraph g = level_graph(c, l);
    if (!g.n()) continue;
    std::vector<int> comp;
    const int ncomp = tarjan(g, comp);
    if (scc_counts) (*scc_counts)[static_cast<size_t>(l)] = ncomp;
    Pieces pc(g.n());
    for (int u = 0; u < g.n(); ++u)
      for (int e = g.start[static_cast<size_t>(u)]; e < g.start[static_cast<size_t>(u) + 1]; ++e)
        if (!g.art[static_cast<size_t>(e)]) pc.join(u, g.to[static_cast<size_t>(e)]);
    std::vector<int> piece_comp(static_cast<size_t>(g.n()), -1);
    for (int u = 0; u < g.n(); ++u) {
      int& pcmp = piece_comp[static_cast<size_t>(pc.find(u))];
      if (pcmp < 0) pcmp = comp[static_cast<size_t>(u)];
      else if (pcmp != comp[static_cast<size_t>(u)]) out[static_cast<size_t>(l)] = false;
    }
  }
  return out;
}

bool aperiodic(const Chain& c) {
  for (int l = 0; l <= c.max_level(); ++l)
    if (!aperiodic_level(c, l)) return false;
  return true;
}

bool aperiodic_level(const Chain& c, int l) {
  {
    const LevelGraph g = level_graph(c, l);
    const int n = g.n();
    Pieces pc(n);
    for (int u = 0; u < n; ++u)
      for (int e = g.start[static_cast<size_t>(u)]; e < g.start[static_cast<size_t>(u) + 1]; ++e)
        pc.join(u, g.to[static_cast<size_t>(e)]);
    // BFS depths from roots in id order; every edge u->v contributes |d(u)+1-d(v)| to the gcd of
    // its piece's cycle lengths.
    std::vector<int> depth(static_cast<size_t>(n), -1);
    std::deque<int> q;
    for (int r = 0; r < n; ++r) {
      if (depth[static_cast<size_t>(r)] >= 0) continue;
      depth[static_cast<size_t>(r)] = 0;
      q.push_back(r);
      while (!q.empty()) {
        const int u = q.front();
        q.pop_front();
        for (int e = g.start[static_cast<size_t>(u)]; e < g.start[static_cast<size_t>(u) + 1]; ++e) {
          const int v = g.to[static_cast<size_t>(e)];
          if (depth[static_cast<size_t>(v)] < 0) {
            depth[static_cast<size_t>(v)] = depth[static_cast<size_t>(u)] + 1;
            q.push_back(v);
          }
        }
      }
    }
    std::vector<int64_t> period(static_cast<size_t>(n), 0);
    std::vector<char> has_edge(static_cast<size_t>(n), 0);
    for (int u = 0; u < n; ++u) {
      const int p = pc.find(u);
      for (int e = g.start[static_cast<size_t>(u)]; e < g.start[static_cast<size_t>(u) + 1]; ++e) {
        const int v = g.to[static_cast<size_t>(e)];
        const int64_t d = std::llabs(static_cast<int64_t>(depth[static_cast<size_t>(u)]) + 1 - depth[static_cast<size_t>(v)]);
        period[static_cast<size_t>(p)] = std::gcd(period[static_cast<size_t>(p)], d);
        has_edge[static_cast<size_t>(p)] = 1;
      }
    }
    for (int r = 0; r < n; ++r)
      if (pc.find(r) == r && has_edge[static_cast<size_t>(r)] && period[static_cast<size_t>(r)] != 1) return false;
  }
  return true;
}

bool power_iteration_converges(const Chain& c, int level) {
  // Irreducible level with period d: from the uniform start, the components along the d-th
  // roots of unity vanish iff every cyclic class (BFS depth mod d) holds the same number of
  // states (their DFT over the class masses is zero); otherwise the iteration oscillates forever.
  const LevelGraph g = level_graph(c, level);
  const int n = g.n();
  if (!n) return false;
  std::vector<int> depth(static_cast<size_t>(n), -1);
  std::deque<int> q{0};
  depth[0] = 0;
  while (!q.empty()) {
    const int u = q.front();
    q.pop_front();
    for (int e = g.start[static_cast<size_t>(u)]; e < g.start[static_cast<size_t>(u) + 1]; ++e) {
      const int v = g.to[static_cast<size_t>(e)];
      if (depth[static_cast<size_t>(v)] < 0) {
        depth[static_cast<size_t>(v)] = depth[static_cast<size_t>(u)] + 1;
        q.push_back(v);
      }
    }
  }
  int64_t d = 0;
  for (int u = 0; u < n; ++u) {
    if (depth[static_cast<size_t>(u)] < 0) return false;
    for (int e = g.start[static_cast<size_t>(u)]; e < g.start[static_cast<size_t>(u) + 1]; ++e)
      d = std::gcd(d, std::llabs(static_cast<int64_t>(depth[static_cast<size_t>(u)]) + 1 -
                                 depth[static_cast<size_t>(g.to[static_cast<size_t>(e)])]));
  }
  if (d <= 1) return true;
  std::vector<int64_t> size(static_cast<size_t>(d), 0);
  for (int u = 0; u < n; ++u) ++size[static_cast<size_t>(depth[static_cast<size_t>(u)] % d)];
  return std::all_of(size.begin(), size.end(), [&](int64_t x) { return x == size[0]; });
}

std::vector<double> stationary(const Chain& c, int level, int* sweeps_out) {
  const LevelGraph g = level_graph(c, level);
  const int n = g.n();
  if (!n) throw Error(Code::NotErgodic, "no states at level " + std::to_string(level));
  std::vector<int> comp;
  tarjan(g, comp);
  for (int u = 0; u < n; ++u) {
    if (comp[static_cast<size_t>(u)] != comp[0]) throw Error(Code::NotErgodic, "level subchain is not irreducible");
    if (g.start[static_cast<size_t>(u)] == g.start[static_cast<size_t>(u) + 1])
      throw Error(Code::NotErgodic, "state without within-level transitions");
  }
  // Row-renormalised restriction of P (edge weights in CSR order).
  std::vector<double> w(g.to.size());
  for (int u = 0; u < n; ++u) {
    const auto& row = c.rows[static_cast<size_t>(g.nodes[static_cast<size_t>(u)])];
    double total = 0.0;
    std::vector<double> ps;
    for (const ChainEdge& e : row)
      if (c.level[static_cast<size_t>(e.to)] == level) {
        total += e.prob;
        ps.push_back(e.prob);
      }
    for (size_t k = 0; k < ps.size(); ++k) w[static_cast<size_t>(g.start[static_cast<size_t>(u)]) + k] = ps[k] / total;
  }
  std::vector<double> pi(static_cast<size_t>(n), 1.0 / n), next(static_cast<size_t>(n));
  int sweep = 0;
  for (;; ++sweep) {
    if (sweep >= 1000000) throw Error(Code::NotErgodic, "power iteration did not converge");
    std::fill(next.begin(), next.end(), 0.0);
    for (int u = 0; u < n; ++u)
      for (int e = g.start[static_cast<size_t>(u)]; e < g.start[static_cast<size_t>(u) + 1]; ++e)
        next[static_cast<size_t>(g.to[static_cast<size_t>(e)])] += pi[static_cast<size_t>(u)] * w[static_cast<size_t>(e)];
    double residual = 0.0;
    for (int u = 0; u < n; ++u) residual += std::fabs(next[static_cast<size_t>(u)] - pi[static_cast<size_t>(u)]);
    pi.swap(next);
    if (residual < 1e-12) break;
  }
  if (sweeps_out) *sweeps_out = sweep + 1;
  std::vector<double> full(static_cast<size_t>(c.size()), 0.0);
  for (int u = 0; u < n; ++u) full[static_cast<size_t>(g.nodes[static_cast<size_t>(u)])] = pi[static_cast<size_t>(u)];
  return full;
}

Values value_iteration(const Chain& c) {
  const int n = c.size();
  Values t;
  t.value.assign(static_cast<size_t>(n), 1.0);
  t.policy.assign(static_cast<size_t>(n), -1);
  for (int i = 0; i < n; ++i)
    if (c.complete[static_cast<size_t>(i)]) t.value[static_cast<size_t>(i)] = c.terminal[static_cast<size_t>(i)];
  auto best_of = [&](int i, const std::vector<double>& v, int* arg) {
    double best = 0.0;
    const auto& row = c.rows[static_cast<size_t>(i)];
    for (size_t k = 0; k < row.size(); ++k) {
      if (row[k].artificial) continue;
      const double x = row[k].prob * v[static_cast<size_t>(row[k].to)];
      if (x > best) {
        best = x;
        if (arg) *arg = static_cast<int>(k);
      }
    }
    return best;
  };
  const int cap = 10 * std::max(n, 1);
  std::vector<double> next(static_cast<size_t>(n));
  for (int sweep = 0;; ++sweep) {
    if (sweep >= cap) throw Error(Code::NoConvergence, "value iteration exceeded " + std::to_string(cap) + " sweeps");
    double delta = 0.0;
    for (int i = 0; i < n; ++i) {
      if (c.complete[static_cast<size_t>(i)]) {
        next[static_cast<size_t>(i)] = t.value[static_cast<size_t>(i)];
        continue;
      }
      next[static_cast<size_t>(i)] = best_of(i, t.value, nullptr);
      delta = std::max(delta, std::fabs(next[static_cast<size_t>(i)] - t.value[static_cast<size_t>(i)]));
    }
    t.value.swap(next);
    t.iterations = sweep + 1;
    if (delta < 1e-12) break;
  }
  for (int i = 0; i < n; ++i)
    if (!c.complete[static_cast<size_t>(i)]) best_of(i, t.value, &t.policy[static_cast<size_t>(i)]);
  return t;
}

namespace {

std::string action_json(const Action& a) {
  std::ostringstream os;
  os << "[" << static_cast<int>(a.kind) << "," << a.axis << "," << a.factor << "]";
  return os.str();
}

}  // namespace

std::string analysis_json(const OpDesc& op, const HwModel& hw, const ChainCaps& caps, bool detail) {
  const Chain c = enumerate_chain(op, hw, caps);
  std::vector<int> sccs;
  const std::vector<bool> irr = irreducible_per_level(c, &sccs);
  std::vector<bool> aper_l(irr.size());
  bool aper = true;
  for (size_t l = 0; l < irr.size(); ++l) aper = aper && (aper_l[l] = aperiodic_level(c, static_cast<int>(l)));
  const Values vt = value_iteration(c);
  int ncomplete = 0, nabsorbing = 0;
  for (int i = 0; i < c.size(); ++i) {
    ncomplete += c.complete[static_cast<size_t>(i)];
    nabsorbing += c.absorbing[static_cast<size_t>(i)];
  }
  std::ostringstream os;
  os << "{\"op\":" << json::quote(op.label()) << ",\"states\":" << c.size() << ",\"complete\":" << ncomplete
     << ",\"absorbing\":" << nabsorbing << ",\"aperiodic\":" << (aper ? "true" : "false") << ",\"levels\":[";
  std::vector<std::vector<double>> pis(irr.size());
  for (size_t l = 0; l < irr.size(); ++l) {
    int count = 0;
    for (int lv : c.level) count += lv == static_cast<int>(l);
    os << (l ? "," : "") << "{\"level\":" << l << ",\"states\":" << count << ",\"sccs\":" << sccs[l]
       << ",\"irreducible\":" << (irr[l] ? "true" : "false") << ",\"aperiodic\":" << (aper_l[l] ? "true" : "false")
       << ",\"stationary\":";
    // The reference's power iteration (markov.cpp:275-317) needs one SCC; on a periodic level it
    // converges only from a class-balanced start, else it spins to its sweep cap and throws.
    if (sccs[l] != 1 || !power_iteration_converges(c, static_cast<int>(l))) {
      os << "{\"error\":\"NotErgodic: "
         << (sccs[l] != 1 ? "level has several SCCs" : "periodic level: power iteration does not converge") << "\"}";
    } else {
      try {
        int sweeps = 0;
        pis[l] = stationary(c, static_cast<int>(l), &sweeps);
        double h = 0.0, sum = 0.0;
        for (double p : pis[l]) {
          sum += p;
          if (p > 0) h -= p * std::log(p);
        }
        os << "{\"entropy\":" << json::num(h) << ",\"sum\":" << json::num(sum) << ",\"sweeps\":" << sweeps << "}";
      } catch (const Error& e) {
        os << "{\"error\":" << json::quote(e.what()) << "}";
      }
    }
    os << "}";
  }
  // Greedy policy path from the unscheduled state and its product-form payoff.
  std::ostringstream path;
  int at = 0, steps = 0;
  double payoff = 1.0;
  path << "[";
  while (!c.complete[static_cast<size_t>(at)] && vt.policy[static_cast<size_t>(at)] >= 0 && steps <= c.size()) {
    const ChainEdge& e = c.rows[static_cast<size_t>(at)][static_cast<size_t>(vt.policy[static_cast<size_t>(at)])];
    path << (steps ? "," : "") << action_json(e.action);
    payoff *= e.prob;
    at = e.to;
    ++steps;
  }
  path << "]";
  payoff *= c.complete[static_cast<size_t>(at)] ? c.terminal[static_cast<size_t>(at)] : 0.0;
  os << "],\"value\":{\"initial\":" << json::num(vt.value[0]) << ",\"iterations\":" << vt.iterations
     << ",\"policy_path\":" << path.str() << ",\"end_state\":" << json::quote(c.states[static_cast<size_t>(at)].repr(op))
     << ",\"end_payoff\":" << json::num(payoff) << "}";
  if (detail) {
    os << ",\"detail\":{\"states\":[";
    for (int i = 0; i < c.size(); ++i) os << (i ? "," : "") << json::quote(c.states[static_cast<size_t>(i)].repr(op));
    os << "],\"complete\":[";
    for (int i = 0; i < c.size(); ++i) os << (i ? "," : "") << static_cast<int>(c.complete[static_cast<size_t>(i)]);
    os << "],\"absorbing\":[";
    for (int i = 0; i < c.size(); ++i) os << (i ? "," : "") << static_cast<int>(c.absorbing[static_cast<size_t>(i)]);
    os << "],\"terminal\":[";
    for (int i = 0; i < c.size(); ++i) os << (i ? "," : "") << json::num(c.terminal[static_cast<size_t>(i)]);
    os << "],\"rows\":[";
    for (int i = 0; i < c.size(); ++i) {
      os << (i ? "," : "") << "[";
      const auto& row = c.rows[static_cast<size_t>(i)];
      for (size_t k = 0; k < row.size(); ++k)
        os << (k ? "," : "") << "[" << row[k].to << "," << json::num(row[k].prob) << "," << action_json(row[k].action)
           << "," << (row[k].artificial ? 1 : 0) << "]";
      os << "]";
    }
    os << "],\"value\":[";
    for (int i = 0; i < c.size(); ++i) os << (i ? "," : "") << json::num(vt.value[static_cast<size_t>(i)]);
    os << "],\"policy\":[";
    for (int i = 0; i < c.size(); ++i) {
      const int p = vt.policy[static_cast<size_t>(i)];
      os << (i ? "," : "") << (p < 0 ? std::string("null") : action_json(c.rows[static_cast<size_t>(i)][static_cast<size_t>(p)].action));
    }
    os << "],\"stationary\":{";
    bool first = true;
    for (size_t l = 0; l < pis.size(); ++l) {
      if (pis[l].empty()) continue;
      os << (first ? "" : ",") << "\"" << l << "\":[";
      for (size_t i = 0; i < pis[l].size(); ++i) os << (i ? "," : "") << json::num(pis[l][i]);
      os << "]";
      first = false;
    }
    os << "}}";
  }
  os << "}";
  return os.str();
}

}  // namespace gb
