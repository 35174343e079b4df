// planner.cpp -- host-side motif decomposition and join-program compiler.
//
// Decomposition follows PAPER.md §3.3 with the motif set {M3-O, M3, M2}
// (triangle, wedge, edge; P:180 naming):
//   * at each iteration the motifs are tried in descending size ("traverse the chosen
//     motif set in descending order of size"); equal sizes in the fixed order M3-O > M3
//     (DESIGN reading Q9);
//   * a single match of the motif in the reduced pattern is found by a first-match
//     backtracking search ("we only require finding a single match");
//   * boundary nodes = slice vertices with still-uncovered incident edges; the
//     non-boundary vertices are removed from the reduced pattern, boundary vertices kept;
//   * the overlap with the union of earlier slices becomes the join constraints (P:250,
//     every shared vertex, as Fig. 2 emits both C1 and C2).
// A match is accepted only if it covers at least one uncovered edge and (after the first
// slice) shares a vertex with the earlier slices, so every join has constraints and
// the loop terminates (M2 always matches an uncovered edge next to the covered part of a
// connected pattern).
//
// Join program: slices are executed left-deep in slice order (reading Q10).  Each
// slice contributes its not-yet-placed vertices as one step; every pattern edge between a new
// vertex and an already-placed vertex is enforced when the later endpoint is placed (the
// slice's own key constraints plus closing edges pushed down from later slices: a selection
// pushdown that leaves the final table unchanged).  Slices whose vertices are all
// placed therefore need no step of their own (their joins are pure closing-edge probes).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <sstream>

#include "dm_internal.h"

namespace dm {

namespace {

struct MotifT {
  int id;
  int nv;
  std::vector<std::pair<int, int>> e;
};

const MotifT kM3O{DM_MOTIF_M3O, 3, {{0, 1}, {1, 2}, {0, 2}}};
const MotifT kM3{DM_MOTIF_M3, 3, {{0, 1}, {1, 2}}};
const MotifT kM2{DM_MOTIF_M2, 2, {{0, 1}}};

struct Pat {
  int k;
  std::vector<std::vector<char>> adj;
  bool has(int a, int b) const { return adj[a][b] != 0; }
};

bool match_rec(const Pat &P, const MotifT &M, const std::vector<char> &alive,
               const std::vector<std::vector<char>> &covered, const std::vector<char> &in_union,
               bool first, int depth, int cur[3]) {
  if (depth == M.nv) {
    bool unc = false, touch = first;
    for (auto &e : M.e)
      if (!covered[cur[e.first]][cur[e.second]]) unc = true;
    for (int s = 0; s < M.nv; ++s)
      if (in_union[cur[s]]) touch = true;
    return unc && touch;
  }
  for (int v = 0; v < P.k; ++v) {
    if (!alive[v]) continue;
    bool ok = true;
    for (int s = 0; s < depth && ok; ++s)
      if (cur[s] == v) ok = false;
    for (auto &e : M.e) {  // motif edges to earlier slots must be pattern edges
      if (!ok) break;
      if (e.first == depth && e.second < depth && !P.has(v, cur[e.second])) ok = false;
      if (e.second == depth && e.first < depth && !P.has(v, cur[e.first])) ok = false;
    }
    if (!ok) continue;
    cur[depth] = v;
    if (match_rec(P, M, alive, covered, in_union, first, depth + 1, cur)) return true;
  }
  return false;
}

// First match (ascending vertex ids per slot) of motif M in the reduced pattern (alive
// vertices, all pattern edges among them), subject to: covers >= 1 uncovered edge and,
// unless `first`, touches the union of earlier slices.
bool first_match(const Pat &P, const MotifT &M, const std::vector<char> &alive,
                 const std::vector<std::vector<char>> &covered, const std::vector<char> &in_union,
                 bool first, int out[3]) {
  int cur[3] = {-1, -1, -1};
  if (!match_rec(P, M, alive, covered, in_union, first, 0, cur)) return false;
  for (int s = 0; s < M.nv; ++s) out[s] = cur[s];
  return true;
}


// Placement order of a slice execution order: the first vertex, then each slice's unplaced
// vertices (each with a placed pattern neighbour -- slices are connected).
bool placement_order(const Pat &P, const Plan &plan, const std::vector<int> &order, int first,
                     std::vector<int> &out) {
  const int k = P.k;
  std::vector<char> placed(k, 0);
  out.assign(1, first);
  placed[first] = 1;
  for (int si : order) {
    const Slice &s = plan.slices[(size_t)si];
    std::vector<int> fresh;
    for (int i = 0; i < s.nv; ++i)
      if (!placed[s.v[i]]) fresh.push_back(s.v[i]);
    while (!fresh.empty()) {
      size_t pick = fresh.size();
      for (size_t j = 0; j < fresh.size() && pick == fresh.size(); ++j)
        for (int u = 0; u < k; ++u)
          if (P.adj[fresh[j]][u] && placed[u]) { pick = j; break; }
      if (pick == fresh.size()) return false;
      placed[fresh[pick]] = 1;
      out.push_back(fresh[pick]);
      fresh.erase(fresh.begin() + (long)pick);
    }
  }
  return (int)out.size() == k;
}

// Frontier-size model for one step placing vertices ord[pos..pos+nv) after `pos` placed
// vertices: the first expansion from the implicit vertex table grows rows by avg_degree, later
// ones by the size-biased degree; every extra join key keeps a fraction
// q = max(closure, d/(n-1)).  A 2-vertex count-only last step whose second vertex has the same
// keys as the first (a "shared-key pair", e.g. both apexes of a diamond) enumerates pairs of
// the first vertex's list.  Cost = candidates x compared columns + bytes of every materialized
// level (written + read).
struct StepCost {
  double rows_out, cost;
};
StepCost step_cost(const Pat &P, const std::vector<int> &ord, int pos, int nv, double rows,
                   bool last, const PlanStats &st) {
  const double n = std::max(2.0, st.n);
  const double d1 = std::max(1.0, st.avg_degree), d2 = std::max(1.0, st.fwd_degree);
  const double q = std::min(1.0, std::max(st.closure, d1 / (n - 1.0)));
  double cost = 0.0, r = rows;
  int keys0 = 0;
  for (int j = 0; j < nv; ++j) {
    const int v = ord[(size_t)(pos + j)];
    int keys = 0;
    for (int i = 0; i < pos + j; ++i) keys += P.adj[v][ord[(size_t)i]] ? 1 : 0;
    const double dexp = (pos == 1 && j == 0) ? d1 : d2;
    const bool shared = j == 1 && last && st.count_only &&
                        keys - (P.adj[v][ord[(size_t)pos]] ? 1 : 0) == keys0;
    if (shared) {
      const double list = std::max(1.0, r / std::max(1.0, rows));  // first vertex's list per row
      cost += r * list * (pos + j + 1);
      r *= list * (P.adj[v][ord[(size_t)pos]] ? q : 1.0);
    } else {
      cost += r * dexp * (pos + j + 1);
      r *= dexp * std::pow(q, keys - 1);
    }
    keys0 = keys;
  }
  if (!last || !st.count_only) cost += 2.0 * 4.0 * r * (double)(((pos + nv) + 3) & ~3);
  return {r, cost};
}

// Compile a placement order into kernel steps: consecutive groups of 1 or 2 vertices chosen
// by dynamic programming over the frontier-size model (the rows after a prefix do not depend
// on the grouping).  Every pattern edge between a new vertex and an earlier one is enforced
// when the later endpoint is placed (selection pushdown, DESIGN R1).
double compile_order(const Pat &P, int mode, const std::vector<int> &ord, Plan &plan,
                     const PlanStats &st) {
  const int k = P.k;
  plan.steps.clear();
  plan.col_pvert = ord;
  plan.pvert_col.assign(k, -1);
  for (int c = 0; c < k; ++c) plan.pvert_col[ord[(size_t)c]] = c;
  plan.first_vertex = ord[0];
  std::vector<double> rows(k + 1, 0.0);  // rows after each prefix (grouping independent)
  rows[1] = std::max(2.0, st.n);
  for (int i = 1; i < k; ++i) rows[i + 1] = step_cost(P, ord, i, 1, rows[i], false, st).rows_out;
  const double INF = 1e300;
  std::vector<double> best(k + 1, INF);
  std::vector<int> take(k + 1, 0);
  best[1] = 0.0;
  const bool deep = st.count_only && st.max_degree <= 4;  // row-serial ELL last step
  for (int i = 2; i <= k; ++i) {
    for (int g = 1; g <= (deep && i == k ? kMaxNew : 2) && g < i; ++g) {
      const int pos = i - g;
      if (best[pos] >= INF) continue;
      const double c = best[pos] + step_cost(P, ord, pos, g, rows[pos], i == k, st).cost;
      if (c < best[i]) {
        best[i] = c;
        take[i] = g;
      }
    }
  }
  std::vector<int> groups;
  for (int i = k; i > 1; i -= take[i]) groups.push_back(take[i]);
  std::reverse(groups.begin(), groups.end());
  int pos = 1;
  for (int g : groups) {
    Step stp;
    stp.in_w = pos;
    for (int j = 0; j < g; ++j) {
      const int v = ord[(size_t)(pos + j)];
      StepVertex sv;
      sv.pvert = v;
      for (int c = 0; c < pos + j; ++c) {
        if (P.adj[v][ord[(size_t)c]]) sv.nbr[sv.n_nbr++] = c;
        else if (mode == DM_INDUCED) sv.non[sv.n_non++] = c;
      }
      stp.nv[stp.n_new++] = sv;
    }
    plan.steps.push_back(stp);
    pos += g;
  }
  return k == 1 ? 0.0 : best[k];
}

}  // namespace


dm_status build_plan(int32_t k, const int32_t *p_edges, int64_t pm, int32_t motifs, int32_t mode,
                     Plan &out, const PlanStats &stats) {
  if (k < 1) return fail(DM_ERR_ARG, "pattern must have k >= 1 vertices");
  if (k > DM_MAX_PATTERN) return fail(DM_ERR_UNSUPPORTED, "pattern larger than DM_MAX_PATTERN");
  if (pm < 0 || (pm > 0 && !p_edges)) return fail(DM_ERR_ARG, "bad pattern edge list");
  if (mode != DM_MONO && mode != DM_INDUCED) return fail(DM_ERR_ARG, "mode must be DM_MONO or DM_INDUCED");
  Pat P{k, std::vector<std::vector<char>>(k, std::vector<char>(k, 0))};
  for (int64_t i = 0; i < pm; ++i) {
    int a = p_edges[2 * i], b = p_edges[2 * i + 1];
    if (a < 0 || b < 0 || a >= k || b >= k) return fail(DM_ERR_VERTEX_RANGE, "pattern edge endpoint out of range");
    if (a == b) return fail(DM_ERR_SELF_LOOP, "pattern self-loop");
    P.adj[a][b] = P.adj[b][a] = 1;
  }
  // connectivity ("we assume all graphs are ... connected")
  {
    std::vector<char> seen(k, 0);
    std::vector<int> st{0};
    seen[0] = 1;
    int cnt = 1;
    while (!st.empty()) {
      int v = st.back();
      st.pop_back();
      for (int u = 0; u < k; ++u)
        if (P.adj[v][u] && !seen[u]) { seen[u] = 1; ++cnt; st.push_back(u); }
    }
    if (cnt != k) return fail(DM_ERR_PATTERN_DISCONNECTED, "pattern graph is not connected");
  }
  Plan plan;
  plan.k = k;
  plan.mode = mode;
  plan.motifs = (motifs & (DM_MOTIF_M2 | DM_MOTIF_M3 | DM_MOTIF_M3O)) | DM_MOTIF_M2;
  for (int a = 0; a < k; ++a)
    for (int b = a + 1; b < k; ++b)
      if (P.adj[a][b]) plan.edges.push_back({a, b});

  // ------------------------------------------------------------ decomposition (§3.3)
  std::vector<const MotifT *> order;
  if (plan.motifs & DM_MOTIF_M3O) order.push_back(&kM3O);
  if (plan.motifs & DM_MOTIF_M3) order.push_back(&kM3);
  order.push_back(&kM2);
  std::vector<char> alive(k, 1), in_union(k, 0);
  std::vector<std::vector<char>> covered(k, std::vector<char>(k, 0));
  for (int a = 0; a < k; ++a)
    for (int b = 0; b < k; ++b)
      if (!P.adj[a][b]) covered[a][b] = 1;  // non-edges never need covering
  auto uncovered_left = [&]() {
    for (auto &e : plan.edges)
      if (!covered[e.first][e.second]) return true;
    return false;
  };
  while (uncovered_left()) {
    int m[3];
    const MotifT *used = nullptr;
    for (const MotifT *M : order)
      if (first_match(P, *M, alive, covered, in_union, plan.slices.empty(), m)) { used = M; break; }
    if (!used) return fail(DM_ERR_ARG, "internal: decomposition stalled");
    Slice s;
    s.motif = used->id;
    s.nv = used->nv;
    for (int i = 0; i < used->nv; ++i) {
      s.v[i] = m[i];
      if (in_union[m[i]]) s.c[s.nc++] = m[i];
    }
    for (auto &e : used->e) covered[m[e.first]][m[e.second]] = covered[m[e.second]][m[e.first]] = 1;
    for (int i = 0; i < used->nv; ++i) in_union[m[i]] = 1;
    for (int i = 0; i < used->nv; ++i) {  // boundary nodes stay, the others are removed
      bool boundary = false;
      for (int u = 0; u < k; ++u)
        if (!covered[m[i]][u]) boundary = true;
      if (!boundary) alive[m[i]] = 0;
    }
    plan.slices.push_back(s);
  }

  // ------------------------------------------------------------ join program
  if (plan.slices.empty()) {  // k == 1: the result is the implicit vertex table
    plan.first_vertex = 0;
    plan.col_pvert = {0};
    plan.pvert_col = {0};
    out = std::move(plan);
    return DM_OK;
  }
  // Candidate execution orders: every (seed slice, first vertex) pair, then greedily the
  // lowest-index slice that shares a vertex with the placed ones (left-deep; the paper's own
  // order is the candidate seeded by slice 0, and "the join order can also be
  // reversed").  The cheapest order under a simple frontier-size model wins.
  const int ns = (int)plan.slices.size();
  double best_cost = -1.0;
  Plan best;
  for (int seed = 0; seed < ns; ++seed) {
    for (int fv = 0; fv < plan.slices[seed].nv; ++fv) {
      std::vector<int> order{seed};
      std::vector<char> used(ns, 0), placed(k, 0);
      used[seed] = 1;
      for (int i = 0; i < plan.slices[seed].nv; ++i) placed[plan.slices[seed].v[i]] = 1;
      while ((int)order.size() < ns) {
        int pick = -1;
        for (int si = 0; si < ns && pick < 0; ++si) {
          if (used[si]) continue;
          for (int i = 0; i < plan.slices[si].nv; ++i)
            if (placed[plan.slices[si].v[i]]) { pick = si; break; }
        }
        if (pick < 0) break;
        used[pick] = 1;
        order.push_back(pick);
        for (int i = 0; i < plan.slices[pick].nv; ++i) placed[plan.slices[pick].v[i]] = 1;
      }
      if ((int)order.size() != ns) continue;
      Plan cand = plan;
      std::vector<int> ord;
      if (!placement_order(P, plan, order, plan.slices[seed].v[fv], ord)) continue;
      cand.order = order;
      const double cost = compile_order(P, mode, ord, cand, stats);
      if (best_cost < 0 || cost < best_cost - 1e-9 * best_cost) {
        best_cost = cost;
        best = std::move(cand);
      }
    }
  }
  if (best_cost < 0) return fail(DM_ERR_ARG, "internal: no valid join order");
  if ((int)best.col_pvert.size() != k) return fail(DM_ERR_ARG, "internal: not all pattern vertices placed");
  if ((int)best.steps.size() > DM_MAX_STEPS) return fail(DM_ERR_UNSUPPORTED, "too many join steps");
  out = std::move(best);
  return DM_OK;
}

std::string Plan::describe() const {
  static const char *names[8] = {"?", "M2", "M3", "?", "M3-O", "?", "?", "?"};
  std::ostringstream o;
  o << "{\"k\":" << k << ",\"mode\":\"" << (mode == DM_INDUCED ? "induced" : "mono")
    << "\",\"first_vertex\":" << first_vertex << ",\"slices\":[";
  for (size_t i = 0; i < slices.size(); ++i) {
    const Slice &s = slices[i];
    o << (i ? "," : "") << "{\"motif\":\"" << names[s.motif] << "\",\"vertices\":[";
    for (int j = 0; j < s.nv; ++j) o << (j ? "," : "") << s.v[j];
    o << "],\"constraints\":[";
    for (int j = 0; j < s.nc; ++j) o << (j ? "," : "") << s.c[j];
    o << "]}";
  }
  o << "],\"steps\":[";
  for (size_t i = 0; i < steps.size(); ++i) {
    const Step &st = steps[i];
    o << (i ? "," : "") << "{\"in_w\":" << st.in_w << ",\"new\":[";
    for (int j = 0; j < st.n_new; ++j) {
      const StepVertex &sv = st.nv[j];
      o << (j ? "," : "") << "{\"pvert\":" << sv.pvert << ",\"nbr_cols\":[";
      for (int t = 0; t < sv.n_nbr; ++t) o << (t ? "," : "") << sv.nbr[t];
      o << "],\"non_cols\":[";
      for (int t = 0; t < sv.n_non; ++t) o << (t ? "," : "") << sv.non[t];
      o << "]}";
    }
    o << "]}";
  }
  o << "],\"col_pvert\":[";
  for (size_t i = 0; i < col_pvert.size(); ++i) o << (i ? "," : "") << col_pvert[i];
  o << "]}";
  return o.str();
}

}  // namespace dm

// ------------------------------------------------------------------------------ C ABI
extern "C" {

dm_status dm_plan_create(int32_t k, const int32_t *p_edges, int64_t pm, int32_t motifs,
                         int32_t mode, dm_plan **out) {
  dm::clear_error();
  if (!out) return dm::fail(DM_ERR_ARG, "out is NULL");
  dm_plan *p = new (std::nothrow) dm_plan;
  if (!p) return dm::fail(DM_ERR_OOM, "host allocation failed");
  dm_status st = dm::build_plan(k, p_edges, pm, motifs, mode, p->p);
  if (st != DM_OK) {
    delete p;
    return st;
  }
  *out = p;
  return DM_OK;
}

dm_status dm_plan_create_ex(int32_t k, const int32_t *p_edges, int64_t pm, int32_t motifs,
                            int32_t mode, double n, double arcs, double sum_d2, double closure,
                            int32_t max_degree, int32_t count_only, dm_plan **out) {
  dm::clear_error();
  if (!out) return dm::fail(DM_ERR_ARG, "out is NULL");
  if (!(n >= 1) || !(arcs >= 0) || !(sum_d2 >= 0) || !(closure >= 0))
    return dm::fail(DM_ERR_ARG, "bad graph statistics");
  dm_plan *p = new (std::nothrow) dm_plan;
  if (!p) return dm::fail(DM_ERR_OOM, "host allocation failed");
  dm::PlanStats st;
  st.n = n;
  st.avg_degree = arcs / n;
  st.fwd_degree = arcs > 0 ? sum_d2 / arcs : 1.0;
  st.closure = closure;
  st.count_only = count_only != 0;
  st.max_degree = max_degree;
  dm_status s = dm::build_plan(k, p_edges, pm, motifs, mode, p->p, st);
  if (s != DM_OK) {
    delete p;
    return s;
  }
  *out = p;
  return DM_OK;
}

void dm_plan_destroy(dm_plan *p) { delete p; }

int32_t dm_plan_num_slices(const dm_plan *p) { return p ? (int32_t)p->p.slices.size() : -1; }

dm_status dm_plan_slice(const dm_plan *p, int32_t i, int32_t *motif, int32_t *n_vertices,
                        int32_t vertices[3], int32_t *n_constraints, int32_t constraints[3]) {
  dm::clear_error();
  if (!p || i < 0 || i >= (int32_t)p->p.slices.size()) return dm::fail(DM_ERR_ARG, "bad slice index");
  const dm::Slice &s = p->p.slices[(size_t)i];
  if (motif) *motif = s.motif;
  if (n_vertices) *n_vertices = s.nv;
  if (n_constraints) *n_constraints = s.nc;
  for (int j = 0; j < 3; ++j) {
    if (vertices) vertices[j] = s.v[j];
    if (constraints) constraints[j] = s.c[j];
  }
  return DM_OK;
}

int32_t dm_plan_num_steps(const dm_plan *p) { return p ? (int32_t)p->p.steps.size() : -1; }
int32_t dm_plan_first_vertex(const dm_plan *p) { return p ? p->p.first_vertex : -1; }

int32_t dm_plan_width(const dm_plan *p, int32_t level) {
  if (!p) return -1;
  const int ns = (int)p->p.steps.size();
  if (level < 0 || level > ns) return -1;
  return level == ns ? p->p.k : p->p.steps[(size_t)level].in_w;
}

int32_t dm_plan_stride(const dm_plan *p, int32_t level) {
  const int32_t w = dm_plan_width(p, level);
  return w < 0 ? -1 : ((w + 3) & ~3);
}

int32_t dm_plan_column_vertex(const dm_plan *p, int32_t column) {
  if (!p || column < 0 || column >= (int32_t)p->p.col_pvert.size()) return -1;
  return p->p.col_pvert[(size_t)column];
}

int64_t dm_plan_describe(const dm_plan *p, char *buf, int64_t len) {
  if (!p) return -1;
  std::string s = p->p.describe();
  if (buf && len > 0) {
    size_t n = std::min<size_t>((size_t)len - 1, s.size());
    std::memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
  return (int64_t)s.size() + 1;
}

}  // extern "C"
