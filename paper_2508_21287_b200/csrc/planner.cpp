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

// Motif templates in decomposition order: descending size, a cycle before the path of the same
// size (reading Q9 extended: M3-O > M3 as before).
const std::vector<const MotifDef *> &motif_defs() {
  static const MotifDef defs[] = {
      {DM_MOTIF_M12O, 12, true, "M12-O"}, {DM_MOTIF_M8, 8, false, "M8"}, {DM_MOTIF_M7, 7, false, "M7"},
      {DM_MOTIF_M6O, 6, true, "M6-O"},    {DM_MOTIF_M6, 6, false, "M6"}, {DM_MOTIF_M5, 5, false, "M5"},
      {DM_MOTIF_M4O, 4, true, "M4-O"},    {DM_MOTIF_M4, 4, false, "M4"}, {DM_MOTIF_M3O, 3, true, "M3-O"},
      {DM_MOTIF_M3, 3, false, "M3"},      {DM_MOTIF_M2, 2, false, "M2"}};
  static const std::vector<const MotifDef *> v = [] {
    std::vector<const MotifDef *> o;
    for (const auto &d : defs) o.push_back(&d);
    return o;
  }();
  return v;
}

const MotifDef *motif_def(int id) {
  for (const MotifDef *d : motif_defs())
    if (d->id == id) return d;
  return nullptr;
}

namespace {

inline bool tmpl_edge(const MotifDef &M, int a, int b) {
  if (a > b) std::swap(a, b);
  if (b == a + 1) return true;
  return M.cycle && a == 0 && b == M.nv - 1 && M.nv > 2;
}

struct Pat {
  int k;
  std::vector<std::vector<char>> adj;
  bool has(int a, int b) const { return adj[a][b] != 0; }
};

// First-match search budget (template vertex placements) per motif try: large motifs on large
// patterns are searched with a bounded backtracking; an exhausted budget counts as "no match"
// (the decomposition then falls through to smaller motifs, which always succeed -- M2).
constexpr long kMatchBudget = 200000;

bool match_rec(const Pat &P, const MotifDef &M, const std::vector<char> &alive,
               const std::vector<std::vector<char>> &covered, const std::vector<char> &in_union,
               bool first, int depth, int *cur, long &budget) {
  if (depth == M.nv) {
    bool unc = false, touch = first;
    for (int a = 0; a + 1 < M.nv; ++a)
      if (!covered[cur[a]][cur[a + 1]]) unc = true;
    if (M.cycle && M.nv > 2 && !covered[cur[0]][cur[M.nv - 1]]) unc = true;
    for (int s = 0; s < M.nv; ++s)
      if (in_union[cur[s]]) touch = true;
    if (!(unc && touch)) return false;
    // a table motif is joined through its index on template position 0: a path slice needs a
    // constrained endpoint (a cycle can be rotated onto any constrained vertex)
    if (motif_is_table(M.id) && !first && !M.cycle && !in_union[cur[0]] && !in_union[cur[M.nv - 1]])
      return false;
    return true;
  }
  for (int v = 0; v < P.k; ++v) {
    if (!alive[v]) continue;
    if (--budget < 0) return false;
    bool ok = true;
    for (int s = 0; s < depth && ok; ++s)
      if (cur[s] == v) ok = false;
    if (ok && depth > 0 && !P.has(v, cur[depth - 1])) ok = false;            // path edge
    if (ok && M.cycle && M.nv > 2 && depth == M.nv - 1 && !P.has(v, cur[0])) ok = false;  // closing
    if (!ok) continue;
    cur[depth] = v;
    if (match_rec(P, M, alive, covered, in_union, first, depth + 1, cur, budget)) return true;
  }
  return false;
}

// First match (ascending vertex ids per template position) of motif M in the reduced pattern
// (alive vertices, all pattern edges among them), subject to: covers >= 1 uncovered edge and,
// unless `first`, touches the union of earlier slices.
bool first_match(const Pat &P, const MotifDef &M, const std::vector<char> &alive,
                 const std::vector<std::vector<char>> &covered, const std::vector<char> &in_union,
                 bool first, int out[kMaxMotifV]) {
  int cur[kMaxMotifV];
  long budget = kMatchBudget;
  if (!match_rec(P, M, alive, covered, in_union, first, 0, cur, budget)) return false;
  for (int s = 0; s < M.nv; ++s) out[s] = cur[s];
  return true;
}

// Placement order of a slice execution order: the first vertex, then each slice's unplaced
// vertices (each with a placed pattern neighbour -- slices are connected).  spans[i] = (slice,
// first position in `out`, number of fresh vertices) in execution order.
struct Span {
  int slice, start, len;
};
bool placement_order(const Pat &P, const Plan &plan, const std::vector<int> &order, int first,
                     std::vector<int> &out, std::vector<Span> &spans) {
  const int k = P.k;
  std::vector<char> placed(k, 0);
  out.assign(1, first);
  spans.clear();
  placed[first] = 1;
  for (int si : order) {
    const Slice &s = plan.slices[(size_t)si];
    std::vector<int> fresh;
    for (int i = 0; i < s.nv; ++i)
      if (!placed[s.v[i]]) fresh.push_back(s.v[i]);
    spans.push_back({si, (int)out.size(), (int)fresh.size()});
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

int motif_bit_index(int id) {
  int b = 0;
  while (b < 31 && (1 << b) != id) ++b;
  return b;
}

// |Res(M)|: the built table's size, else a non-backtracking walk estimate (paths) times the
// closing probability (cycles).
double table_rows_estimate(const MotifDef &M, const PlanStats &st) {
  const double known = st.tab_rows[motif_bit_index(M.id)];
  if (known > 0) return known;
  const double n = std::max(2.0, st.n);
  const double d1 = std::max(1.0, st.avg_degree), d2 = std::max(1.0, st.fwd_degree);
  const double q = std::min(1.0, std::max(st.closure, d1 / (n - 1.0)));
  double r = n * d1 * std::pow(std::max(1.0, d2 - 1.0), M.nv - 2);
  if (M.cycle) r *= std::max(q, 1e-3);
  return r;
}

// Table step for slice T placing ord[pos..pos+g): choose the template automorphism that binds
// template position 0 (and, if possible, 1) to placed vertices; fill the step.  False if no
// placed vertex can take template position 0 (the slice is then joined by CSR steps).
bool make_table_step(const Pat &P, int mode, const std::vector<int> &ord, const std::vector<int> &col_of,
                     int pos, int g, const Slice &T, Step &stp) {
  const MotifDef &M = *motif_def(T.motif);
  const int L = M.nv;
  std::vector<std::vector<int>> autos;  // autos[a][p] = slice index of template position p
  for (int r = 0; r < (M.cycle ? L : 1); ++r)
    for (int refl = 0; refl < 2; ++refl) {
      std::vector<int> a((size_t)L);
      for (int p = 0; p < L; ++p) {
        const int q = refl ? (M.cycle ? (r - p + L) % L : L - 1 - p) : (M.cycle ? (r + p) % L : p);
        a[(size_t)p] = q;
      }
      autos.push_back(a);
    }
  auto placed = [&](int pv) { return col_of[(size_t)pv] >= 0 && col_of[(size_t)pv] < pos; };
  int best = -1, best_score = 0;
  for (size_t ai = 0; ai < autos.size(); ++ai) {
    const int v0 = T.v[autos[ai][0]], v1 = T.v[autos[ai][1]];
    if (!placed(v0)) continue;
    int score = 1 + (placed(v1) ? 2 : 0);
    if (score > best_score) {
      best_score = score;
      best = (int)ai;
    }
  }
  if (best < 0) return false;
  const std::vector<int> &A = autos[(size_t)best];
  stp = Step();
  stp.in_w = pos;
  stp.n_new = g;
  stp.tab_motif = M.id;
  stp.key0 = col_of[(size_t)T.v[A[0]]];
  stp.key1 = placed(T.v[A[1]]) ? col_of[(size_t)T.v[A[1]]] : -1;
  std::vector<int> tpos_of(P.k, -1);  // pattern vertex -> template position (this slice)
  for (int p = 0; p < L; ++p) tpos_of[(size_t)T.v[A[p]]] = p;
  for (int p = (stp.key1 >= 0 ? 2 : 1); p < L; ++p) {
    const int pv = T.v[A[p]];
    if (placed(pv)) {
      stp.eq_pos[stp.n_eq] = p;
      stp.eq_col[stp.n_eq] = col_of[(size_t)pv];
      ++stp.n_eq;
    }
  }
  for (int j = 0; j < g; ++j) {
    const int u = ord[(size_t)(pos + j)];
    if (tpos_of[(size_t)u] < 0) return false;  // not a vertex of this slice
    stp.newpos[j] = tpos_of[(size_t)u];
  }
  if (stp.key1 < 0) {  // a placed pattern neighbour of the key vertex: its image at template pos 1 is a duplicate
    const int kv = T.v[A[0]];
    for (int c = pos - 1; c >= 0 && stp.skip < 0; --c)
      if (P.adj[kv][ord[(size_t)c]]) stp.skip = c;
  }
  for (int j = 0; j < g; ++j) {
    const int u = ord[(size_t)(pos + j)];
    for (int c = 0; c < pos + j; ++c) {
      const int x = ord[(size_t)c];
      const bool in_t = tpos_of[(size_t)x] >= 0;
      const bool covered = in_t && tmpl_edge(M, tpos_of[(size_t)u], tpos_of[(size_t)x]);
      if (P.adj[u][x]) {
        if (!covered) stp.probes.push_back({j, c, 0});
      } else if (mode == DM_INDUCED) {
        stp.probes.push_back({j, c, 1});
      }
    }
  }
  return (int)stp.probes.size() <= kMaxTabProbes;
}

// Compile a placement order into kernel steps by dynamic programming over the frontier-size
// model (the rows after a prefix do not depend on the grouping): consecutive groups of 1 or 2
// vertices joined on the CSR, or (table motifs) one slice's fresh vertices joined with its
// Res(M) table.  Every pattern edge between a new vertex and an earlier one is enforced when
// the later endpoint is placed (selection pushdown, DESIGN R1).
double compile_order(const Pat &P, int mode, const std::vector<int> &ord, const std::vector<Span> &spans,
                     Plan &plan, const PlanStats &st) {
  const int k = P.k;
  plan.steps.clear();
  plan.col_pvert = ord;
  plan.pvert_col.assign(k, -1);
  for (int c = 0; c < k; ++c) plan.pvert_col[ord[(size_t)c]] = c;
  plan.first_vertex = ord[0];
  std::vector<double> rows(k + 1, 0.0);  // rows after each prefix (grouping independent)
  rows[1] = std::max(2.0, st.n);
  for (int i = 1; i < k; ++i) rows[i + 1] = step_cost(P, ord, i, 1, rows[i], false, st).rows_out;
  // table-step options: at position `start` of a table slice's fresh vertices
  std::vector<std::vector<std::pair<int, Step>>> tab_at(k + 1);
  for (const Span &sp : spans) {
    const Slice &T = plan.slices[(size_t)sp.slice];
    if (!motif_is_table(T.motif) || sp.len < 1 || sp.start < 1) continue;
    Step stp;
    if (make_table_step(P, mode, ord, plan.pvert_col, sp.start, sp.len, T, stp))
      tab_at[(size_t)sp.start].push_back({sp.slice, std::move(stp)});
  }
  const double INF = 1e300;
  std::vector<double> best(k + 1, INF);
  std::vector<int> take(k + 1, 0), take_tab(k + 1, -1);
  best[1] = 0.0;
  const bool deep = st.count_only && st.max_degree <= 4;  // row-serial ELL last step
  const double n = std::max(2.0, st.n);
  const double d1 = std::max(1.0, st.avg_degree), d2 = std::max(1.0, st.fwd_degree);
  for (int pos = 1; pos < k; ++pos) {
    if (best[pos] >= INF) continue;
    for (int g = 1; g <= kMaxNew && pos + g <= k; ++g) {
      const int i = pos + g;
      if (g > 2 && !(deep && i == k)) continue;
      const double c = best[pos] + step_cost(P, ord, pos, g, rows[pos], i == k, st).cost;
      if (c < best[i]) {
        best[i] = c;
        take[i] = g;
        take_tab[i] = -1;
      }
    }
    for (size_t t = 0; t < tab_at[(size_t)pos].size(); ++t) {
      const Step &stp = tab_at[(size_t)pos][t].second;
      const int i = pos + stp.n_new;
      const MotifDef &M = *motif_def(stp.tab_motif);
      double per_row = table_rows_estimate(M, st) / (stp.key1 >= 0 ? std::max(1.0, d1 * n) : n);
      if (stp.key1 < 0 && stp.skip >= 0) per_row *= std::max(0.0, 1.0 - 1.0 / d2);
      const double entries = rows[pos] * per_row;
      const bool last = i == k && st.count_only;
      double c = best[pos] + entries * (double)(pos + stp.n_new);
      if (!last) c += 2.0 * 4.0 * rows[i] * (double)((i + 3) & ~3);
      if (c < best[i]) {
        best[i] = c;
        take[i] = stp.n_new;
        take_tab[i] = (int)t;
      }
    }
  }
  std::vector<std::pair<int, int>> groups;  // (size, table option or -1)
  for (int i = k; i > 1; i -= take[i]) groups.push_back({take[i], take_tab[i]});
  std::reverse(groups.begin(), groups.end());
  int pos = 1;
  for (auto &gr : groups) {
    const int g = gr.first;
    if (gr.second >= 0) {
      Step stp = tab_at[(size_t)pos][(size_t)gr.second].second;
      stp.slice = tab_at[(size_t)pos][(size_t)gr.second].first;
      plan.steps.push_back(std::move(stp));
      pos += g;
      continue;
    }
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
  if (motifs & ~DM_MOTIF_ALL) return fail(DM_ERR_ARG, "unknown motif bit");
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
  plan.motifs = (motifs & DM_MOTIF_ALL) | DM_MOTIF_M2;
  for (int a = 0; a < k; ++a)
    for (int b = a + 1; b < k; ++b)
      if (P.adj[a][b]) plan.edges.push_back({a, b});

  // ------------------------------------------------------------ decomposition (§3.3)
  std::vector<const MotifDef *> order;
  for (const MotifDef *M : motif_defs())
    if ((plan.motifs & M->id) && M->nv <= k) order.push_back(M);
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
    int m[kMaxMotifV];
    const MotifDef *used = nullptr;
    for (const MotifDef *M : order)
      if (first_match(P, *M, alive, covered, in_union, plan.slices.empty(), m)) { used = M; break; }
    if (!used) return fail(DM_ERR_ARG, "internal: decomposition stalled");
    Slice s;
    s.motif = used->id;
    s.nv = used->nv;
    for (int i = 0; i < used->nv; ++i) {
      s.v[i] = m[i];
      if (in_union[m[i]]) s.c[s.nc++] = m[i];
    }
    for (int a = 0; a < used->nv; ++a)
      for (int b = a + 1; b < used->nv; ++b)
        if (tmpl_edge(*used, a, b)) covered[m[a]][m[b]] = covered[m[b]][m[a]] = 1;
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
  // Candidate execution orders: every (seed slice, first vertex) pair, then greedily either
  // the lowest-index slice that shares a vertex with the placed ones (left-deep; the paper's
  // own order is the candidate seeded by slice 0, and "the join order can also be
  // reversed") or, constraint-first, the slice with the most placed vertices (ties: the
  // lowest index) -- the most-constrained-first rule that closes the pattern's cycles as early
  // as possible and keeps tree-like stretches of large sparse patterns (Table 2) short.  The
  // cheapest order under a simple frontier-size model wins.
  const int ns = (int)plan.slices.size();
  double best_cost = -1.0;
  Plan best;
  for (int seed = 0; seed < ns; ++seed) {
    for (int fv = 0; fv < plan.slices[seed].nv; ++fv) {
     for (int cf = 0; cf < 2; ++cf) {
      std::vector<int> order{seed};
      std::vector<char> used(ns, 0), placed(k, 0);
      used[seed] = 1;
      for (int i = 0; i < plan.slices[seed].nv; ++i) placed[plan.slices[seed].v[i]] = 1;
      while ((int)order.size() < ns) {
        int pick = -1, pick_n = 0;
        for (int si = 0; si < ns; ++si) {
          if (used[si]) continue;
          int np = 0;
          for (int i = 0; i < plan.slices[si].nv; ++i) np += placed[plan.slices[si].v[i]] ? 1 : 0;
          if (np > pick_n) {
            pick = si;
            pick_n = np;
            if (!cf) break;  // lowest-index adjacent slice
          }
        }
        if (pick < 0) break;
        used[pick] = 1;
        order.push_back(pick);
        for (int i = 0; i < plan.slices[pick].nv; ++i) placed[plan.slices[pick].v[i]] = 1;
      }
      if ((int)order.size() != ns) continue;
      Plan cand = plan;
      std::vector<int> ord;
      std::vector<Span> spans;
      if (!placement_order(P, plan, order, plan.slices[seed].v[fv], ord, spans)) continue;
      cand.order = order;
      const double cost = compile_order(P, mode, ord, spans, cand, stats);
      if (best_cost < 0 || cost < best_cost - 1e-9 * best_cost) {
        best_cost = cost;
        best = std::move(cand);
      }
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
  auto mname = [](int id) { const MotifDef *d = motif_def(id); return d ? d->name : "?"; };
  std::ostringstream o;
  o << "{\"k\":" << k << ",\"mode\":\"" << (mode == DM_INDUCED ? "induced" : "mono")
    << "\",\"first_vertex\":" << first_vertex << ",\"slices\":[";
  for (size_t i = 0; i < slices.size(); ++i) {
    const Slice &s = slices[i];
    o << (i ? "," : "") << "{\"motif\":\"" << mname(s.motif) << "\",\"vertices\":[";
    for (int j = 0; j < s.nv; ++j) o << (j ? "," : "") << s.v[j];
    o << "],\"constraints\":[";
    for (int j = 0; j < s.nc; ++j) o << (j ? "," : "") << s.c[j];
    o << "]}";
  }
  o << "],\"steps\":[";
  for (size_t i = 0; i < steps.size(); ++i) {
    const Step &st = steps[i];
    o << (i ? "," : "") << "{\"in_w\":" << st.in_w;
    if (st.tab_motif) {
      o << ",\"table\":\"" << mname(st.tab_motif) << "\",\"slice\":" << st.slice << ",\"key0\":" << st.key0
        << ",\"key1\":" << st.key1 << ",\"skip\":" << st.skip << ",\"n_new\":" << st.n_new << ",\"newpos\":[";
      for (int j = 0; j < st.n_new; ++j) o << (j ? "," : "") << st.newpos[j];
      o << "],\"eq\":[";
      for (int j = 0; j < st.n_eq; ++j) o << (j ? "," : "") << "[" << st.eq_pos[j] << "," << st.eq_col[j] << "]";
      o << "],\"probes\":[";
      for (size_t j = 0; j < st.probes.size(); ++j)
        o << (j ? "," : "") << "[" << st.probes[j].j << "," << st.probes[j].col << "," << st.probes[j].neg << "]";
      o << "]}";
      continue;
    }
    o << ",\"new\":[";
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
                        int32_t vertices[DM_MAX_MOTIF_VERTICES], int32_t *n_constraints,
                        int32_t constraints[DM_MAX_MOTIF_VERTICES]) {
  dm::clear_error();
  if (!p || i < 0 || i >= (int32_t)p->p.slices.size()) return dm::fail(DM_ERR_ARG, "bad slice index");
  const dm::Slice &s = p->p.slices[(size_t)i];
  if (motif) *motif = s.motif;
  if (n_vertices) *n_vertices = s.nv;
  if (n_constraints) *n_constraints = s.nc;
  for (int j = 0; j < DM_MAX_MOTIF_VERTICES; ++j) {
    if (vertices) vertices[j] = j < s.nv ? s.v[j] : -1;
    if (constraints) constraints[j] = j < s.nc ? s.c[j] : -1;
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
