// dm_internal.h -- internal declarations of libdeltamotif.so (not part of the C ABI).
// Citations: P:n = PAPER.md line n, S:n = SPEC.md line n (see include/deltamotif.h).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "deltamotif.h"

namespace dm {

// ----------------------------------------------------------------------------- errors
dm_status fail(dm_status code, const std::string &msg);  // sets the thread-local message
void clear_error();

// ---------------------------------------------------------------------------- planner
// Motif templates (P:180 naming: M_i = path of i vertices, "-O" = cycle).  M2, M3 and M3-O are
// joined implicitly on the CSR (Res(M3) = Res(M2) ⋈ Res(M2)); the larger ones are
// materialized tables Res(M) built by Delta-Motif itself (Alg. 2) and joined by
// table steps.
constexpr int kMaxMotifV = DM_MAX_MOTIF_VERTICES;
struct MotifDef {
  int id;      // DM_MOTIF_* bit
  int nv;      // template vertices 0..nv-1
  bool cycle;  // edges i-(i+1) (+ (nv-1)-0 for a cycle)
  const char *name;
};
const MotifDef *motif_def(int id);           // nullptr for an unknown bit
const std::vector<const MotifDef *> &motif_defs();  // every motif, decomposition order
inline bool motif_is_table(int id) { return id >= DM_MOTIF_M4; }

// One motif slice S_i of the decomposition: motif template, the pattern
// vertices it is matched onto (template position order) and the join constraints (shared
// vertices).
struct Slice {
  int motif = DM_MOTIF_M2;
  int nv = 0;
  int v[kMaxMotifV];
  int nc = 0;
  int c[kMaxMotifV];
};

// A vertex placed by an executed step: the join key columns it must be adjacent to (the
// equi-join constraints with Res(M2) / the closing-edge probes) and, in induced
// mode, the columns it must NOT be adjacent to.  Column indices refer to the row being built
// (input columns 0..in_w-1, then the step's new vertices in order).
struct StepVertex {
  int pvert = -1;
  int n_nbr = 0;
  int nbr[DM_MAX_PATTERN];
  int n_non = 0;
  int non[DM_MAX_PATTERN];
};

// One executed join step.  CSR step (tab_motif == 0): 1 or 2 new vertices (up to kMaxNew for a
// count-only last step on a max-degree-4 graph, where the tail kernel enumerates them without
// materializing the levels).  Table step (tab_motif != 0): the fresh vertices of one slice S
// joined with Res(M_S) (Alg. 1 l.6 InnerJoin): the row's image of the pattern vertex on
// template position 0 (and 1, key1 >= 0) selects the index range of the table; further bound
// template positions are equality filters (the remaining join constraints);
// pattern edges the motif does not cover are closing-edge probes (and non-edges in induced
// mode); the all-distinct filter covers the new vertices.
constexpr int kMaxNew = 4;
constexpr int kMaxTabProbes = 256;
struct TabProbe {
  int j;    // new vertex (0-based within the step)
  int col;  // row column it is probed against (may be a new column in_w + j' with j' < j)
  int neg;  // 1: must NOT be adjacent (induced non-edge)
};
struct Step {
  int slice = -1;
  int in_w = 0;
  int n_new = 0;
  StepVertex nv[kMaxNew];
  // table step
  int tab_motif = 0;
  int key0 = -1, key1 = -1;      // row columns bound to template positions 0 and 1 (key1 < 0: one key)
  int skip = -1;                 // one-key step: a column whose image, as template position 1, is a
                                 // known duplicate (a pattern neighbour of the key): skipped range
  int newpos[kMaxMotifV];        // template position of new column in_w + j
  int n_eq = 0;
  int eq_pos[kMaxMotifV], eq_col[kMaxMotifV];  // template position eq_pos[i] must equal row[eq_col[i]]
  std::vector<TabProbe> probes;
};

// Data-graph statistics for the join-order cost model (defaults: a sparse lattice).
struct PlanStats {
  double tab_rows[32] = {};  // |Res(M)| of built motif tables, by DM_MOTIF_* bit index (0 = estimate)
  double n = 10000.0;
  double avg_degree = 3.0;   // arcs / n: expansion from the implicit vertex table
  double fwd_degree = 3.0;   // sum d^2 / arcs: degree of a vertex reached along an edge
  double closure = 0.0;      // P[extra join key holds] beyond the random-pair probability
  bool count_only = false;   // last level is counted, not materialized
  int max_degree = 1 << 30;  // deep (3-4 vertex) last steps need max degree <= 4
};

struct Plan {
  int k = 0;
  int mode = DM_MONO;
  int motifs = DM_MOTIF_M2;
  std::vector<std::pair<int, int>> edges;  // deduplicated pattern edges (a < b)
  std::vector<Slice> slices;
  std::vector<int> order;      // slice execution order (left-deep)
  std::vector<Step> steps;
  std::vector<int> col_pvert;  // column -> pattern vertex (match order)
  std::vector<int> pvert_col;  // pattern vertex -> column
  int first_vertex = 0;        // pattern vertex of column 0 (the sharded seed vertex)
  std::string describe() const;
};

// Validates the pattern and builds the plan.  Returns DM_OK or an error (message set).
dm_status build_plan(int32_t k, const int32_t *p_edges, int64_t pm, int32_t motifs, int32_t mode,
                     Plan &out, const PlanStats &stats = PlanStats());

}  // namespace dm

struct dm_plan {
  dm::Plan p;
};
