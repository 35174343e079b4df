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
// One motif slice S_i of the decomposition: motif template, the pattern
// vertices it is matched onto (slot order) and the join constraints (shared vertices).
struct Slice {
  int motif = DM_MOTIF_M2;  // DM_MOTIF_M2 / DM_MOTIF_M3 / DM_MOTIF_M3O
  int nv = 0;
  int v[3] = {-1, -1, -1};
  int nc = 0;
  int c[3] = {-1, -1, -1};
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

// One executed join step: 1 or 2 new vertices (up to kMaxNew for a count-only last step on a
// max-degree-4 graph, where the tail kernel enumerates them without materializing the levels).
constexpr int kMaxNew = 4;
struct Step {
  int slice = -1;
  int in_w = 0;
  int n_new = 0;
  StepVertex nv[kMaxNew];
};

// Data-graph statistics for the join-order cost model (defaults: a sparse lattice).
struct PlanStats {
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
