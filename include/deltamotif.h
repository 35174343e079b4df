/*
 * deltamotif.h -- C ABI of libdeltamotif.so, the B200-native (sm_100a) hot path of
 * Delta-Motif (arXiv 2508.21287, "Subgraph Isomorphism at Scale via Data-Centric
 * Parallelism").  Citations: P:n = PAPER.md line n; S:n = SPEC.md line n.
 *
 * What the library computes (§3.1): for a data graph G_d and a connected pattern G_p,
 * every injective map f : V_p -> V_d with (u,v) in E_p => (f(u),f(v)) in E_d (DM_MONO, the
 * join-and-filter pipeline of §3.2, and §3.4) or with <=> for every pattern
 * pair (DM_INDUCED, the literal reading of P:167).  It gets there the paper's way: both
 * graphs become edge tables, the pattern is decomposed into motif slices (§3.3),
 * and a table of partial embeddings is grown by equi-joins with the motif tables followed by
 * the overlapping-node filter (Alg. 1).  Each join step is one fused sm_100a kernel
 * (join + filters + single-pass compaction; an exact-offset re-run only for tiles that do not
 * fit the estimated capacity), see DESIGN.md §5.
 *
 * Conventions
 *  - Vertex ids are int32 in [0, n); counts are uint64; row offsets int64.
 *  - All functions are thread-safe.  A dm_graph is immutable after creation and may be
 *    matched concurrently from several host threads / CUDA streams.
 *  - Errors: every dm_status-returning call returns DM_OK (0) or a negative code and sets a
 *    thread-local message readable with dm_last_error().  Nothing is written to stderr.
 *    Output pointers are left untouched (NULL) on error.
 *  - Host pointers are read during the call only (copied); device memory is owned by the
 *    handle that allocated it.
 *  - No CPU fallback: every computational entry point requires a CUDA device; without one it
 *    returns DM_ERR_CUDA.
 */
#ifndef DELTAMOTIF_H
#define DELTAMOTIF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define DM_API __attribute__((visibility("default")))
#else
#define DM_API
#endif

#define DM_ABI_VERSION 4
#define DM_MAX_PATTERN 128 /* max pattern vertices k (the paper's Table 2 goes to 100) */

typedef struct dm_graph dm_graph;   /* device CSR of G_d (Res(M2), both orientations) */
typedef struct dm_result dm_result; /* count + optional canonical host table + stats   */
typedef struct dm_plan dm_plan;     /* host join program (decomposition + steps)       */
typedef struct dm_frontier dm_frontier; /* a materialized partial-embedding level (device) */

typedef enum {
  DM_OK = 0,
  DM_ERR_ARG = -1,                  /* NULL pointer, negative size, bad option value       */
  DM_ERR_VERTEX_RANGE = -2,         /* edge endpoint outside [0, n)                 */
  DM_ERR_SELF_LOOP = -3,            /* self-loop in G_d without DM_GRAPH_DROP_SELF_LOOPS, or
                                       any self-loop in G_p ("excluding self-loops") */
  DM_ERR_PATTERN_DISCONNECTED = -4, /* G_p not connected             */
  DM_ERR_OOM = -5,                  /* device or host allocation failed                    */
  DM_ERR_ROW_BUDGET = -6,           /* table mode: result larger than row_budget   */
  DM_ERR_CUDA = -7,                 /* CUDA runtime error / no device                      */
  DM_ERR_UNSUPPORTED = -8,          /* k > DM_MAX_PATTERN, ...                             */
  DM_ERR_IO = -9                    /* motif database file missing / unreadable / corrupt  */
} dm_status;

enum { DM_MONO = 0, DM_INDUCED = 1 };                      /* isomorphism variant (DESIGN Q1) */
enum { DM_OUT_COUNT = 1, DM_OUT_TABLE = 2 };               /* output bit flags                */
/* Planner motif set (bitmask).  P:180 naming: M_i = path of i vertices, "-O" = cycle.
 * M2 = edge, M3 = wedge, M3-O = triangle are joined implicitly on the CSR; the larger
 * motifs are materialized tables Res(M) built by Delta-Motif itself (Alg. 2, P:264-279:
 * dm_graph_build_motifs, or lazily by the first dm_match that asks for them) and joined by
 * table steps.  The paper's topology-aware sets: {M2, M4} heavy-hex,
 * {M2, M4-O, M6-O} square grid; M12-O for heavy-hex hexagons. */
enum {
  DM_MOTIF_M2 = 1, DM_MOTIF_M3 = 2, DM_MOTIF_M3O = 4,
  DM_MOTIF_M4 = 8, DM_MOTIF_M5 = 16, DM_MOTIF_M6 = 32, DM_MOTIF_M7 = 64, DM_MOTIF_M8 = 128,
  DM_MOTIF_M4O = 256, DM_MOTIF_M6O = 512, DM_MOTIF_M12O = 1024,
  /* Res(M3-O) materialized as the triangle-apex table keyed by directed edge (
   * P:262, Alg. 2): apex(a,b) = N(a) ∩ N(b) for every arc.  Not a decomposition motif
   * (the planner keeps M3-O implicit); when it is in the set, shared-key pair steps on arc rows
   * (diamond, 4-clique) take both new vertices' candidates from it (dm_graph_apex_table). */
  DM_MOTIF_APEX = 2048
};
#define DM_MOTIF_IMPLICIT (DM_MOTIF_M2 | DM_MOTIF_M3 | DM_MOTIF_M3O)
#define DM_MOTIF_TABLES (DM_MOTIF_M4 | DM_MOTIF_M5 | DM_MOTIF_M6 | DM_MOTIF_M7 | DM_MOTIF_M8 | \
                         DM_MOTIF_M4O | DM_MOTIF_M6O | DM_MOTIF_M12O)
#define DM_MOTIF_ALL (DM_MOTIF_IMPLICIT | DM_MOTIF_TABLES | DM_MOTIF_APEX)
#define DM_MAX_MOTIF_VERTICES 12
enum { DM_GRAPH_DROP_SELF_LOOPS = 1 };                     /* dm_graph_create flags           */
enum { DM_MATCH_PROFILE = 1 };                             /* dm_match_opts.flags: time every
                                                              kernel with CUDA events          */

typedef struct dm_match_opts_s {
  int32_t mode;        /* DM_MONO (default) or DM_INDUCED                                     */
  int32_t output;      /* DM_OUT_COUNT and/or DM_OUT_TABLE (default DM_OUT_COUNT)             */
  int32_t motifs;      /* planner motif set, bitmask of DM_MOTIF_*; M2 is always added*/
  int32_t flags;       /* DM_MATCH_PROFILE ...                                                */
  uint64_t row_budget; /* table mode: max result rows, 0 -> 2^27                      */
  uint64_t mem_budget; /* bytes for one materialized frontier chunk, 0 -> auto (free/4)       */
  int64_t seed_begin;  /* shard of the seed: the first plan vertex ranges over data vertices  */
  int64_t seed_end;    /*   [seed_begin, seed_end); seed_end < 0 means n (whole graph)         */
  void *cuda_stream;   /* cudaStream_t to launch on; NULL = legacy default stream             */
} dm_match_opts;

/* Per-match statistics (DM_MATCH_PROFILE fills the timing fields). */
#define DM_MAX_STEPS 128
typedef struct {
  int32_t num_steps;             /* executed join steps (seed included)                    */
  int32_t num_launches;          /* kernels launched by this dm_match call                 */
  int32_t num_chunks;            /* frontier chunks processed (>= num_steps when chunked)  */
  int32_t elem_bytes;            /* bytes per stored vertex id in frontier levels (4 or 2)  */
  uint64_t rows_in[DM_MAX_STEPS];    /* |F_i| summed over chunks                           */
  uint64_t rows_out[DM_MAX_STEPS];   /* |F_{i+1}| (survivors)                              */
  uint64_t candidates[DM_MAX_STEPS]; /* C_i: join matches before filters (first new vertex,
                                        plus second-level matches for 2-vertex steps)      */
  uint64_t probes[DM_MAX_STEPS];     /* Q_i: closing-edge / non-edge probe targets         */
  int32_t width_in[DM_MAX_STEPS];    /* w_i                                                */
  int32_t width_out[DM_MAX_STEPS];   /* w_{i+1}                                            */
  double bytes_model[DM_MAX_STEPS];  /* SURVEY §8(d) algorithmic bytes of step i, as written:
                                        4 B per id (seed's 1-column input included):
                                        4 w_i |F_i| + 8 |F_i| + 4 C_i + 4 Q_i + 4 w_{i+1} |F_{i+1}|
                                        (no write for the count-only last step)              */
  double bytes_stored[DM_MAX_STEPS]; /* the same with the STORED id width (2 B for 16-bit levels)
                                        and no read for the implicit seed                     */
  double ms_count[DM_MAX_STEPS];     /* device ms in count-pass kernels of step i          */
  double ms_write[DM_MAX_STEPS];     /* device ms in write-pass kernels of step i          */
  double ms_other;                   /* scans, canonical sort, copies                      */
  double ms_total;                   /* device ms from first to last launch                */
  int32_t pipelined;                 /* 1: every step was enqueued without an intermediate host
                                        synchronisation (repeated count query whose level
                                        capacities came from the previous identical run)    */
  int32_t reserved;
} dm_match_stats;

/* Fill *opt with defaults (DM_MONO, DM_OUT_COUNT, all motifs, whole graph, NULL stream). */
DM_API void dm_match_opts_init(dm_match_opts *opt);

/* ABI version (DM_ABI_VERSION) -- lets bindings detect a stale library. */
DM_API int32_t dm_abi_version(void);

/*
 * dm_graph_create -- build Res(M2) = E_d \ E_self in both orientations (Alg. 2
 * l.2) as a device CSR: int64 off[n+1], int32 adj[2m'] with every adjacency list sorted
 * ascending; duplicates and reversed pairs collapse.
 *   n      number of data vertices (>= 0)
 *   edges  HOST array int32[m][2] of undirected edges (row-major pairs); may be NULL if m == 0
 *   flags  DM_GRAPH_DROP_SELF_LOOPS: drop (u,u) instead of failing with DM_ERR_SELF_LOOP
 *   device CUDA device ordinal the CSR lives on
 *   out    receives the handle (free with dm_graph_destroy)
 * Errors: DM_ERR_ARG, DM_ERR_VERTEX_RANGE, DM_ERR_SELF_LOOP, DM_ERR_OOM, DM_ERR_CUDA.
 * The build runs on device (sort, dedup, degree scan) and is the "data preparation" phase
 * the paper times separately.  All device buffers of a graph (CSR, motif tables,
 * apex table) come from the device's stream-ordered memory pool, whose release threshold the
 * library raises so create / destroy cycles reuse memory.  dm_graph_destroy must not be called
 * while work on g is in flight (every dm_* call returns after its stream work completed); it
 * returns the buffers to the pool without a device-wide synchronisation.
 */
DM_API dm_status dm_graph_create(int32_t n, const int32_t *edges, int64_t m, int32_t flags,
                          int32_t device, dm_graph **out);
DM_API void dm_graph_destroy(dm_graph *g);
DM_API int32_t dm_graph_num_vertices(const dm_graph *g);
DM_API int64_t dm_graph_num_arcs(const dm_graph *g);  /* 2 |E_d| after dedup / self-loop removal */
DM_API int32_t dm_graph_max_degree(const dm_graph *g);
DM_API int32_t dm_graph_device(const dm_graph *g);
/* Statistics the planner's cost model uses: sum of squared degrees and the triangle-closure
 * probability sampled on 4,096 arcs at creation (pass them to dm_plan_create_ex to reproduce
 * the plan dm_match builds). */
DM_API dm_status dm_graph_stats(const dm_graph *g, double *sum_d2, double *closure);
/*
 * Motif database (Alg. 2 BuildDatabase): Res(M) for every table motif in `motifs`
 * (DM_MOTIF_M4 ... DM_MOTIF_M12O), each computed by Delta-Motif itself (a table-mode match of the
 * motif template over {M2, M3, M3-O}), stored on g's device in canonical order and indexed by the
 * CSR arc of the first two template positions.  Already built tables are kept; the build is the
 * paper's data-preparation phase (GPU vs GPU*).  dm_match builds what it needs on first
 * use; thread-safe.  opt: stream and row_budget (max rows per table, default 2^28); may be NULL.
 * Errors: DM_ERR_ARG (unknown motif bit), DM_ERR_ROW_BUDGET, DM_ERR_OOM, DM_ERR_CUDA.
 *   dm_graph_motif_rows: |Res(M)| of a built table, -1 if not built.
 *   dm_graph_motif_build_ms: host wall time the build took, -1 if not built.
 *   dm_graph_motif_table: copy Res(M) to HOST rows_out[rows][L] (template position order, rows
 *       ascending lexicographic) and/or the index toff_out[num_arcs + 1] (either may be NULL).
 */
DM_API dm_status dm_graph_build_motifs(dm_graph *g, int32_t motifs, const dm_match_opts *opt);
DM_API int64_t dm_graph_motif_rows(const dm_graph *g, int32_t motif);
DM_API double dm_graph_motif_build_ms(const dm_graph *g, int32_t motif);
DM_API dm_status dm_graph_motif_table(const dm_graph *g, int32_t motif, int32_t *rows_out, int64_t *toff_out);
/*
 * Triangle-apex table (Res(M3-O) of P:262 keyed by directed edge, built once
 * per graph like the Alg. 2 tables): dm_graph_build_motifs(g, DM_MOTIF_APEX, opt)
 * builds it on the device (two-pass: per-arc |N(a) ∩ N(b)|, exclusive scan, write).
 *   dm_graph_apex_entries: total entries (= 6 x #triangles = tr(A^3)), -1 if not built.
 *   dm_graph_apex_build_ms: host wall time of the build, -1 if not built.
 *   dm_graph_apex_table: copy to HOST toff_out[num_arcs + 1] (int64 offsets: arc e = (a, adj[e])
 *       owns entries [toff[e], toff[e+1])) and/or apex_out[entries]: each entry is the CSR arc
 *       index of (a, c) for c in N(a) ∩ N(b), ascending (vertex c = adj[entry]).  Either may be NULL.
 * Errors: DM_ERR_ARG (not built), DM_ERR_CUDA; the build: DM_ERR_UNSUPPORTED (>= 2^31 arcs),
 * DM_ERR_OOM, DM_ERR_CUDA.
 */
DM_API int64_t dm_graph_apex_entries(const dm_graph *g);
DM_API double dm_graph_apex_build_ms(const dm_graph *g);
DM_API dm_status dm_graph_apex_table(const dm_graph *g, int64_t *toff_out, int32_t *apex_out);
/*
 * Motif database persistence (SPEC save_database / load_database; the "performed
 * once, cached, and reused" preparation of P:336-338): dm_graph_save_motifs writes every built
 * Res(M) table of g, and the triangle-apex table if built, to one file (atomically: path.tmp then
 * rename); dm_graph_load_motifs adds the file's tables to g without rebuilding them.  The file is bound to the graph by a fingerprint
 * (FNV-1a over n and the sorted, deduplicated CSR = an order-independent hash of the edge set);
 * every table carries a checksum.
 * Errors: DM_ERR_IO (cannot open / write, bad magic or version, truncated file, checksum
 * mismatch), DM_ERR_ARG (fingerprint mismatch: the file was built for another graph), DM_ERR_OOM,
 * DM_ERR_CUDA.  Tables already resident in g are kept.
 */
DM_API dm_status dm_graph_save_motifs(const dm_graph *g, const char *path);
DM_API dm_status dm_graph_load_motifs(dm_graph *g, const char *path);
/* Device pointers of the CSR (owned by g, valid until dm_graph_destroy). */
DM_API dm_status dm_graph_device_csr(const dm_graph *g, const int64_t **d_off, const int32_t **d_adj);
/* Copy the CSR to host buffers off_out[n+1] and adj_out[num_arcs] (either may be NULL). */
DM_API dm_status dm_graph_copy_csr(const dm_graph *g, int64_t *off_out, int32_t *adj_out);

/*
 * dm_match -- all embeddings of the pattern (k vertices, pm edges p_edges[pm][2] on HOST) in
 * g (Alg. 1).  opt may be NULL (defaults).
 *   output & DM_OUT_COUNT: dm_result_count() = number of labelled mappings f (DESIGN Q2).
 *   output & DM_OUT_TABLE: dm_result_rows() = host int32[count][k], row-major, column j =
 *       f(j), rows in ascending lexicographic order.
 * Only mappings with f(first plan vertex) in [seed_begin, seed_end) are produced, so disjoint
 * seed ranges partition the result (multi-GPU sharding, DESIGN "Multi-GPU").  Use
 * dm_plan_create + dm_plan_first_vertex to learn which pattern vertex that is.
 * Errors: DM_ERR_ARG, DM_ERR_VERTEX_RANGE / DM_ERR_SELF_LOOP (pattern), DM_ERR_PATTERN_
 * DISCONNECTED, DM_ERR_ROW_BUDGET (table mode only; count mode chunks instead), DM_ERR_OOM,
 * DM_ERR_CUDA, DM_ERR_UNSUPPORTED (k > DM_MAX_PATTERN).
 * The call is synchronous with respect to opt->cuda_stream (it reads back per-step sizes).
 */
DM_API dm_status dm_match(const dm_graph *g, int32_t k, const int32_t *p_edges, int64_t pm,
                   const dm_match_opts *opt, dm_result **out);
DM_API uint64_t dm_result_count(const dm_result *r);
DM_API int32_t dm_result_width(const dm_result *r);          /* = k                                 */
DM_API const int32_t *dm_result_rows(const dm_result *r);    /* host table or NULL (count only)     */
DM_API dm_status dm_result_stats(const dm_result *r, dm_match_stats *out);
DM_API void dm_result_free(dm_result *r);

/*
 * Step-level entry points for multi-GPU frontier rebalancing (C2 all-to-all).
 * The plan dm_match builds is deterministic for (g, pattern, opt), so a level produced by
 * dm_match_prefix can be exchanged between ranks and finished by dm_match_resume with the same
 * arguments.
 *   dm_match_prefix: run join steps [0, upto_step) for the seed range in opt and return level
 *       `upto_step` (1 <= upto_step < num_steps) as device rows: int32 [rows][stride],
 *       stride = dm_frontier_stride (16-byte padded, padding -1), columns in plan (match) order,
 *       plus a per-row uint64 work estimate of the next step (anchor degree ^ new vertices).
 *       The dm_frontier owns both device buffers (dm_frontier_free).
 *   dm_match_resume: finish the plan from level `from_step` given device rows in that layout
 *       (d_rows is read only; caller keeps ownership); result as dm_match.  Disjoint row sets
 *       give disjoint results, so the per-rank counts / tables of a repartitioned level sum up.
 * Errors: DM_ERR_ARG (step out of range, NULL rows with rows > 0) plus dm_match's.
 */
DM_API dm_status dm_match_prefix(const dm_graph *g, int32_t k, const int32_t *p_edges, int64_t pm,
                                 const dm_match_opts *opt, int32_t upto_step, dm_frontier **out);
DM_API int64_t dm_frontier_rows(const dm_frontier *f);
DM_API int32_t dm_frontier_width(const dm_frontier *f);
DM_API int32_t dm_frontier_stride(const dm_frontier *f);
DM_API const int32_t *dm_frontier_device_rows(const dm_frontier *f);
DM_API const uint64_t *dm_frontier_device_work(const dm_frontier *f);
DM_API uint64_t dm_frontier_work_total(const dm_frontier *f);   /* sum of the work estimates     */
/* Frees the frontier's buffers stream-ordered on the stream it was produced on (no device-wide
 * synchronisation); that stream must still exist (NULL = legacy default stream). */
DM_API void dm_frontier_free(dm_frontier *f);
DM_API dm_status dm_match_resume(const dm_graph *g, int32_t k, const int32_t *p_edges, int64_t pm,
                                 const dm_match_opts *opt, int32_t from_step, const int32_t *d_rows,
                                 int64_t rows, dm_result **out);

/*
 * Step-level entry points: the join program of Alg. 1 executed one
 * step at a time on device rows, for drivers that move levels between ranks (§8(e)).
 *   dm_plan_create_for: the plan dm_match would execute for (g, pattern, opt): the §3.3
 *       decomposition plus the join order chosen with g's statistics; count_only planning when
 *       !(opt->output & DM_OUT_TABLE).  Free with dm_plan_destroy.
 *   dm_plan_width / dm_plan_stride: columns / int32 words per row of level `level` (the input of
 *       step `level`; level num_steps is the final level, width k).  Level rows are row-major
 *       int32 [rows][stride], stride = round_up(width, 4), padding -1, columns in plan (match)
 *       order (dm_plan_column_vertex maps a column to its pattern vertex).
 *   dm_plan_seed_work: HOST work_prefix[0..seed_end-seed_begin] = exclusive prefix of the seed
 *       step's estimated work (deg(v)^n_new + 1) over the seed vertices v in [seed_begin,
 *       seed_end) (seed_end < 0 means n).  dm_plan_seed_cuts: HOST cuts[0..parts] = equal-work
 *       cut points of [0, n) over that prefix (rank r's seed range is [cuts[r], cuts[r+1])).
 *   dm_plan_seed = dm_plan_step(step 0): the first slice's table (Alg. 1 l.2/l.6, reading Q3)
 *       for opt's seed range, as a level.
 *   dm_plan_step: run step `step` (0 <= step < num_steps) on the device rows d_in [in_rows]
 *       of level `step` (step 0: d_in must be NULL, the seed range of opt is used).  Returns
 *       level step+1 in *out_level (owned by the caller, dm_frontier_free; the final level's
 *       work pointer is NULL) and its row count in *count when count != NULL.  For the last
 *       step out_level may be NULL: then only *count (the count-only last step) is produced.
 *   dm_plan_finish_table: final-level rows (plan order, stride round_up(k,4)) -> d_canon_out
 *       [rows][k] in pattern-vertex column order and ascending lexicographic row order (a9).
 *   dm_plan_run: dm_match with this plan.
 * All run on opt->cuda_stream and return after the stream work they issued has completed.
 * Errors: DM_ERR_ARG (NULL / ranges / a plan this graph cannot execute) plus dm_match's.
 */
DM_API dm_status dm_plan_create_for(const dm_graph *g, int32_t k, const int32_t *p_edges, int64_t pm,
                                    const dm_match_opts *opt, dm_plan **out);
DM_API int32_t dm_plan_width(const dm_plan *p, int32_t level);
DM_API int32_t dm_plan_stride(const dm_plan *p, int32_t level);
DM_API int32_t dm_plan_column_vertex(const dm_plan *p, int32_t column);
DM_API dm_status dm_plan_seed_work(const dm_graph *g, const dm_plan *p, int64_t seed_begin,
                                   int64_t seed_end, uint64_t *work_prefix);
DM_API dm_status dm_plan_seed_cuts(const dm_graph *g, const dm_plan *p, int32_t parts, int64_t *cuts);
DM_API dm_status dm_plan_seed(const dm_graph *g, const dm_plan *p, const dm_match_opts *opt,
                              dm_frontier **out);
DM_API dm_status dm_plan_step(const dm_graph *g, const dm_plan *p, const dm_match_opts *opt,
                              int32_t step, const int32_t *d_in, int64_t in_rows,
                              dm_frontier **out_level, uint64_t *count);
DM_API dm_status dm_plan_finish_table(const dm_graph *g, const dm_plan *p, const dm_match_opts *opt,
                                      const int32_t *d_rows, int64_t rows, int32_t *d_canon_out);
DM_API dm_status dm_plan_run(const dm_graph *g, const dm_plan *p, const dm_match_opts *opt,
                             dm_result **out);

/*
 * Multi-GPU exchange helpers (collectives C2 and C4).  Every row of a level is an
 * independent candidate (§4.1), so any row partition is valid.  Device buffers on one
 * device (the device of d_rows); stream-ordered on `stream` (cudaStream_t, NULL = legacy);
 * the per-part row counts are written to the HOST array counts[parts] (the call synchronises).
 *   dm_rows_partition_by_work: d_out = the n rows (stride int32 words each) grouped by
 *       destination part, stable within a part; a row's part is floor(parts * (work_base + the
 *       exclusive prefix of d_work at that row) / work_total) -- its position in the GLOBAL
 *       work order of all ranks (work_base = total work of lower ranks), i.e. an equal-work cut.
 *   dm_rows_partition_by_key: the same with part = #{splitters <= row[col]} (splitters: HOST
 *       int32[parts-1], ascending): the range partition of a table by one column.
 *   dm_table_sort: rows of d_rows [n][k] (packed) into ascending lexicographic order, in place
 *       (ids in [0, n_vertices)).
 * d_out must hold n * stride int32 and must not alias d_rows.
 * Errors: DM_ERR_ARG (bad sizes, not device memory, unsorted splitters), DM_ERR_OOM, DM_ERR_CUDA.
 */
DM_API dm_status dm_rows_partition_by_work(const int32_t *d_rows, const uint64_t *d_work, int64_t n,
                                           int32_t stride, uint64_t work_base, uint64_t work_total,
                                           int32_t parts, int32_t *d_out, int64_t *counts, void *stream);
DM_API dm_status dm_rows_partition_by_key(const int32_t *d_rows, int64_t n, int32_t stride, int32_t col,
                                          const int32_t *splitters, int32_t parts, int32_t *d_out,
                                          int64_t *counts, void *stream);
DM_API dm_status dm_table_sort(int32_t *d_rows, int64_t n, int32_t k, int32_t n_vertices, void *stream);

/*
 * dm_score_layouts -- layout generation + scoring + ranking (quantum layout selection, PAPER.md
 * §6.5; SPEC layout-scoring S:472-508): every embedding f of the pattern in g (as
 * dm_match in table mode with opt's mode / motif set), scored
 *     score(f) = prod_{v in V_p} node_fid[f(v)] * prod_{(a,b) in p_edges} edge_fid(f(a), f(b))
 * in float64 (vertex factors in pattern-vertex order, then the edges in the given order), and
 * the top_k rows by descending score, ties in ascending lexicographic row order.
 *   node_fid   HOST double[n], each in (0, 1]
 *   fid_edges  HOST int32[fm][2] undirected data edges, fid_vals HOST double[fm] in (0, 1]; every
 *              data edge needs a fidelity (duplicates: the last one wins)
 *   rows_out   HOST int32[top_k][k], scores_out HOST double[top_k]; *n_out = min(top_k, count),
 *              *count_out (may be NULL) = number of layouts
 * Errors: DM_ERR_ARG (top_k <= 0, fidelity outside (0, 1], fidelity for a non-edge, a data edge
 * without fidelity), DM_ERR_VERTEX_RANGE, plus dm_match's.  Synchronous on opt->cuda_stream.
 */
DM_API dm_status dm_score_layouts(const dm_graph *g, int32_t k, const int32_t *p_edges, int64_t pm,
                                  const double *node_fid, const int32_t *fid_edges, const double *fid_vals,
                                  int64_t fm, const dm_match_opts *opt, int64_t top_k, int32_t *rows_out,
                                  double *scores_out, int64_t *n_out, uint64_t *count_out);

/* Thread-local message of the last failing call on this thread ("" if none). */
DM_API const char *dm_last_error(void);

/*
 * Host planner (no device needed).  dm_plan_create decomposes the pattern into motif slices
 * exactly as §3.3 describes (motifs tried in descending size, first single match
 * found by a backtracking matcher on the reduced pattern, boundary nodes kept, non-boundary
 * nodes removed, shared vertices recorded as join constraints) and compiles the join program.
 * motifs: DM_MOTIF_* bitmask (M2 always included); mode: DM_MONO / DM_INDUCED.
 */
DM_API dm_status dm_plan_create(int32_t k, const int32_t *p_edges, int64_t pm, int32_t motifs,
                         int32_t mode, dm_plan **out);
/* Same, with the data-graph statistics the join-order cost model uses (dm_match takes them
 * from the dm_graph): n vertices, arcs (= 2|E|), sum of squared degrees, sampled triangle
 * closure probability (0 for triangle-free graphs), max degree (<= 4 allows a 3-4 vertex
 * count-only last step), count_only (1: last level is counted, not materialized).
 * dm_plan_create uses n=1e4, arcs=3e4, sum_d2=9e4, closure=0, max degree 2^30, count_only=0. */
DM_API dm_status dm_plan_create_ex(int32_t k, const int32_t *p_edges, int64_t pm, int32_t motifs,
                                   int32_t mode, double n, double arcs, double sum_d2,
                                   double closure, int32_t max_degree, int32_t count_only,
                                   dm_plan **out);
DM_API void dm_plan_destroy(dm_plan *p);
DM_API int32_t dm_plan_num_slices(const dm_plan *p);
/* Slice i: motif id (DM_MOTIF_*), its pattern vertices (template position order, n_vertices <=
 * DM_MAX_MOTIF_VERTICES) and the join constraints = vertices shared with the union of earlier
 * slices (decomposition order). */
DM_API dm_status dm_plan_slice(const dm_plan *p, int32_t i, int32_t *motif, int32_t *n_vertices,
                               int32_t vertices[DM_MAX_MOTIF_VERTICES], int32_t *n_constraints,
                               int32_t constraints[DM_MAX_MOTIF_VERTICES]);
DM_API int32_t dm_plan_num_steps(const dm_plan *p);          /* executed kernel steps             */
DM_API int32_t dm_plan_first_vertex(const dm_plan *p);       /* pattern vertex sharded by seed    */
/* Human-readable JSON description of slices and steps (for tests / debugging).  Writes at
 * most len bytes including the NUL; returns the full length needed. */
DM_API int64_t dm_plan_describe(const dm_plan *p, char *buf, int64_t len);

#ifdef __cplusplus
}
#endif
#endif /* DELTAMOTIF_H */
