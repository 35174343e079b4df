/*
 * dm_oracle.c -- TEST INFRASTRUCTURE ONLY.  The plain, slow, obviously-correct CPU oracle for
 * Delta-Motif's hot path.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header or table with the
 * CUDA path (paper_2508_21287_b200/csrc); both sides only read the same generated edge lists.
 *
 * What it computes (§3.1 l.167, "Subgraph Isomorphism"): every injective map
 * f : V_p -> V_d such that (u,v) in E_p  =>  (f(u),f(v)) in E_d   (monomorphism, the reading
 * the join-and-filter pipeline of §3.2 l.237 / §3.4 l.262 reaches; reading Q1), or
 * (u,v) in E_p <=> (f(u),f(v)) in E_d for all pattern pairs (induced = the literal l.167
 * definition).  The result is the set of labelled mappings (Q2): row j = f(j).
 *
 * Algorithm (SURVEY.md §8(c) "Oracle algorithm"): plain depth-first backtracking over a
 * connectivity-first pattern order; no joins, no motif tables, no frontier.
 *   1. data graph: validate ids, drop (or reject) self-loops (§3.4 l.260 "excluding
 *      self-loops"), store both orientations (l.262), sort, dedup -> sorted adjacency arrays.
 *   2. order pi: start at the max-degree pattern vertex (ties: lowest id); then repeatedly the
 *      unmatched vertex with most matched neighbours (ties: higher degree, then lower id).
 *   3. for each root s (threads pull roots from an atomic counter): f(pi_0)=s; at depth i the
 *      candidates for pi_i are N(f(anchor)) for the matched neighbour whose image has the
 *      smallest degree; reject used vertices; reject c if c not in N(f(q)) for another matched
 *      neighbour q; in induced mode also reject c if c in N(f(q)) for a matched NON-neighbour q.
 *   4. at depth k emit (f(0..k-1)) or count it.  Table rows are sorted lexicographically.
 *
 * Error codes: 0 ok, -1 bad argument, -2 vertex out of range, -3 self-loop (when rejected),
 * -4 pattern disconnected, -5 out of memory.
 */
#define _GNU_SOURCE
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define OR_OK 0
#define OR_ARG (-1)
#define OR_RANGE (-2)
#define OR_SELF (-3)
#define OR_DISC (-4)
#define OR_OOM (-5)

typedef struct {
  int64_t n;
  int64_t *off;  /* n+1 */
  int32_t *adj;  /* sorted, both orientations */
} og_graph;

static int cmp_u64(const void *a, const void *b) {
  uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
  return (x > y) - (x < y);
}

static int build_graph(int64_t n, const int32_t *edges, int64_t m, int drop_self, og_graph *g) {
  uint64_t *keys = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(2 * m + 1));
  if (!keys) return OR_OOM;
  int64_t t = 0;
  for (int64_t i = 0; i < m; ++i) {
    int64_t a = edges[2 * i], b = edges[2 * i + 1];
    if (a < 0 || b < 0 || a >= n || b >= n) { free(keys); return OR_RANGE; }
    if (a == b) {
      if (drop_self) continue;
      free(keys);
      return OR_SELF;
    }
    keys[t++] = ((uint64_t)a << 32) | (uint64_t)b;
    keys[t++] = ((uint64_t)b << 32) | (uint64_t)a;
  }
  qsort(keys, (size_t)t, sizeof(uint64_t), cmp_u64);
  int64_t u = 0;
  for (int64_t i = 0; i < t; ++i)
    if (i == 0 || keys[i] != keys[i - 1]) keys[u++] = keys[i];
  g->n = n;
  g->off = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
  g->adj = (int32_t *)malloc(sizeof(int32_t) * (size_t)(u + 1));
  if (!g->off || !g->adj) { free(keys); return OR_OOM; }
  for (int64_t i = 0; i < u; ++i) {
    g->off[(keys[i] >> 32) + 1]++;
    g->adj[i] = (int32_t)(keys[i] & 0xffffffffu);
  }
  for (int64_t v = 0; v < n; ++v) g->off[v + 1] += g->off[v];
  free(keys);
  return OR_OK;
}

static void free_graph(og_graph *g) {
  free(g->off);
  free(g->adj);
}

static int has_edge(const og_graph *g, int32_t a, int32_t b) {
  int64_t lo = g->off[a], hi = g->off[a + 1];
  while (lo < hi) {
    int64_t mid = lo + (hi - lo) / 2;
    if (g->adj[mid] < b) lo = mid + 1;
    else hi = mid;
  }
  return lo < g->off[a + 1] && g->adj[lo] == b;
}

typedef struct {
  const og_graph *g;
  int32_t k;
  const uint8_t *padj;  /* k*k pattern adjacency */
  const int32_t *order; /* pi */
  int induced;
  int want_table;
  int64_t root_begin, root_end;
  int64_t next_root; /* atomic */
} og_job;

typedef struct {
  og_job *job;
  uint64_t count;
  int32_t *rows;
  int64_t nrows, cap;
  int err;
} og_worker;

static int emit(og_worker *w, const int32_t *f, int32_t k) {
  if (w->nrows == w->cap) {
    int64_t nc = w->cap ? 2 * w->cap : 1024;
    int32_t *nr = (int32_t *)realloc(w->rows, sizeof(int32_t) * (size_t)(nc * k));
    if (!nr) return OR_OOM;
    w->rows = nr;
    w->cap = nc;
  }
  memcpy(w->rows + w->nrows * k, f, sizeof(int32_t) * (size_t)k);
  w->nrows++;
  return OR_OK;
}

/* depth-first extension of the partial map f (indexed by pattern vertex) */
static void extend(og_worker *w, int32_t depth, int32_t *f, uint8_t *used) {
  const og_job *J = w->job;
  const og_graph *g = J->g;
  const int32_t k = J->k;
  if (w->err) return;
  if (depth == k) {
    w->count++;
    if (J->want_table && emit(w, f, k) != OR_OK) w->err = OR_OOM;
    return;
  }
  const int32_t v = J->order[depth];
  /* anchor: matched pattern neighbour of v whose image has the smallest degree */
  int32_t anchor = -1;
  int64_t best = -1;
  for (int32_t i = 0; i < depth; ++i) {
    int32_t q = J->order[i];
    if (!J->padj[v * k + q]) continue;
    int64_t d = g->off[f[q] + 1] - g->off[f[q]];
    if (anchor < 0 || d < best) { anchor = q; best = d; }
  }
  /* connectivity-first order guarantees an anchor for depth >= 1 */
  const int32_t a = f[anchor];
  for (int64_t e = g->off[a]; e < g->off[a + 1]; ++e) {
    const int32_t c = g->adj[e];
    if (used[c]) continue;                       /* injectivity */
    int ok = 1;
    for (int32_t i = 0; i < depth && ok; ++i) {
      int32_t q = J->order[i];
      if (q == anchor) continue;
      if (J->padj[v * k + q]) {
        if (!has_edge(g, f[q], c)) ok = 0;       /* pattern edge must map to a data edge */
      } else if (J->induced) {
        if (has_edge(g, f[q], c)) ok = 0;        /* induced: non-edge must map to non-edge */
      }
    }
    if (!ok) continue;
    f[v] = c;
    used[c] = 1;
    extend(w, depth + 1, f, used);
    used[c] = 0;
  }
}

static void *worker_main(void *arg) {
  og_worker *w = (og_worker *)arg;
  og_job *J = w->job;
  int32_t *f = (int32_t *)malloc(sizeof(int32_t) * (size_t)J->k);
  uint8_t *used = (uint8_t *)calloc((size_t)J->g->n + 1, 1);
  if (!f || !used) { w->err = OR_OOM; free(f); free(used); return NULL; }
  const int32_t root = J->order[0];
  for (;;) {
    int64_t s = __atomic_fetch_add(&J->next_root, 1, __ATOMIC_RELAXED);
    if (s >= J->root_end || w->err) break;
    f[root] = (int32_t)s;
    used[s] = 1;
    extend(w, 1, f, used);
    used[s] = 0;
  }
  free(f);
  free(used);
  return NULL;
}

static int cmp_row(const void *a, const void *b, void *karg) {
  const int32_t *x = (const int32_t *)a, *y = (const int32_t *)b;
  const int32_t kk = *(const int32_t *)karg;
  for (int32_t i = 0; i < kk; ++i)
    if (x[i] != y[i]) return (x[i] > y[i]) - (x[i] < y[i]);
  return 0;
}

/* Pattern order pi. */
static void pattern_order(int32_t k, const uint8_t *padj, int32_t *order) {
  int32_t *deg = (int32_t *)calloc((size_t)k, sizeof(int32_t));
  uint8_t *done = (uint8_t *)calloc((size_t)k, 1);
  for (int32_t i = 0; i < k; ++i)
    for (int32_t j = 0; j < k; ++j) deg[i] += padj[i * k + j];
  for (int32_t d = 0; d < k; ++d) {
    int32_t best = -1, bm = -1;
    for (int32_t v = 0; v < k; ++v) {
      if (done[v]) continue;
      int32_t mm = 0;
      for (int32_t u = 0; u < k; ++u) mm += done[u] && padj[v * k + u];
      if (best < 0 || mm > bm || (mm == bm && deg[v] > deg[best])) { best = v; bm = mm; }
    }
    order[d] = best;
    done[best] = 1;
  }
  free(deg);
  free(done);
}

double oracle_wall_seconds(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/*
 * oracle_match: enumerate (want_table=1) or count all embeddings of the pattern
 * (k vertices, pm edges p_edges[pm][2]) in the data graph (n vertices, m edges edges[m][2]).
 * Only roots f(pi_0) in [root_begin, root_end) are explored (root_end < 0 means n), so a
 * contiguous root range is a bounded sample of the full enumeration.
 * Outputs: *count_out; *rows_out (malloc'd, sorted, [count][k], caller frees with
 * oracle_free) when want_table; *seconds_out = wall time of the enumeration (graph build
 * excluded); *threads_used.  Returns 0 or a negative error code.
 */
int oracle_match(int64_t n, const int32_t *edges, int64_t m, int drop_self_loops, int32_t k,
                 const int32_t *p_edges, int64_t pm, int induced, int64_t root_begin,
                 int64_t root_end, int threads, int want_table, uint64_t *count_out,
                 int32_t **rows_out, double *seconds_out, int *threads_used,
                 int32_t *order_out) {
  if (n < 0 || m < 0 || k < 1 || pm < 0 || !count_out) return OR_ARG;
  *count_out = 0;
  if (rows_out) *rows_out = NULL;
  if (seconds_out) *seconds_out = 0.0;
  uint8_t *padj = (uint8_t *)calloc((size_t)k * (size_t)k, 1);
  if (!padj) return OR_OOM;
  for (int64_t i = 0; i < pm; ++i) {
    int32_t a = p_edges[2 * i], b = p_edges[2 * i + 1];
    if (a < 0 || b < 0 || a >= k || b >= k) { free(padj); return OR_RANGE; }
    if (a == b) { free(padj); return OR_SELF; }
    padj[a * k + b] = padj[b * k + a] = 1;
  }
  /* pattern connectivity (§3.1 l.167 "we assume all graphs are ... connected") */
  {
    int32_t *st = (int32_t *)malloc(sizeof(int32_t) * (size_t)k);
    uint8_t *seen = (uint8_t *)calloc((size_t)k, 1);
    int32_t sp = 0, nseen = 1;
    st[sp++] = 0;
    seen[0] = 1;
    while (sp) {
      int32_t v = st[--sp];
      for (int32_t u = 0; u < k; ++u)
        if (padj[v * k + u] && !seen[u]) { seen[u] = 1; nseen++; st[sp++] = u; }
    }
    free(st);
    free(seen);
    if (nseen != k) { free(padj); return OR_DISC; }
  }
  og_graph g;
  int rc = build_graph(n, edges, m, drop_self_loops, &g);
  if (rc != OR_OK) { free(padj); return rc; }
  int32_t *order = (int32_t *)malloc(sizeof(int32_t) * (size_t)k);
  pattern_order(k, padj, order);
  if (order_out) memcpy(order_out, order, sizeof(int32_t) * (size_t)k);
  if (root_end < 0 || root_end > n) root_end = n;
  if (root_begin < 0) root_begin = 0;
  if (threads < 1) threads = 1;
  og_job job = {&g, k, padj, order, induced, want_table, root_begin, root_end, root_begin};
  og_worker *ws = (og_worker *)calloc((size_t)threads, sizeof(og_worker));
  pthread_t *tid = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
  double t0 = oracle_wall_seconds();
  if (k > n) {
    /* no injective map exists */
  } else if (threads == 1) {
    ws[0].job = &job;
    worker_main(&ws[0]);
  } else {
    for (int i = 0; i < threads; ++i) {
      ws[i].job = &job;
      pthread_create(&tid[i], NULL, worker_main, &ws[i]);
    }
    for (int i = 0; i < threads; ++i) pthread_join(tid[i], NULL);
  }
  uint64_t total = 0;
  int64_t nrows = 0;
  for (int i = 0; i < threads; ++i) {
    total += ws[i].count;
    nrows += ws[i].nrows;
    if (ws[i].err) rc = ws[i].err;
  }
  if (rc == OR_OK && want_table && rows_out) {
    int32_t *all = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nrows * k + 1));
    if (!all) rc = OR_OOM;
    else {
      int64_t p = 0;
      for (int i = 0; i < threads; ++i) {
        if (ws[i].nrows) memcpy(all + p * k, ws[i].rows, sizeof(int32_t) * (size_t)(ws[i].nrows * k));
        p += ws[i].nrows;
      }
      qsort_r(all, (size_t)nrows, sizeof(int32_t) * (size_t)k, cmp_row, &k);
      *rows_out = all;
    }
  }
  double t1 = oracle_wall_seconds();
  for (int i = 0; i < threads; ++i) free(ws[i].rows);
  free(ws);
  free(tid);
  free(order);
  free(padj);
  free_graph(&g);
  *count_out = total;
  if (seconds_out) *seconds_out = t1 - t0;
  if (threads_used) *threads_used = threads;
  return rc;
}

void oracle_free(void *p) { free(p); }
