/*
 * pins_native.c -- TEST INFRASTRUCTURE: independent exact counters used as full-scale pins
 * (SURVEY.md §8(c) P-tri, P-dia, P-K4) where the backtracking oracle is too slow (R-MAT-20:
 * 1.5e12 labelled diamonds).  Shares nothing with the oracle or the CUDA path.
 *
 *   triangles(labelled)  = sum over arcs (u,v) of |N(u) & N(v)|            (= tr(A^3))
 *   diamonds (labelled)  = 2 * sum over edges e of t_e (t_e - 1), t_e = |N(u) & N(v)|
 *   K4 (distinct)        = degree-ordered counting: orient u->v iff (deg u, u) < (deg v, v);
 *                          sum over arcs u->v of sum over w in N+(u) & N+(v) of
 *                          |N+(u) & N+(v) & N+(w)|; labelled = 24 * distinct
 * Sorted-list merges, pthreads over source vertices.
 */
#define _GNU_SOURCE
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int64_t n;
  int64_t *off;
  int32_t *adj;
} csr_t;

static int cmp_u64(const void *a, const void *b) {
  uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
  return (x > y) - (x < y);
}

/* undirected simple graph (self-loops dropped, duplicates collapsed), both orientations */
static int build(int64_t n, const int32_t *e, int64_t m, csr_t *g) {
  uint64_t *k = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(2 * m + 1));
  if (!k) return -1;
  int64_t t = 0;
  for (int64_t i = 0; i < m; ++i) {
    int64_t a = e[2 * i], b = e[2 * i + 1];
    if (a == b || a < 0 || b < 0 || a >= n || b >= n) continue;
    k[t++] = ((uint64_t)a << 32) | (uint64_t)b;
    k[t++] = ((uint64_t)b << 32) | (uint64_t)a;
  }
  qsort(k, (size_t)t, sizeof(uint64_t), cmp_u64);
  int64_t u = 0;
  for (int64_t i = 0; i < t; ++i)
    if (i == 0 || k[i] != k[i - 1]) k[u++] = k[i];
  g->n = n;
  g->off = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
  g->adj = (int32_t *)malloc(sizeof(int32_t) * (size_t)(u + 1));
  for (int64_t i = 0; i < u; ++i) {
    g->off[(k[i] >> 32) + 1]++;
    g->adj[i] = (int32_t)(k[i] & 0xffffffffu);
  }
  for (int64_t v = 0; v < n; ++v) g->off[v + 1] += g->off[v];
  free(k);
  return 0;
}

static int64_t isect(const int32_t *a, int64_t na, const int32_t *b, int64_t nb) {
  int64_t i = 0, j = 0, c = 0;
  while (i < na && j < nb) {
    if (a[i] < b[j]) ++i;
    else if (a[i] > b[j]) ++j;
    else { ++c; ++i; ++j; }
  }
  return c;
}

typedef struct {
  const csr_t *g;
  const csr_t *h; /* oriented graph for K4 */
  int kind;       /* 0 triangles(labelled), 1 diamonds(labelled), 2 K4(distinct) */
  int64_t next;   /* shared vertex counter */
} shared_t;

typedef struct {
  shared_t *sh;
  uint64_t result;
} job_t;

static void *work(void *arg) {
  job_t *Jt = (job_t *)arg;
  shared_t *J = Jt->sh;
  const csr_t *g = J->g, *h = J->h;
  uint64_t s = 0;
  int32_t *buf = NULL;
  int64_t cap = 0;
  for (;;) {
    int64_t u = __atomic_fetch_add(&J->next, 1, __ATOMIC_RELAXED);
    if (u >= g->n) break;
    if (J->kind <= 1) {
      for (int64_t e = g->off[u]; e < g->off[u + 1]; ++e) {
        int64_t v = g->adj[e];
        if (J->kind == 1 && v <= u) continue; /* each undirected edge once */
        uint64_t t = (uint64_t)isect(g->adj + g->off[u], g->off[u + 1] - g->off[u], g->adj + g->off[v],
                                     g->off[v + 1] - g->off[v]);
        s += J->kind == 0 ? t : 2 * t * (t ? t - 1 : 0);
      }
    } else {
      const int32_t *nu = h->adj + h->off[u];
      int64_t du = h->off[u + 1] - h->off[u];
      if (cap < du + 1) {
        cap = du + 1;
        buf = (int32_t *)realloc(buf, sizeof(int32_t) * (size_t)cap);
      }
      for (int64_t i = 0; i < du; ++i) {
        int64_t v = nu[i];
        /* S = N+(u) & N+(v) */
        const int32_t *nv = h->adj + h->off[v];
        int64_t dv = h->off[v + 1] - h->off[v], a = 0, b = 0, ns = 0;
        while (a < du && b < dv) {
          if (nu[a] < nv[b]) ++a;
          else if (nu[a] > nv[b]) ++b;
          else { buf[ns++] = nu[a]; ++a; ++b; }
        }
        for (int64_t x = 0; x < ns; ++x) {
          int64_t w = buf[x];
          s += (uint64_t)isect(buf, ns, h->adj + h->off[w], h->off[w + 1] - h->off[w]);
        }
      }
    }
  }
  free(buf);
  Jt->result = s;
  return NULL;
}

static uint64_t run(int64_t n, const int32_t *e, int64_t m, int kind, int threads) {
  csr_t g, h = {0, NULL, NULL};
  if (build(n, e, m, &g)) return 0;
  if (kind == 2) { /* orientation by (degree, id) */
    h.n = n;
    h.off = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    h.adj = (int32_t *)malloc(sizeof(int32_t) * (size_t)(g.off[n] / 2 + 1));
    int64_t p = 0;
    for (int64_t u = 0; u < n; ++u) {
      int64_t du = g.off[u + 1] - g.off[u];
      for (int64_t e2 = g.off[u]; e2 < g.off[u + 1]; ++e2) {
        int64_t v = g.adj[e2], dv = g.off[v + 1] - g.off[v];
        if (du < dv || (du == dv && u < v)) h.adj[p++] = (int32_t)v; /* sorted: adj sorted */
      }
      h.off[u + 1] = p;
    }
  }
  if (threads < 1) threads = 1;
  pthread_t *tid = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
  job_t *jobs = (job_t *)calloc((size_t)threads, sizeof(job_t));
  shared_t sh = {&g, &h, kind, 0};
  for (int i = 0; i < threads; ++i) {
    jobs[i].sh = &sh;
    pthread_create(&tid[i], NULL, work, &jobs[i]);
  }
  uint64_t tot = 0;
  for (int i = 0; i < threads; ++i) {
    pthread_join(tid[i], NULL);
    tot += jobs[i].result;
  }
  free(tid);
  free(jobs);
  free(g.off);
  free(g.adj);
  free(h.off);
  free(h.adj);
  return tot;
}

uint64_t pins_triangles_labelled(int64_t n, const int32_t *e, int64_t m, int threads) {
  return run(n, e, m, 0, threads);
}
uint64_t pins_diamonds_labelled(int64_t n, const int32_t *e, int64_t m, int threads) {
  return run(n, e, m, 1, threads);
}
uint64_t pins_k4_distinct(int64_t n, const int32_t *e, int64_t m, int threads) {
  return run(n, e, m, 2, threads);
}
