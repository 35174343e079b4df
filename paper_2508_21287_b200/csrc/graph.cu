// graph.cu -- GPU edge-table / CSR builder: Res(M2) = E_d \ E_self in both orientations
// (§3.4, Alg. 2 l.2 P:270).
//
//   H2D edge list -> k_make_arcs (validate ids, drop/reject self-loops, emit both
//   orientations as 64-bit keys (u << 32 | v)) -> CUB radix sort -> CUB unique -> k_bounds
//   (CSR offsets from the sorted keys, no atomics) + k_split (adjacency ids) -> max degree.
// Every adjacency list comes out sorted ascending (the probe kernels binary-search it).
#include <atomic>
#include <cub/cub.cuh>

#include <algorithm>
#include <new>

#include "dm_device.cuh"

namespace dm {
namespace {

__global__ void k_make_arcs(const int32_t *__restrict__ edges, int64_t m, int32_t n, int drop_self,
                            unsigned long long *__restrict__ keys, int *__restrict__ err) {
  const unsigned long long marker = (unsigned long long)n << 32;  // sorts after every real arc
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    int2 e = reinterpret_cast<const int2 *>(edges)[i];
    unsigned long long k0 = marker, k1 = marker;
    if (e.x < 0 || e.y < 0 || e.x >= n || e.y >= n) {
      atomicOr(err, 1);
    } else if (e.x == e.y) {
      if (!drop_self) atomicOr(err, 2);
    } else {
      k0 = ((unsigned long long)(uint32_t)e.x << 32) | (uint32_t)e.y;
      k1 = ((unsigned long long)(uint32_t)e.y << 32) | (uint32_t)e.x;
    }
    keys[2 * i] = k0;
    keys[2 * i + 1] = k1;
  }
}

// off[v] = index of the first arc with source >= v (arcs sorted by key, `arcs` real arcs)
__global__ void k_bounds(const unsigned long long *__restrict__ keys, int64_t arcs, int32_t n,
                         int64_t *__restrict__ off, int32_t *__restrict__ adj) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= arcs;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t src = (i < arcs) ? (int64_t)(keys[i] >> 32) : (int64_t)n;
    int64_t prev = (i > 0) ? (int64_t)(keys[i - 1] >> 32) : -1;
    for (int64_t v = prev + 1; v <= src; ++v) off[v] = i;
    if (i < arcs) adj[i] = (int32_t)(keys[i] & 0xffffffffULL);
  }
}

__global__ void k_max_degree(const int64_t *__restrict__ off, int32_t n, int *__restrict__ out) {
  int best = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    best = max(best, (int)(off[v + 1] - off[v]));
  typedef cub::BlockReduce<int, 256> BR;
  __shared__ typename BR::TempStorage tmp;
  int r = BR(tmp).Reduce(best, cub::Max());
  if (threadIdx.x == 0) atomicMax(out, r);
}

// ELL copy of a max-degree-4 adjacency: one 16-byte load returns a vertex's whole sorted list
__global__ void k_build_ell(const int64_t *__restrict__ off, const int32_t *__restrict__ adj,
                            int32_t n, int4 *__restrict__ ell) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = off[v], d = off[v + 1] - b;
    int4 e;
    e.x = d > 0 ? adj[b] : -1;
    e.y = d > 1 ? adj[b + 1] : -1;
    e.z = d > 2 ? adj[b + 2] : -1;
    e.w = d > 3 ? adj[b + 3] : -1;
    ell[v] = e;
  }
}

// sum of squared degrees (double, one atomic per block)
__global__ void k_sum_d2(const int64_t *__restrict__ off, int32_t n, double *__restrict__ out) {
  double acc = 0.0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const double d = (double)(off[v + 1] - off[v]);
    acc += d * d;
  }
  typedef cub::BlockReduce<double, 256> BR;
  __shared__ typename BR::TempStorage tmp;
  const double r = BR(tmp).Sum(acc);
  if (threadIdx.x == 0) atomicAdd(out, r);
}

// Triangle closure on a deterministic sample of arcs (a,b): sum over samples of
// |N(a) & N(b)| and of (deg(b) - 1) (wedges a-b-c); ratio = closure probability.
__global__ void k_sample_closure(const int64_t *__restrict__ off, const int32_t *__restrict__ adj,
                                 int32_t n, int64_t arcs, int samples, double *__restrict__ out) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < samples; s += gridDim.x * blockDim.x) {
    const uint64_t h = (uint64_t)(s + 1) * 0x9E3779B97F4A7C15ull;
    const int64_t e = (int64_t)((h >> 11) % (uint64_t)arcs);
    int64_t lo = 0, hi = n;  // source vertex a of arc e: largest a with off[a] <= e
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (off[mid] <= e) lo = mid;
      else hi = mid;
    }
    const int32_t a = (int32_t)lo, b = adj[e];
    int64_t i = off[a], ie = off[a + 1], j = off[b], je = off[b + 1];
    const double wedges = (double)(je - j - 1);
    double t = 0.0;
    while (i < ie && j < je) {  // merge intersection of two sorted lists
      const int32_t x = adj[i], y = adj[j];
      t += (x == y);
      i += (x <= y);
      j += (y <= x);
    }
    atomicAdd(out, t);
    atomicAdd(out + 1, wedges);
  }
}

int grid_for(int64_t work) {
  int64_t b = (work + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 16));
}

}  // namespace

void configure_pool(int device) {
  static std::mutex mu;
  static bool done[64] = {};
  std::lock_guard<std::mutex> lk(mu);
  if (device < 0 || device >= 64 || done[device]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[device] = true;
}

static dm_status graph_create_impl(int32_t n, const int32_t *edges, int64_t m, int32_t flags,
                                   int32_t device, dm_graph **out) {
  if (!out) return fail(DM_ERR_ARG, "out is NULL");
  if (n < 0 || m < 0 || (m > 0 && !edges)) return fail(DM_ERR_ARG, "bad graph arguments");
  if (n >= INT32_MAX) return fail(DM_ERR_ARG, "n too large");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(DM_ERR_CUDA, "no CUDA device available (libdeltamotif has no CPU fallback)");
  if (device < 0 || device >= ndev) return fail(DM_ERR_ARG, "bad device ordinal");
  DeviceGuard dg(device);
  if (!dg.ok) return fail(DM_ERR_CUDA, "cudaSetDevice failed");
  configure_pool(device);
  cudaStream_t s;
  DM_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamDestroy(s); }
  } sg{s};

  dm_graph *g = new (std::nothrow) dm_graph;
  static std::atomic<uint64_t> next_gen{1};
  if (g) g->gen = next_gen.fetch_add(1);
  if (!g) return fail(DM_ERR_OOM, "host allocation failed");
  g->tabs = new (std::nothrow) TabStore;
  if (!g->tabs) {
    delete g;
    return fail(DM_ERR_OOM, "host allocation failed");
  }
  g->device = device;
  g->n = n;
  const int64_t nk = 2 * m;
  int32_t *d_edges = nullptr;
  unsigned long long *d_keys = nullptr, *d_sorted = nullptr, *d_uniq = nullptr;
  int64_t *d_nsel = nullptr;
  int *d_err = nullptr;
  void *d_tmp = nullptr;
  // every device buffer comes from the stream-ordered pool (create / destroy cycles reuse memory)
  auto release = [&](void *p) {
    if (p) cudaFreeAsync(p, s);
  };
  auto cleanup = [&]() {
    release(d_edges);
    release(d_keys);
    release(d_sorted);
    release(d_uniq);
    release(d_nsel);
    release(d_err);
    release(d_tmp);
  };
  auto bail = [&](dm_status st) {
    cleanup();
    release(g->d_off);
    release(g->d_adj);
    release(g->d_ell);
    cudaStreamSynchronize(s);
    delete g->tabs;
    delete g;
    return st;
  };
#define GC(call)                                                                           \
  do {                                                                                     \
    cudaError_t _e = (call);                                                               \
    if (_e != cudaSuccess)                                                                 \
      return bail(fail(_e == cudaErrorMemoryAllocation ? DM_ERR_OOM : DM_ERR_CUDA,         \
                       std::string(#call " failed: ") + cudaGetErrorString(_e)));          \
  } while (0)

  GC(cudaMallocAsync(&g->d_off, sizeof(int64_t) * ((size_t)n + 1), s));
  GC(cudaMallocAsync(&d_err, sizeof(int), s));
  GC(cudaMemsetAsync(d_err, 0, sizeof(int), s));
  int64_t arcs = 0;
  if (m > 0) {
    GC(cudaMallocAsync(&d_edges, sizeof(int32_t) * 2 * (size_t)m, s));
    GC(cudaMallocAsync(&d_keys, sizeof(unsigned long long) * (size_t)nk, s));
    GC(cudaMallocAsync(&d_sorted, sizeof(unsigned long long) * (size_t)nk, s));
    GC(cudaMallocAsync(&d_uniq, sizeof(unsigned long long) * (size_t)nk, s));
    GC(cudaMallocAsync(&d_nsel, sizeof(int64_t), s));
    GC(cudaMemcpyAsync(d_edges, edges, sizeof(int32_t) * 2 * (size_t)m, cudaMemcpyHostToDevice, s));
    k_make_arcs<<<grid_for(m), 256, 0, s>>>(d_edges, m, n, flags & DM_GRAPH_DROP_SELF_LOOPS,
                                            d_keys, d_err);
    GC(cudaGetLastError());
    int herr = 0;
    GC(cudaMemcpyAsync(&herr, d_err, sizeof(int), cudaMemcpyDeviceToHost, s));
    GC(cudaStreamSynchronize(s));
    if (herr & 1) return bail(fail(DM_ERR_VERTEX_RANGE, "edge endpoint outside [0, n)"));
    if (herr & 2) return bail(fail(DM_ERR_SELF_LOOP, "self-loop in data graph (pass DM_GRAPH_DROP_SELF_LOOPS to drop)"));
    int end_bit = 32;
    while (end_bit < 64 && ((unsigned long long)n >> (end_bit - 32)) != 0) ++end_bit;
    size_t tmp_sort = 0, tmp_uniq = 0;
    GC(cub::DeviceRadixSort::SortKeys(nullptr, tmp_sort, d_keys, d_sorted, nk, 0, end_bit, s));
    GC(cub::DeviceSelect::Unique(nullptr, tmp_uniq, d_sorted, d_uniq, d_nsel, nk, s));
    size_t tmp = std::max(tmp_sort, tmp_uniq);
    GC(cudaMallocAsync(&d_tmp, tmp, s));
    GC(cub::DeviceRadixSort::SortKeys(d_tmp, tmp, d_keys, d_sorted, nk, 0, end_bit, s));
    GC(cub::DeviceSelect::Unique(d_tmp, tmp, d_sorted, d_uniq, d_nsel, nk, s));
    int64_t nsel = 0;
    GC(cudaMemcpyAsync(&nsel, d_nsel, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    GC(cudaStreamSynchronize(s));
    arcs = nsel;
    if (nsel > 0) {
      unsigned long long last = 0;
      GC(cudaMemcpy(&last, d_uniq + nsel - 1, sizeof(last), cudaMemcpyDeviceToHost));
      if ((last >> 32) == (unsigned long long)n) arcs = nsel - 1;  // the dropped-edge marker
    }
  }
  g->arcs = arcs;
  GC(cudaMallocAsync(&g->d_adj, sizeof(int32_t) * (size_t)std::max<int64_t>(arcs, 1), s));
  if (arcs > 0) {
    k_bounds<<<grid_for(arcs + 1), 256, 0, s>>>(d_uniq, arcs, n, g->d_off, g->d_adj);
    GC(cudaGetLastError());
  } else {
    GC(cudaMemsetAsync(g->d_off, 0, sizeof(int64_t) * ((size_t)n + 1), s));
  }
  int hmax = 0;
  if (n > 0) {
    GC(cudaMemsetAsync(d_err, 0, sizeof(int), s));
    k_max_degree<<<grid_for(n), 256, 0, s>>>(g->d_off, n, d_err);
    GC(cudaGetLastError());
    GC(cudaMemcpyAsync(&hmax, d_err, sizeof(int), cudaMemcpyDeviceToHost, s));
  }
  GC(cudaStreamSynchronize(s));
  g->max_deg = hmax;
  if (n > 0 && arcs > 0) {  // statistics for the join-order cost model
    double *d_stat = nullptr;
    GC(cudaMallocAsync(&d_stat, 3 * sizeof(double), s));
    GC(cudaMemsetAsync(d_stat, 0, 3 * sizeof(double), s));
    k_sum_d2<<<grid_for(n), 256, 0, s>>>(g->d_off, n, d_stat);
    const int samples = 4096;
    k_sample_closure<<<16, 256, 0, s>>>(g->d_off, g->d_adj, n, arcs, samples, d_stat + 1);
    double hs[3] = {0, 0, 0};
    cudaError_t e1 = cudaGetLastError();
    cudaError_t e2 = cudaMemcpyAsync(hs, d_stat, sizeof(hs), cudaMemcpyDeviceToHost, s);
    cudaError_t e3 = cudaStreamSynchronize(s);
    cudaFreeAsync(d_stat, s);
    GC(e1);
    GC(e2);
    GC(e3);
    g->sum_d2 = hs[0];
    g->closure = hs[2] > 0 ? hs[1] / hs[2] : 0.0;
  }
  if (n > 0 && hmax <= 4) {
    GC(cudaMallocAsync(&g->d_ell, sizeof(int4) * (size_t)n, s));
    k_build_ell<<<grid_for(n), 256, 0, s>>>(g->d_off, g->d_adj, n, reinterpret_cast<int4 *>(g->d_ell));
    GC(cudaGetLastError());
    GC(cudaStreamSynchronize(s));
  }
#undef GC
  cleanup();
  *out = g;
  return DM_OK;
}

}  // namespace dm

extern "C" {

dm_status dm_graph_create(int32_t n, const int32_t *edges, int64_t m, int32_t flags,
                          int32_t device, dm_graph **out) {
  dm::clear_error();
  dm::NvtxRange nvtx("dm_graph_create");
  return dm::graph_create_impl(n, edges, m, flags, device, out);
}

// Every buffer of a graph comes from the device's stream-ordered pool; no work on g is in flight
// when it is destroyed (dm_match and the step-level calls return after their stream work), so
// the buffers go back to the pool in legacy-stream order without a device-wide synchronisation.
void dm_graph_destroy(dm_graph *g) {
  if (!g) return;
  dm::DeviceGuard dg(g->device);
  auto release = [](void *p) {
    if (p) cudaFreeAsync(p, nullptr);
  };
  if (g->tabs) {
    for (auto &t : g->tabs->t) {
      release(t.d_rows);
      release(t.d_toff);
    }
    release(g->tabs->apex.d_toff);
    release(g->tabs->apex.d_apex);
    delete g->tabs;
  }
  release(g->d_off);
  release(g->d_adj);
  release(g->d_ell);
  delete g;
}

int32_t dm_graph_num_vertices(const dm_graph *g) { return g ? g->n : -1; }
int64_t dm_graph_num_arcs(const dm_graph *g) { return g ? g->arcs : -1; }
int32_t dm_graph_max_degree(const dm_graph *g) { return g ? g->max_deg : -1; }
int32_t dm_graph_device(const dm_graph *g) { return g ? g->device : -1; }

dm_status dm_graph_stats(const dm_graph *g, double *sum_d2, double *closure) {
  dm::clear_error();
  if (!g) return dm::fail(DM_ERR_ARG, "graph is NULL");
  if (sum_d2) *sum_d2 = g->sum_d2;
  if (closure) *closure = g->closure;
  return DM_OK;
}

dm_status dm_graph_device_csr(const dm_graph *g, const int64_t **d_off, const int32_t **d_adj) {
  dm::clear_error();
  if (!g) return dm::fail(DM_ERR_ARG, "graph is NULL");
  if (d_off) *d_off = g->d_off;
  if (d_adj) *d_adj = g->d_adj;
  return DM_OK;
}

dm_status dm_graph_copy_csr(const dm_graph *g, int64_t *off_out, int32_t *adj_out) {
  dm::clear_error();
  if (!g) return dm::fail(DM_ERR_ARG, "graph is NULL");
  dm::DeviceGuard dg(g->device);
  if (off_out)
    DM_CUDA(cudaMemcpy(off_out, g->d_off, sizeof(int64_t) * ((size_t)g->n + 1), cudaMemcpyDeviceToHost));
  if (adj_out && g->arcs > 0)
    DM_CUDA(cudaMemcpy(adj_out, g->d_adj, sizeof(int32_t) * (size_t)g->arcs, cudaMemcpyDeviceToHost));
  return DM_OK;
}

}  // extern "C"
