// scoring.cu -- layout scoring and top-k selection (§6.5, P:501-503:
// "layout scoring ... applies a well-defined cost function to each candidate subgraph and then
// outputs the optimal one"; SPEC layout-scoring).
//
// The score of an embedding f is the product of the node fidelities of its k data vertices and
// the edge fidelities of its pattern edges' images.  The paper multiplies fidelity
// columns through the joins; edges are never shared between slices but boundary
// vertices are, so the node factors would be counted twice at every join.  This
// implementation therefore evaluates the canonical product once per final row, in the same
// float64 order as the definition (vertices 0..k-1, then pattern edges in the given order), on
// the device over the canonical table, and ranks with one stable radix sort on the score
// (descending; equal scores keep the canonical, lexicographic row order).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstring>
#include <vector>

#include "dm_device.cuh"

namespace dm {
namespace {

__device__ __forceinline__ int64_t find_arc(const int64_t *__restrict__ off, const int32_t *__restrict__ adj,
                                            int32_t u, int32_t v) {
  int64_t lo = off[u], hi = off[u + 1];
  const int64_t end = hi;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (adj[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return (lo < end && adj[lo] == v) ? lo : -1;
}

// score[i] of row i of the canonical table; key[i] = descending-order radix key of the score
__global__ void k_score(const int32_t *__restrict__ rows, int64_t n, int k, const int32_t *__restrict__ pe,
                        int pm, const double *__restrict__ node, const double *__restrict__ arcf,
                        const int64_t *__restrict__ off, const int32_t *__restrict__ adj,
                        double *__restrict__ score, unsigned long long *__restrict__ key, uint32_t *__restrict__ idx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t *r = rows + i * k;
    double s = 1.0;
    for (int v = 0; v < k; ++v) s = s * node[r[v]];
    for (int t = 0; t < pm; ++t) {
      const int64_t a = find_arc(off, adj, r[pe[2 * t]], r[pe[2 * t + 1]]);
      s = s * (a >= 0 ? arcf[a] : 0.0);
    }
    score[i] = s;
    unsigned long long b;
    memcpy(&b, &s, sizeof(b));  // s > 0: the IEEE bit pattern orders like the value
    key[i] = ~b;                 // ascending sort of ~bits = descending score
    idx[i] = (uint32_t)i;
  }
}

__global__ void k_pick(const int32_t *__restrict__ rows, int k, const double *__restrict__ score,
                       const uint32_t *__restrict__ order, int64_t m, int32_t *__restrict__ rows_out,
                       double *__restrict__ score_out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m * k; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / k;
    const int c = (int)(t - i * k);
    const uint32_t src = order[i];
    rows_out[t] = rows[(int64_t)src * k + c];
    if (c == 0) score_out[i] = score[src];
  }
}

int grid_sc(int64_t work) {
  const int64_t b = (work + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 16));
}

template <typename T>
struct DBuf {
  T *p = nullptr;
  cudaStream_t s = nullptr;
  cudaError_t alloc(size_t n, cudaStream_t st) {
    s = st;
    return cudaMallocAsync((void **)&p, sizeof(T) * std::max<size_t>(n, 1), st);
  }
  ~DBuf() {
    if (p) cudaFreeAsync(p, s);
  }
};

#define SC(call, what)                                                                        \
  do {                                                                                        \
    cudaError_t _e = (call);                                                                  \
    if (_e != cudaSuccess)                                                                    \
      return ::dm::fail(_e == cudaErrorMemoryAllocation ? DM_ERR_OOM : DM_ERR_CUDA,           \
                        std::string(what) + ": " + cudaGetErrorString(_e));                   \
  } while (0)

}  // namespace
}  // namespace dm

extern "C" {

dm_status dm_score_layouts(const dm_graph *g, int32_t k, const int32_t *p_edges, int64_t pm,
                           const double *node_fid, const int32_t *fid_edges, const double *fid_vals,
                           int64_t fm, const dm_match_opts *opt, int64_t top_k, int32_t *rows_out,
                           double *scores_out, int64_t *n_out, uint64_t *count_out) {
  dm::clear_error();
  dm::NvtxRange nvtx("dm_score_layouts");
  if (!g || !node_fid || (fm > 0 && (!fid_edges || !fid_vals)) || fm < 0 || !n_out)
    return dm::fail(DM_ERR_ARG, "NULL argument");
  if (top_k <= 0) return dm::fail(DM_ERR_ARG, "top_k must be positive");
  if (top_k > 0 && (!rows_out || !scores_out)) return dm::fail(DM_ERR_ARG, "NULL output buffers");
  const int64_t n = g->n;
  for (int64_t v = 0; v < n; ++v)
    if (!(node_fid[v] > 0.0 && node_fid[v] <= 1.0)) return dm::fail(DM_ERR_ARG, "node fidelity outside (0, 1]");
  // edge fidelities -> per arc of the CSR (both orientations); every data edge needs one
  std::vector<int64_t> off((size_t)n + 1);
  std::vector<int32_t> adj((size_t)std::max<int64_t>(g->arcs, 1));
  dm::DeviceGuard dg(g->device);
  if (!dg.ok) return dm::fail(DM_ERR_CUDA, "cudaSetDevice failed");
  cudaStream_t s = opt ? (cudaStream_t)opt->cuda_stream : nullptr;
  SC(cudaMemcpy(off.data(), g->d_off, sizeof(int64_t) * off.size(), cudaMemcpyDeviceToHost), "D2H offsets");
  if (g->arcs > 0) SC(cudaMemcpy(adj.data(), g->d_adj, sizeof(int32_t) * (size_t)g->arcs, cudaMemcpyDeviceToHost), "D2H adjacency");
  std::vector<double> arcf((size_t)std::max<int64_t>(g->arcs, 1), -1.0);
  for (int64_t i = 0; i < fm; ++i) {
    const int32_t u = fid_edges[2 * i], v = fid_edges[2 * i + 1];
    const double f = fid_vals[i];
    if (u < 0 || v < 0 || u >= n || v >= n) return dm::fail(DM_ERR_VERTEX_RANGE, "fidelity edge endpoint out of range");
    if (!(f > 0.0 && f <= 1.0)) return dm::fail(DM_ERR_ARG, "edge fidelity outside (0, 1]");
    for (int o = 0; o < 2; ++o) {
      const int32_t a = o ? v : u, b = o ? u : v;
      const auto it = std::lower_bound(adj.begin() + off[(size_t)a], adj.begin() + off[(size_t)a + 1], b);
      if (it == adj.begin() + off[(size_t)a + 1] || *it != b) return dm::fail(DM_ERR_ARG, "fidelity given for a non-edge");
      arcf[(size_t)(it - adj.begin())] = f;
    }
  }
  for (int64_t a = 0; a < g->arcs; ++a)
    if (arcf[(size_t)a] < 0) return dm::fail(DM_ERR_ARG, "a data edge has no fidelity");
  int32_t *d_tab = nullptr;
  uint64_t cnt = 0;
  dm_status st = dm::match_device_table(g, k, p_edges, pm, opt, &d_tab, &cnt);
  if (st != DM_OK) return st;
  struct Own {
    int32_t *p;
    cudaStream_t s;
    ~Own() {
      if (p) cudaFreeAsync(p, s);
    }
  } own{d_tab, s};
  if (count_out) *count_out = cnt;
  const int64_t m = std::min<int64_t>((int64_t)cnt, top_k);
  *n_out = m;
  if (cnt == 0) return DM_OK;
  if (cnt >= (uint64_t)UINT32_MAX) return dm::fail(DM_ERR_ROW_BUDGET, "too many layouts to rank");
  dm::DBuf<double> d_node, d_arcf, d_score, d_sout;
  dm::DBuf<int32_t> d_pe, d_rout;
  dm::DBuf<unsigned long long> d_key, d_key2;
  dm::DBuf<uint32_t> d_idx, d_idx2;
  SC(d_node.alloc((size_t)n, s), "alloc");
  SC(d_arcf.alloc(arcf.size(), s), "alloc");
  SC(d_pe.alloc((size_t)std::max<int64_t>(2 * pm, 1), s), "alloc");
  SC(d_score.alloc(cnt, s), "alloc");
  SC(d_key.alloc(cnt, s), "alloc");
  SC(d_key2.alloc(cnt, s), "alloc");
  SC(d_idx.alloc(cnt, s), "alloc");
  SC(d_idx2.alloc(cnt, s), "alloc");
  SC(d_rout.alloc((size_t)m * k, s), "alloc");
  SC(d_sout.alloc((size_t)m, s), "alloc");
  SC(cudaMemcpyAsync(d_node.p, node_fid, sizeof(double) * (size_t)n, cudaMemcpyHostToDevice, s), "H2D");
  SC(cudaMemcpyAsync(d_arcf.p, arcf.data(), sizeof(double) * arcf.size(), cudaMemcpyHostToDevice, s), "H2D");
  if (pm > 0) SC(cudaMemcpyAsync(d_pe.p, p_edges, sizeof(int32_t) * 2 * (size_t)pm, cudaMemcpyHostToDevice, s), "H2D");
  dm::k_score<<<dm::grid_sc((int64_t)cnt), 256, 0, s>>>(d_tab, (int64_t)cnt, k, d_pe.p, (int)pm, d_node.p, d_arcf.p,
                                                        g->d_off, g->d_adj, d_score.p, d_key.p, d_idx.p);
  SC(cudaGetLastError(), "score kernel");
  cub::DoubleBuffer<unsigned long long> dk(d_key.p, d_key2.p);
  cub::DoubleBuffer<uint32_t> dv(d_idx.p, d_idx2.p);
  size_t tb = 0;
  SC(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, (int64_t)cnt, 0, 64, s), "sort");
  dm::DBuf<unsigned char> tmp;
  SC(tmp.alloc(tb, s), "sort temp");
  SC(cub::DeviceRadixSort::SortPairs(tmp.p, tb, dk, dv, (int64_t)cnt, 0, 64, s), "sort");
  dm::k_pick<<<dm::grid_sc(m * k), 256, 0, s>>>(d_tab, k, d_score.p, dv.Current(), m, d_rout.p, d_sout.p);
  SC(cudaGetLastError(), "pick kernel");
  SC(cudaMemcpyAsync(rows_out, d_rout.p, sizeof(int32_t) * (size_t)m * k, cudaMemcpyDeviceToHost, s), "D2H");
  SC(cudaMemcpyAsync(scores_out, d_sout.p, sizeof(double) * (size_t)m, cudaMemcpyDeviceToHost, s), "D2H");
  SC(cudaStreamSynchronize(s), "sync");
  return DM_OK;
}

}  // extern "C"
