// extend.cu -- the join step of Alg. 1 as one fused sm_100a kernel,
// launched twice per materialized step (count pass, write pass):
//
//   R <- InnerJoin(R, Res(M), C)        (equi-join on the key columns)
//   R <- FilterOverlappingNodes(R)      (all-distinct rule, P:237 / S:213)
//
// Res(M2) is the device CSR (sorted, both orientations), so the equi-join of a frontier row
// with Res(M2) on one key column is the CSR range of that key ("sort-merge join" with the
// sorted edge table), and every further join key is a lookup of (key, candidate) in the
// sorted edge table (a 2-key equi-join with Res(M2), i.e. the closing-edge probe of Fig. 2
// C1/C2).  Per frontier row and new pattern vertex, the key column whose data vertex has the
// smallest degree supplies the candidates (iterating the smaller side of the join); the
// other keys are probed by binary search in the shorter of the two adjacency lists.
//
// CTA = one tile of kTileRows consecutive frontier rows (one contiguous block of memory):
//   1. coalesced 16-byte loads of the tile into shared memory;
//   2. per row: choose the key (anchor) for the first new vertex, candidate count = degree;
//      CTA exclusive scan -> the tile's candidate space (load-balanced across the CTA even
//      when one row owns a hub);
//   3. each thread takes candidates j, tid + j*NT: injectivity against the row (FilterOverlapping-
//      Nodes) + closing-edge probes (+ non-edge probes in induced mode); for 2-vertex steps
//      (wedge / triangle slices) the second new vertex is enumerated the same way;
//   4. count pass: CTA sum -> block_cnt[tile] (and the running total / statistics);
//      write pass: CTA scan of survivors -> survivor list staged in shared memory -> warp-
//      cooperative coalesced row writes at the tile's offset from the exclusive scan of the
//      count pass.  Output order is deterministic (row order, then candidate order).
#include <cub/cub.cuh>

#include <mutex>

#include "dm_device.cuh"

namespace dm {

namespace {

__device__ __forceinline__ int64_t degree(const int64_t *__restrict__ off, int32_t v) {
  return __ldg(off + v + 1) - __ldg(off + v);
}

// is x in N(u)?  binary search in the shorter of N(u), N(x) (both sorted ascending)
__device__ __forceinline__ bool has_edge(const int64_t *__restrict__ off,
                                         const int32_t *__restrict__ adj, int32_t u, int32_t x) {
  int64_t lo = __ldg(off + u), hi = __ldg(off + u + 1);
  int64_t lo2 = __ldg(off + x), hi2 = __ldg(off + x + 1);
  int32_t key = x;
  if (hi2 - lo2 < hi - lo) {
    lo = lo2;
    hi = hi2;
    key = u;
  }
  const int64_t end = hi;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (__ldg(adj + mid) < key) lo = mid + 1;
    else hi = mid;
  }
  return lo < end && __ldg(adj + lo) == key;
}

// value of column c of the row being built (c == w -> first new vertex)
__device__ __forceinline__ int32_t colval(const int32_t *row, int w, int c, int32_t x0) {
  return c < w ? row[c] : x0;
}

// Filters for new vertex j with candidate value x (anchor column `acol` already satisfied):
// all-distinct, closing-edge probes, induced non-edge probes.
template <bool STATS>
__device__ __forceinline__ bool accept(const DevStep &st, int j, const int32_t *row, int w,
                                       int32_t x0, int32_t x, int acol,
                                       const int64_t *__restrict__ off,
                                       const int32_t *__restrict__ adj, uint64_t &probes) {
  for (int c = 0; c < w; ++c)
    if (row[c] == x) return false;
  if (j == 1 && x == x0) return false;
  for (int t = 0; t < st.n_nbr[j]; ++t) {
    int c = st.nbr[j][t];
    if (c == acol) continue;
    if (STATS) ++probes;
    if (!has_edge(off, adj, colval(row, w, c, x0), x)) return false;
  }
  for (int t = 0; t < st.n_non[j]; ++t) {
    int c = st.non[j][t];
    if (STATS) ++probes;
    if (has_edge(off, adj, colval(row, w, c, x0), x)) return false;
  }
  return true;
}

// key column with the smallest-degree image for new vertex j
__device__ __forceinline__ int pick_anchor(const DevStep &st, int j, const int32_t *row, int w,
                                           int32_t x0, const int64_t *__restrict__ off,
                                           int32_t &av, int64_t &ad) {
  int best = st.nbr[j][0];
  av = colval(row, w, best, x0);
  ad = degree(off, av);
  for (int t = 1; t < st.n_nbr[j]; ++t) {
    int c = st.nbr[j][t];
    int32_t v = colval(row, w, c, x0);
    int64_t d = degree(off, v);
    if (d < ad) {
      ad = d;
      av = v;
      best = c;
    }
  }
  return best;
}

struct SmemLayout {
  int32_t *rows;
  long long *pref;
  int32_t *anc;
  int32_t *acol;
  int32_t *sv_row;
  int32_t *sv_x;
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }

__host__ __device__ inline size_t smem_bytes(int in_w, bool write) {
  size_t b = align16(sizeof(int32_t) * (size_t)kTileRows * in_w);
  b += align16(sizeof(long long) * (kTileRows + 1));
  b += align16(sizeof(int32_t) * kTileRows) * 2;
  if (write) b += align16(sizeof(int32_t) * kSurvBuf) + align16(sizeof(int32_t) * 2 * kSurvBuf);
  return b;
}

__device__ inline SmemLayout carve(unsigned char *base, int in_w, bool write) {
  SmemLayout L;
  size_t o = 0;
  L.rows = reinterpret_cast<int32_t *>(base + o);
  o += align16(sizeof(int32_t) * (size_t)kTileRows * in_w);
  L.pref = reinterpret_cast<long long *>(base + o);
  o += align16(sizeof(long long) * (kTileRows + 1));
  L.anc = reinterpret_cast<int32_t *>(base + o);
  o += align16(sizeof(int32_t) * kTileRows);
  L.acol = reinterpret_cast<int32_t *>(base + o);
  o += align16(sizeof(int32_t) * kTileRows);
  if (write) {
    L.sv_row = reinterpret_cast<int32_t *>(base + o);
    o += align16(sizeof(int32_t) * kSurvBuf);
    L.sv_x = reinterpret_cast<int32_t *>(base + o);
  } else {
    L.sv_row = L.sv_x = nullptr;
  }
  return L;
}

// Write `fill` staged survivors as rows [base, base+fill) of out (width W): each warp writes
// whole rows, lanes map to columns, consecutive rows are contiguous -> coalesced stores.
__device__ __forceinline__ void flush_rows(const SmemLayout &L, int w, int W, int fill,
                                           int32_t *__restrict__ out, int64_t base) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = kStepThreads / 32;
  if (W <= 32) {
    const int rpi = 32 / W;
    const int lr = lane / W, lc = lane - lr * W;
    if (lr < rpi) {
      for (int s = warp * rpi + lr; s < fill; s += nwarps * rpi) {
        int32_t v = lc < w ? L.rows[L.sv_row[s] * w + lc] : L.sv_x[2 * s + (lc - w)];
        out[(base + s) * W + lc] = v;
      }
    }
  } else {
    for (int s = warp; s < fill; s += nwarps) {
      for (int c = lane; c < W; c += 32) {
        int32_t v = c < w ? L.rows[L.sv_row[s] * w + c] : L.sv_x[2 * s + (c - w)];
        out[(base + s) * W + c] = v;
      }
    }
  }
}

template <bool WRITE>
__global__ void __launch_bounds__(kStepThreads)
    k_step(const DevStep st, const StepIO io, const int64_t *__restrict__ off,
           const int32_t *__restrict__ adj) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  typedef cub::BlockScan<long long, kStepThreads> ScanLL;
  typedef cub::BlockScan<int, kStepThreads> ScanI;
  typedef cub::BlockReduce<unsigned long long, kStepThreads> RedU;
  __shared__ union {
    typename ScanLL::TempStorage ll;
    typename ScanI::TempStorage i;
    typename RedU::TempStorage r;
  } tmp;

  const int w = st.in_w;
  const int W = w + st.n_new;
  const int tid = threadIdx.x;
  const int64_t tile = io.block_begin + blockIdx.x;
  const int64_t r0 = tile * kTileRows;
  if (r0 >= io.in_rows) return;
  const int nrows = (int)(io.in_rows - r0 < kTileRows ? io.in_rows - r0 : kTileRows);
  SmemLayout L = carve(smem_raw, w, WRITE);

  // ---- 1. tile -> shared memory (contiguous rows; 16-byte vector loads)
  if (io.in) {
    const int32_t *src = io.in + r0 * w;
    const int nw = nrows * w;
    const int n4 = nw >> 2;
    const int4 *src4 = reinterpret_cast<const int4 *>(src);  // r0*w % 4 == 0 (kTileRows % 4 == 0)
    int4 *dst4 = reinterpret_cast<int4 *>(L.rows);
#pragma unroll 4
    for (int i = tid; i < n4; i += kStepThreads) dst4[i] = __ldcs(src4 + i);
    for (int i = (n4 << 2) + tid; i < nw; i += kStepThreads) L.rows[i] = __ldcs(src + i);
  } else {
    for (int i = tid; i < nrows; i += kStepThreads) L.rows[i] = (int32_t)(io.seed_base + r0 + i);
  }
  __syncthreads();

  // ---- 2. per-row join key for the first new vertex; tile candidate space
  long long cnt = 0;
  if (tid < nrows) {
    int32_t av;
    int64_t ad;
    L.acol[tid] = pick_anchor(st, 0, L.rows + tid * w, w, 0, off, av, ad);
    L.anc[tid] = av;
    cnt = ad;
  }
  long long pref, C;
  ScanLL(tmp.ll).ExclusiveSum(cnt, pref, C);
  L.pref[tid] = pref;
  __syncthreads();

  // ---- 3. candidates
  uint64_t my_surv = 0, my_cand = 0, my_probe = 0;
  int fill = 0;            // staged survivors (WRITE)
  int64_t base = 0;        // next output row (WRITE)
  if (WRITE) base = (int64_t)(io.block_off[tile] - io.out_base);

  for (long long j0 = 0; j0 < C; j0 += kStepThreads) {
    const long long j = j0 + tid;
    int r = -1, ns = 0;
    int32_t x0 = -1;
    if (j < C) {
      int lo = 0, hi = nrows;  // largest r with pref[r] <= j
      while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (L.pref[mid] <= j) lo = mid;
        else hi = mid;
      }
      r = lo;
      const int32_t *row = L.rows + r * w;
      const int32_t a = L.anc[r];
      x0 = __ldg(adj + __ldg(off + a) + (j - L.pref[r]));
      if (!WRITE) ++my_cand;
      if (accept<!WRITE>(st, 0, row, w, 0, x0, L.acol[r], off, adj, my_probe)) {
        if (st.n_new == 1) {
          ns = 1;
        } else {
          int32_t av;
          int64_t ad;
          const int ac = pick_anchor(st, 1, row, w, x0, off, av, ad);
          const int64_t e0 = __ldg(off + av);
          for (int64_t e = e0; e < e0 + ad; ++e) {
            const int32_t x1 = __ldg(adj + e);
            if (!WRITE) ++my_cand;
            if (accept<!WRITE>(st, 1, row, w, x0, x1, ac, off, adj, my_probe)) ++ns;
          }
        }
      }
    }
    if (!WRITE) {
      my_surv += ns;
      continue;
    }
    // ---- 4. (write) stage survivors, flush when the buffer would overflow
    int pos, rtot;
    ScanI(tmp.i).ExclusiveSum(ns, pos, rtot);
    if (fill + rtot > kSurvBuf) {
      __syncthreads();
      flush_rows(L, w, W, fill, io.out, base);
      __syncthreads();
      base += fill;
      fill = 0;
    }
    if (rtot > kSurvBuf) {
      // hub rows: this round alone overflows the buffer -> write directly (uncoalesced, rare)
      if (ns) {
        const int32_t *row = L.rows + r * w;
        int64_t o = base + pos;
        auto put = [&](int32_t x1) {
          int32_t *dst = io.out + o * W;
          for (int c = 0; c < w; ++c) dst[c] = row[c];
          dst[w] = x0;
          if (st.n_new == 2) dst[w + 1] = x1;
          ++o;
        };
        if (st.n_new == 1) {
          put(-1);
        } else {
          int32_t av;
          int64_t ad;
          const int ac = pick_anchor(st, 1, row, w, x0, off, av, ad);
          const int64_t e0 = __ldg(off + av);
          uint64_t dummy = 0;
          for (int64_t e = e0; e < e0 + ad; ++e) {
            const int32_t x1 = __ldg(adj + e);
            if (accept<false>(st, 1, row, w, x0, x1, ac, off, adj, dummy)) put(x1);
          }
        }
      }
      base += rtot;
      __syncthreads();
      continue;
    }
    if (ns) {
      int p = fill + pos;
      if (st.n_new == 1) {
        L.sv_row[p] = r;
        L.sv_x[2 * p] = x0;
      } else {
        const int32_t *row = L.rows + r * w;
        int32_t av;
        int64_t ad;
        const int ac = pick_anchor(st, 1, row, w, x0, off, av, ad);
        const int64_t e0 = __ldg(off + av);
        uint64_t dummy = 0;
        for (int64_t e = e0; e < e0 + ad; ++e) {
          const int32_t x1 = __ldg(adj + e);
          if (accept<false>(st, 1, row, w, x0, x1, ac, off, adj, dummy)) {
            L.sv_row[p] = r;
            L.sv_x[2 * p] = x0;
            L.sv_x[2 * p + 1] = x1;
            ++p;
          }
        }
      }
    }
    fill += rtot;
    __syncthreads();  // scan temp storage reuse + staged entries visible
  }

  if (WRITE) {
    __syncthreads();
    flush_rows(L, w, W, fill, io.out, base);
    return;
  }
  // ---- 4. (count) tile total + statistics
  unsigned long long t = RedU(tmp.r).Sum((unsigned long long)my_surv);
  __syncthreads();
  unsigned long long tc = RedU(tmp.r).Sum((unsigned long long)my_cand);
  __syncthreads();
  unsigned long long tp = RedU(tmp.r).Sum((unsigned long long)my_probe);
  if (tid == 0) {
    if (io.block_cnt) io.block_cnt[tile] = t;
    if (io.total) atomicAdd(io.total, t);
    if (io.stats) {
      atomicAdd(io.stats, tc);
      atomicAdd(io.stats + 1, tp);
    }
  }
}

}  // namespace

size_t step_smem_bytes(int in_w, bool write_pass) { return smem_bytes(in_w, write_pass); }

// Raise the dynamic shared-memory limit of a kernel once per (device, size) growth.
static cudaError_t prep(const void *fn, int which, size_t smem) {
  static std::mutex mu;
  static size_t configured[64][2] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 64 && configured[dev][which] >= smem) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess && dev < 64) configured[dev][which] = smem;
  return e;
}

cudaError_t launch_step_count(const DevStep &st, const StepIO &io, const dm_graph &g,
                              int64_t num_tiles, cudaStream_t s) {
  if (num_tiles <= 0) return cudaSuccess;
  size_t smem = smem_bytes(st.in_w, false);
  cudaError_t e = prep((const void *)k_step<false>, 0, smem);
  if (e != cudaSuccess) return e;
  k_step<false><<<(unsigned)num_tiles, kStepThreads, smem, s>>>(st, io, g.d_off, g.d_adj);
  return cudaGetLastError();
}

cudaError_t launch_step_write(const DevStep &st, const StepIO &io, const dm_graph &g,
                              int64_t num_tiles, cudaStream_t s) {
  if (num_tiles <= 0) return cudaSuccess;
  size_t smem = smem_bytes(st.in_w, true);
  cudaError_t e = prep((const void *)k_step<true>, 1, smem);
  if (e != cudaSuccess) return e;
  k_step<true><<<(unsigned)num_tiles, kStepThreads, smem, s>>>(st, io, g.d_off, g.d_adj);
  return cudaGetLastError();
}

DevStep make_dev_step(const Step &st) {
  DevStep d{};
  d.in_w = st.in_w;
  d.n_new = st.n_new;
  for (int j = 0; j < st.n_new; ++j) {
    d.n_nbr[j] = st.nv[j].n_nbr;
    d.n_non[j] = st.nv[j].n_non;
    for (int t = 0; t < st.nv[j].n_nbr; ++t) d.nbr[j][t] = (uint8_t)st.nv[j].nbr[t];
    for (int t = 0; t < st.nv[j].n_non; ++t) d.non[j][t] = (uint8_t)st.nv[j].non[t];
  }
  return d;
}

}  // namespace dm
