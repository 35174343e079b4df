// extend.cu -- the join step of Alg. 1 as one fused sm_100a kernel:
//
//   R <- InnerJoin(R, Res(M), C)        (equi-join on the key columns)
//   R <- FilterOverlappingNodes(R)      (all-distinct rule, P:237 / S:213)
//
// Res(M2) is the device CSR (sorted, both orientations), so the equi-join of a frontier row
// with Res(M2) on one key column is the CSR range of that key (a sort-merge join against the
// sorted edge table), and every further join key is a lookup of (key, candidate) in the
// sorted edge table (a 2-key equi-join with Res(M2): the closing-edge probe of Fig. 2 C1/C2).
// Per frontier row and new pattern vertex, the key column whose data vertex has the smallest
// degree supplies the candidates (iterating the smaller side of the join); the other keys are
// probed by binary search in the shorter of the two adjacency lists.
//
// CTA = one tile of kTileRows consecutive frontier rows (one contiguous block of memory):
//   1. tile -> shared memory with one TMA bulk copy (cp.async.bulk + mbarrier);
//   2. per row: join key (anchor) of the first new vertex, candidate count = its degree; CTA
//      exclusive scan -> the tile's candidate space (a hub row is spread over the CTA);
//   3. rounds of kStepThreads candidates: injectivity + closing-edge (+ induced non-edge)
//      probes; for 2-vertex steps (wedge / triangle slices) the accepted first vertices of the
//      round and their second-vertex candidate counts are scanned again, so every second-level
//      candidate is one thread too (each candidate is evaluated exactly once per launch);
//   4. survivors are staged in shared memory (CTA scan -> deterministic order: row order, then
//      candidate order) and written with warp-cooperative coalesced row stores.
//
// Launch modes:
//   kModeCount  : count only (the count-mode last step: the last level is never materialized);
//   kModeWrite  : write at offsets from an exclusive prefix over tiles (re-run / chunked path);
//   kModeSingle : single pass with decoupled look-back -- each tile publishes its survivor
//                 count, looks back for its exclusive prefix and writes immediately if the
//                 output capacity allows; tiles that do not fit (capacity or staging buffer)
//                 record themselves and are re-run by the host with kModeWrite.
#include <cub/cub.cuh>

#include <mutex>

#include "dm_device.cuh"

namespace dm {

namespace {

constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagPrefix = 2ull << 62;
constexpr unsigned long long kValueMask = (1ull << 62) - 1;

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

// x in row?  branch-free, unrolled by 4 (rows sit at stride w in shared memory; for odd w a
// warp's rows fall in distinct banks).
__device__ __forceinline__ bool in_row(const int32_t *row, int w, int32_t x) {
  bool hit = false;
  int c = 0;
  for (; c + 4 <= w; c += 4) {
    const int32_t a = row[c], b = row[c + 1], d = row[c + 2], e = row[c + 3];
    hit |= (a == x) | (b == x) | (d == x) | (e == x);
  }
  for (; c < w; ++c) hit |= row[c] == x;
  return hit;
}

// ---- TMA 1-D bulk copy global -> shared, completion tracked by an mbarrier (sm_90+ / sm_100a)
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
  unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
  unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
      "l"(src), "r"(bytes), "r"(b)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned phase) {
  unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(a), "r"(phase)
        : "memory");
  }
}

// value of column c of the row being built (c == w -> first new vertex)
__device__ __forceinline__ int32_t colval(const int32_t *row, int w, int c, int32_t x0) {
  return c < w ? row[c] : x0;
}

// Filters for new vertex j with candidate value x (anchor column `acol` is satisfied by
// construction): all-distinct, closing-edge probes, induced non-edge probes.
__device__ __forceinline__ bool accept(const DevStep &st, int j, const int32_t *row, int w,
                                       int32_t x0, int32_t x, int acol,
                                       const int64_t *__restrict__ off,
                                       const int32_t *__restrict__ adj, uint32_t &probes) {
  if (in_row(row, w, x)) return false;
  if (j == 1 && x == x0) return false;
  for (int t = 0; t < st.n_nbr[j]; ++t) {
    int c = st.nbr[j][t];
    if (c == acol) continue;
    ++probes;
    if (!has_edge(off, adj, colval(row, w, c, x0), x)) return false;
  }
  for (int t = 0; t < st.n_non[j]; ++t) {
    ++probes;
    if (has_edge(off, adj, colval(row, w, st.non[j][t], x0), x)) return false;
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

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }

struct SmemLayout {
  int32_t *rows;     // [kTileRows][w] (the tile, contiguous as in global memory)
  long long *pref;   // [kTileRows]    first-vertex candidate prefix
  int32_t *anc;      // [kTileRows]    first-vertex anchor vertex
  int32_t *acol;     // [kTileRows]    first-vertex anchor column
  long long *apref;  // [kStepThreads] second-vertex candidate prefix (per round)
  int32_t *ar;       // [kStepThreads] row of the accepted first vertex
  int32_t *ax0;      // [kStepThreads] accepted first vertex
  int32_t *aav;      // [kStepThreads] second-vertex anchor vertex
  int32_t *aacol;    // [kStepThreads] second-vertex anchor column
  int32_t *sv_row;   // [kSurvBuf]
  int32_t *sv_x;     // [kSurvBuf][2]
};

__host__ __device__ inline size_t smem_bytes(int in_w, bool stage) {
  size_t b = align16(sizeof(int32_t) * (size_t)kTileRows * in_w);
  b += align16(sizeof(long long) * kTileRows);
  b += 2 * align16(sizeof(int32_t) * kTileRows);
  b += align16(sizeof(long long) * kStepThreads);
  b += 4 * align16(sizeof(int32_t) * kStepThreads);
  if (stage) b += align16(sizeof(int32_t) * kSurvBuf) + align16(sizeof(int32_t) * 2 * kSurvBuf);
  return b;
}

__device__ inline SmemLayout carve(unsigned char *base, int in_w, bool stage) {
  SmemLayout L;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    unsigned char *p = base + o;
    o += align16(bytes);
    return p;
  };
  L.rows = reinterpret_cast<int32_t *>(take(sizeof(int32_t) * (size_t)kTileRows * in_w));
  L.pref = reinterpret_cast<long long *>(take(sizeof(long long) * kTileRows));
  L.anc = reinterpret_cast<int32_t *>(take(sizeof(int32_t) * kTileRows));
  L.acol = reinterpret_cast<int32_t *>(take(sizeof(int32_t) * kTileRows));
  L.apref = reinterpret_cast<long long *>(take(sizeof(long long) * kStepThreads));
  L.ar = reinterpret_cast<int32_t *>(take(sizeof(int32_t) * kStepThreads));
  L.ax0 = reinterpret_cast<int32_t *>(take(sizeof(int32_t) * kStepThreads));
  L.aav = reinterpret_cast<int32_t *>(take(sizeof(int32_t) * kStepThreads));
  L.aacol = reinterpret_cast<int32_t *>(take(sizeof(int32_t) * kStepThreads));
  if (stage) {
    L.sv_row = reinterpret_cast<int32_t *>(take(sizeof(int32_t) * kSurvBuf));
    L.sv_x = reinterpret_cast<int32_t *>(take(sizeof(int32_t) * 2 * kSurvBuf));
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

__device__ __forceinline__ unsigned long long ld_volatile(const unsigned long long *p) {
  return *reinterpret_cast<const volatile unsigned long long *>(p);
}
__device__ __forceinline__ void st_volatile(unsigned long long *p, unsigned long long v) {
  *reinterpret_cast<volatile unsigned long long *>(p) = v;
}

template <int MODE>
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
  __shared__ unsigned long long s_bc;
  __shared__ __align__(8) uint64_t s_bar;
  constexpr bool kStage = MODE != kModeCount;

  const int w = st.in_w;
  const int W = w + st.n_new;
  const int tid = threadIdx.x;
  int64_t tile;
  if (MODE == kModeSingle) {
    if (tid == 0) s_bc = atomicAdd(io.ctrl + 0, 1ull);  // dynamic tile id: forward progress
    __syncthreads();
    tile = (int64_t)s_bc;
  } else {
    tile = io.block_begin + blockIdx.x;
  }
  const int64_t r0 = tile * kTileRows;
  if (r0 >= io.in_rows) return;
  const int nrows = (int)(io.in_rows - r0 < kTileRows ? io.in_rows - r0 : kTileRows);
  SmemLayout L = carve(smem_raw, w, kStage);

  // ---- 1. tile -> shared memory: one TMA bulk copy of the contiguous tile (16-byte multiple;
  //         the <= 3-word tail of the last tile with plain loads), mbarrier completion
  if (io.in) {
    const int32_t *src = io.in + r0 * w;
    const int nw = nrows * w;
    const unsigned bulk = (unsigned)(nw & ~3) * 4u;
    const bool aligned = ((reinterpret_cast<uintptr_t>(src) & 15) == 0);
    if (aligned && bulk > 0) {
      if (tid == 0) mbar_init(&s_bar, 1);
      __syncthreads();
      if (tid == 0) {
        mbar_expect_tx(&s_bar, bulk);
        tma_bulk_g2s(L.rows, src, bulk, &s_bar);
      }
      for (int i = (nw & ~3) + tid; i < nw; i += kStepThreads) L.rows[i] = __ldcs(src + i);
      mbar_wait(&s_bar, 0);
    } else {
      for (int i = tid; i < nw; i += kStepThreads) L.rows[i] = __ldcs(src + i);
    }
  } else {
    for (int r = tid; r < nrows; r += kStepThreads) L.rows[r] = (int32_t)(io.seed_base + r0 + r);
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
  long long pref, C0;
  ScanLL(tmp.ll).ExclusiveSum(cnt, pref, C0);
  L.pref[tid] = pref;
  __syncthreads();

  uint32_t my_cand = 0, my_probe = 0;
  unsigned long long my_surv = 0;  // kModeCount
  int fill = 0;                    // staged survivors
  long long agg = 0;               // kModeSingle: survivors of the tile
  bool ovf = false;                // kModeSingle: staging buffer overflowed
  int64_t base = 0;                // kModeWrite: next output row
  if (MODE == kModeWrite) base = (int64_t)(io.block_off[tile] - io.out_base);

  // block-wide: at most one survivor per thread
  auto emit = [&](bool s, int r, int32_t x0, int32_t x1) {
    if (MODE == kModeCount) {
      my_surv += s;
      return;
    }
    int pos, tot;
    ScanI(tmp.i).ExclusiveSum(s ? 1 : 0, pos, tot);
    if (MODE == kModeWrite && fill + tot > kSurvBuf) {
      __syncthreads();
      flush_rows(L, w, W, fill, io.out, base);
      __syncthreads();
      base += fill;
      fill = 0;
    }
    if (MODE == kModeSingle) {
      agg += tot;
      if (fill + tot > kSurvBuf) ovf = true;
    }
    if (s && !ovf) {
      const int p = fill + pos;
      L.sv_row[p] = r;
      L.sv_x[2 * p] = x0;
      L.sv_x[2 * p + 1] = x1;
    }
    if (!ovf) fill += tot;
    __syncthreads();  // scan storage reuse
  };

  // ---- 3. candidate rounds
  for (long long j0 = 0; j0 < C0; j0 += kStepThreads) {
    const long long j = j0 + tid;
    int r = 0;
    int32_t x0 = -1;
    bool ok = false;
    if (j < C0) {
      int lo = 0, hi = nrows;  // largest r with pref[r] <= j
      while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (L.pref[mid] <= j) lo = mid;
        else hi = mid;
      }
      r = lo;
      x0 = __ldg(adj + __ldg(off + L.anc[r]) + (j - L.pref[r]));
      ++my_cand;
      ok = accept(st, 0, L.rows + r * w, w, 0, x0, L.acol[r], off, adj, my_probe);
    }
    if (st.n_new == 1) {
      emit(ok, r, x0, -1);
      continue;
    }
    // second new vertex: candidate space over this round's accepted first vertices
    long long d1 = 0;
    if (ok) {
      int32_t av;
      int64_t ad;
      L.aacol[tid] = pick_anchor(st, 1, L.rows + r * w, w, x0, off, av, ad);
      L.aav[tid] = av;
      L.ar[tid] = r;
      L.ax0[tid] = x0;
      d1 = ad;
    }
    long long p1, C1;
    ScanLL(tmp.ll).ExclusiveSum(d1, p1, C1);
    L.apref[tid] = p1;
    __syncthreads();
    for (long long q0 = 0; q0 < C1; q0 += kStepThreads) {
      const long long q = q0 + tid;
      int ra = 0;
      int32_t xa = -1, x1 = -1;
      bool ok1 = false;
      if (q < C1) {
        int lo = 0, hi = kStepThreads;  // largest t with apref[t] <= q
        while (hi - lo > 1) {
          int mid = (lo + hi) >> 1;
          if (L.apref[mid] <= q) lo = mid;
          else hi = mid;
        }
        ra = L.ar[lo];
        xa = L.ax0[lo];
        x1 = __ldg(adj + __ldg(off + L.aav[lo]) + (q - L.apref[lo]));
        ++my_cand;
        ok1 = accept(st, 1, L.rows + ra * w, w, xa, x1, L.aacol[lo], off, adj, my_probe);
      }
      emit(ok1, ra, xa, x1);
    }
    __syncthreads();  // second-vertex arrays are rewritten next round
  }

  // ---- 4. finish
  if (MODE == kModeWrite) {
    __syncthreads();
    flush_rows(L, w, W, fill, io.out, base);
    return;
  }
  if (io.stats) {
    unsigned long long tc = RedU(tmp.r).Sum((unsigned long long)my_cand);
    __syncthreads();
    unsigned long long tp = RedU(tmp.r).Sum((unsigned long long)my_probe);
    __syncthreads();
    if (tid == 0) {
      atomicAdd(io.stats, tc);
      atomicAdd(io.stats + 1, tp);
    }
  }
  if (MODE == kModeCount) {
    unsigned long long t = RedU(tmp.r).Sum(my_surv);
    if (tid == 0) {
      if (io.block_cnt) io.block_cnt[tile] = t;
      if (io.total) atomicAdd(io.total, t);
    }
    return;
  }
  // kModeSingle: decoupled look-back for the tile's exclusive prefix
  if (tid == 0) {
    unsigned long long excl = 0;
    if (tile == 0) {
      st_volatile(io.status, kFlagPrefix | (unsigned long long)agg);
    } else {
      st_volatile(io.status + tile, kFlagAgg | (unsigned long long)agg);
      int64_t p = tile - 1;
      while (true) {
        unsigned long long v = ld_volatile(io.status + p);
        if (v == 0) continue;  // predecessor not published yet (dynamic ids: it is resident)
        excl += v & kValueMask;
        if (v & kFlagPrefix) break;
        --p;
      }
      st_volatile(io.status + tile, kFlagPrefix | (excl + (unsigned long long)agg));
    }
    atomicAdd(io.ctrl + 2, (unsigned long long)agg);
    const bool fits = !ovf && excl + (unsigned long long)agg <= io.cap;
    if (!fits) atomicMin(io.ctrl + 1, (unsigned long long)tile);
    s_bc = fits ? excl : ~0ull;
  }
  __syncthreads();
  if (s_bc != ~0ull) flush_rows(L, w, W, fill, io.out, (int64_t)s_bc);
}

// exclusive prefix over tiles from the look-back status words: excl[t] = inclusive[t-1]
__global__ void k_status_to_excl(const unsigned long long *__restrict__ status, int64_t tiles,
                                 uint64_t *__restrict__ excl) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t <= tiles;
       t += (int64_t)gridDim.x * blockDim.x)
    excl[t] = t == 0 ? 0 : (status[t - 1] & kValueMask);
}

// Raise the dynamic shared-memory limit of a kernel once per (device, kernel) growth.
cudaError_t prep(const void *fn, int which, size_t smem) {
  static std::mutex mu;
  static size_t configured[64][3] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 64 && configured[dev][which] >= smem) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess && dev < 64) configured[dev][which] = smem;
  return e;
}

template <int MODE>
cudaError_t launch(const DevStep &st, const StepIO &io, const dm_graph &g, int64_t num_tiles,
                   cudaStream_t s) {
  if (num_tiles <= 0) return cudaSuccess;
  size_t smem = smem_bytes(st.in_w, MODE != kModeCount);
  cudaError_t e = prep((const void *)k_step<MODE>, MODE, smem);
  if (e != cudaSuccess) return e;
  k_step<MODE><<<(unsigned)num_tiles, kStepThreads, smem, s>>>(st, io, g.d_off, g.d_adj);
  return cudaGetLastError();
}

}  // namespace

size_t step_smem_bytes(int in_w, bool write_pass) { return smem_bytes(in_w, write_pass); }

cudaError_t launch_step_count(const DevStep &st, const StepIO &io, const dm_graph &g,
                              int64_t num_tiles, cudaStream_t s) {
  return launch<kModeCount>(st, io, g, num_tiles, s);
}

cudaError_t launch_step_write(const DevStep &st, const StepIO &io, const dm_graph &g,
                              int64_t num_tiles, cudaStream_t s) {
  return launch<kModeWrite>(st, io, g, num_tiles, s);
}

cudaError_t launch_step_single(const DevStep &st, const StepIO &io, const dm_graph &g,
                               int64_t num_tiles, cudaStream_t s) {
  return launch<kModeSingle>(st, io, g, num_tiles, s);
}

cudaError_t launch_status_to_excl(const unsigned long long *status, int64_t tiles, uint64_t *excl,
                                  cudaStream_t s) {
  int64_t b = (tiles + 1 + 255) / 256;
  if (b < 1) b = 1;
  if (b > 2048) b = 2048;
  k_status_to_excl<<<(unsigned)b, 256, 0, s>>>(status, tiles, excl);
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
