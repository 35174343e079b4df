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
//   1. tile -> shared memory with one TMA bulk copy (cp.async.bulk + mbarrier); frontier rows
//      are stored with a 16-byte stride (row_stride(w) words, padding = -1), so every row is
//      int4-aligned: LDS.128 all-distinct tests and STG.128 row writes;
//   2. per row: join key (anchor) of the first new vertex, candidate count = its degree; CTA
//      exclusive scan -> the tile's candidate space (a hub row is spread over the CTA); each
//      round maps candidates to rows by scattering segment starts + a max-scan;
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

#include <map>
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

// x in row?  The row is 16-byte aligned and padded with -1 to a multiple of 4 words, so the
// all-distinct test is ws/4 LDS.128 + predicated compares, branch-free.  In shared memory the
// rows sit at an odd number of 16-byte chunks (smem_stride), so the LDS.128 of 8 consecutive
// rows hit 8 distinct bank groups (conflict-free).
__device__ __forceinline__ bool in_row(const int32_t *row, int ws, int32_t x) {
  const int4 *r4 = reinterpret_cast<const int4 *>(row);
  const int nq = ws >> 2;
  bool hit = false;
#pragma unroll 4
  for (int q = 0; q < nq; ++q) {
    const int4 v = r4[q];
    hit |= (v.x == x) | (v.y == x) | (v.z == x) | (v.w == x);
  }
  return hit;
}

// compile-time width variant (NQ = ws/4 chunks, fully unrolled; NQ == 0 -> runtime loop)
template <int NQ>
__device__ __forceinline__ bool in_row_q(const int32_t *row, int ws, int32_t x) {
  if (NQ == 0) return in_row(row, ws, x);
  const int4 *r4 = reinterpret_cast<const int4 *>(row);
  bool hit = false;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int4 v = r4[q];
    hit |= (v.x == x) | (v.y == x) | (v.z == x) | (v.w == x);
  }
  return hit;
}

// shared-memory row stride (words): the global stride padded to an odd number of int4 chunks
__host__ __device__ inline int smem_stride(int w) {
  const int ws = row_stride(w);
  return ((ws >> 2) & 1) ? ws : ws + 4;
}

// cp.async 16-byte copy global -> shared (LDGSTS), for tiles whose smem stride differs
__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
  unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
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


// Tile of nrows frontier rows -> shared memory at stride ss.  Contiguous case (ss == ws): one
// TMA bulk copy completing on an mbarrier; padded case: 16-byte cp.async per chunk, one warp
// per row.  Implicit seed: row r = vertex seed_base + r0 + r.  Ends with a CTA barrier.
__device__ __forceinline__ void load_tile(int32_t *rows, int ss, int ws, const StepIO &io,
                                          int64_t r0, int nrows, uint64_t *bar) {
  const int tid = threadIdx.x;
  if (!io.in) {
    for (int r = tid; r < nrows; r += kStepThreads) {
      int4 *d = reinterpret_cast<int4 *>(rows + r * ss);
      d[0] = make_int4((int32_t)(io.seed_base + r0 + r), -1, -1, -1);
    }
    __syncthreads();
    return;
  }
  if (io.elem == 2) {  // 16-bit rows: 16-byte loads of 8 ids, widened to int32 in shared memory
    const int s16 = row_stride16(ws > 0 ? ws : 1);  // ws is row_stride(w); chunks of 8 ids
    const int nq8 = s16 >> 3;
    const uint4 *src16 = reinterpret_cast<const uint4 *>(
        reinterpret_cast<const uint16_t *>(io.in) + (int64_t)r0 * s16);
    const int total = nrows * nq8;  // chunks of the tile are contiguous in global memory
    for (int i0 = 0; i0 < total; i0 += 4 * kStepThreads) {
      uint4 v[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {  // issue all loads first (memory-level parallelism)
        const int i = i0 + k * kStepThreads + tid;
        v[k] = i < total ? __ldcs(src16 + i) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int i = i0 + k * kStepThreads + tid;
        if (i >= total) break;
        const int r = i / nq8, q = i - r * nq8;
        const uint32_t u[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
        int32_t o[8];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const uint32_t lo = u[t] & 0xffffu, hi = u[t] >> 16;
          o[2 * t] = lo == 0xffffu ? -1 : (int32_t)lo;
          o[2 * t + 1] = hi == 0xffffu ? -1 : (int32_t)hi;
        }
        // chunk q covers ids [8q, 8q+8); smem rows hold ss >= ws int32 words (ws multiple of 4)
        int32_t *d = rows + r * ss + 8 * q;
        if (8 * q < ws) reinterpret_cast<int4 *>(d)[0] = make_int4(o[0], o[1], o[2], o[3]);
        if (8 * q + 4 < ws) reinterpret_cast<int4 *>(d)[1] = make_int4(o[4], o[5], o[6], o[7]);
      }
    }
    __syncthreads();
    return;
  }
  const int32_t *src = io.in + r0 * ws;
  if (ss == ws) {
    if (tid == 0) {
      mbar_init(bar, 1);
      const unsigned bytes = (unsigned)(nrows * ws) * 4u;
      mbar_expect_tx(bar, bytes);
      tma_bulk_g2s(rows, src, bytes, bar);
    }
    __syncthreads();  // barrier initialised before anyone waits on it
    mbar_wait(bar, 0);
    return;
  }
  const int nq = ws >> 2;
  const int lane = tid & 31, warp = tid >> 5;
  int lpr = 1;
  while (lpr < nq) lpr <<= 1;
  const int rpi = 32 / lpr, q = lane & (lpr - 1), sub = lane / lpr;
  if (q < nq)
    for (int r = warp * rpi + sub; r < nrows; r += (kStepThreads / 32) * rpi)
      cp_async16(rows + r * ss + 4 * q, src + (int64_t)r * ws + 4 * q);
  cp_async_wait_all();
  __syncthreads();
}


// CTA-wide sum of three counters (result valid in thread 0)
__device__ __forceinline__ void block_sum3(unsigned long long v[3]) {
  __shared__ unsigned long long part[kStepThreads / 32][3];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
  if (lane == 0)
    for (int i = 0; i < 3; ++i) part[warp][i] = v[i];
  __syncthreads();
  if (threadIdx.x == 0)
    for (int i = 0; i < 3; ++i) {
      unsigned long long t = 0;
      for (int k = 0; k < kStepThreads / 32; ++k) t += part[k][i];
      v[i] = t;
    }
}

// value of column c of the row being built (c == w -> first new vertex)
__device__ __forceinline__ int32_t colval(const int32_t *row, int w, int c, int32_t x0) {
  return c < w ? row[c] : x0;
}

// Filters for new vertex j with candidate value x (anchor column `acol` is satisfied by
// construction): all-distinct, closing-edge probes, induced non-edge probes.
template <int NQ = 0>
__device__ __forceinline__ bool accept(const DevStep &st, int j, const int32_t *row, int w, int ws,
                                       int32_t x0, int32_t x, int acol,
                                       const int64_t *__restrict__ off,
                                       const int32_t *__restrict__ adj, uint32_t &probes) {
  if (in_row_q<NQ>(row, ws, x)) return false;
  if (j == 1 && x == x0) return false;
  if (st.n_nbr[j] <= 1 && st.n_non[j] == 0) return true;  // the anchor is the only key
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

// 64-bit Bloom filter of a row's vertex set: a candidate whose bit is clear cannot be in the
// row; only set bits pay for the exact LDS.128 scan
__device__ __forceinline__ unsigned long long bloom_bit(int32_t v) {
  return 1ull << (((uint32_t)v * 0x9E3779B1u) >> 26);
}

// ---- ELL (max degree <= 4) variants: a vertex's whole sorted neighbour list is one int4
__device__ __forceinline__ int4 ell_row(const int4 *__restrict__ ell, int32_t v) { return __ldg(ell + v); }
__device__ __forceinline__ int ell_deg(const int4 &e) {
  return (e.x >= 0) + (e.y >= 0) + (e.z >= 0) + (e.w >= 0);
}
__device__ __forceinline__ int32_t ell_at(const int4 &e, int i) {
  return i == 0 ? e.x : (i == 1 ? e.y : (i == 2 ? e.z : e.w));
}
__device__ __forceinline__ bool ell_has(const int4 *__restrict__ ell, int32_t u, int32_t x) {
  const int4 e = ell_row(ell, u);
  return (e.x == x) | (e.y == x) | (e.z == x) | (e.w == x);
}

// key column with the smallest-degree image for new vertex j; returns its ELL row in `nb`
__device__ __forceinline__ int pick_anchor_ell(const DevStep &st, int j, const int32_t *row, int w,
                                               int32_t x0, const int4 *__restrict__ ell, int4 &nb) {
  int best = st.nbr[j][0];
  nb = ell_row(ell, colval(row, w, best, x0));
  if (st.n_nbr[j] == 1) return best;
  int bd = ell_deg(nb);
  for (int t = 1; t < st.n_nbr[j]; ++t) {
    const int c = st.nbr[j][t];
    const int4 e = ell_row(ell, colval(row, w, c, x0));
    const int d = ell_deg(e);
    if (d < bd) {
      bd = d;
      nb = e;
      best = c;
    }
  }
  return best;
}

template <int NQ>
__device__ __forceinline__ bool accept_ell(const DevStep &st, int j, const int32_t *row, int w,
                                           int ws, unsigned long long bloom, int32_t x0, int32_t x,
                                           int acol, const int4 *__restrict__ ell,
                                           uint32_t &probes) {
  if (j == 1 && x == x0) return false;
  if ((bloom & bloom_bit(x)) && in_row_q<NQ>(row, ws, x)) return false;
  if (st.n_nbr[j] <= 1 && st.n_non[j] == 0) return true;
  for (int t = 0; t < st.n_nbr[j]; ++t) {
    const int c = st.nbr[j][t];
    if (c == acol) continue;
    ++probes;
    if (!ell_has(ell, colval(row, w, c, x0), x)) return false;
  }
  for (int t = 0; t < st.n_non[j]; ++t) {
    ++probes;
    if (ell_has(ell, colval(row, w, st.non[j][t], x0), x)) return false;
  }
  return true;
}


// ---- depth-first enumeration of a 3-4 vertex count-only last step (ELL graphs): the larger
// motif joins of PAPER.md §3.5 executed per row without materializing the levels
__device__ __forceinline__ int32_t colval4(const int32_t *row, int w, int c, const int32_t (&x)[kMaxNew]) {
  const int k = c - w;
  return k < 0 ? row[c] : (k == 0 ? x[0] : (k == 1 ? x[1] : (k == 2 ? x[2] : x[3])));
}

template <int J, int NQ>
__device__ __forceinline__ unsigned dfs_ell(const DevStep &st, const int32_t *row, int w, int ws,
                                            unsigned long long bloom, int32_t (&x)[kMaxNew],
                                            const int4 *__restrict__ ell, uint32_t &cand,
                                            uint32_t &probes) {
  if constexpr (J >= kMaxNew) {
    return 1u;
  } else {
    if (J >= st.n_new) return 1u;
    int best = st.nbr[J][0];
    int4 nb = ell_row(ell, colval4(row, w, best, x));
    const bool extra = st.n_nbr[J] > 1 || st.n_non[J] > 0;
    if (st.n_nbr[J] > 1) {
      int bd = ell_deg(nb);
      for (int t = 1; t < st.n_nbr[J]; ++t) {
        const int c = st.nbr[J][t];
        const int4 e = ell_row(ell, colval4(row, w, c, x));
        const int d = ell_deg(e);
        if (d < bd) {
          bd = d;
          nb = e;
          best = c;
        }
      }
    }
    unsigned tot = 0;
#pragma unroll 1
    for (int i = 0; i < 4; ++i) {
      const int32_t y = nb.x;  // candidates in ascending order: shift the int4 down
      nb.x = nb.y;
      nb.y = nb.z;
      nb.z = nb.w;
      nb.w = -1;
      if (y < 0) break;
      ++cand;
      bool ok = true;
#pragma unroll
      for (int t = 0; t < J; ++t) ok &= x[t] != y;  // distinct from the other new vertices
      if (!ok) continue;
      if ((bloom & bloom_bit(y)) && in_row_q<NQ>(row, ws, y)) continue;  // ... and from the row
      if (extra) {
        for (int t = 0; t < st.n_nbr[J] && ok; ++t) {
          const int c = st.nbr[J][t];
          if (c == best) continue;
          ++probes;
          ok = ell_has(ell, colval4(row, w, c, x), y);
        }
        for (int t = 0; t < st.n_non[J] && ok; ++t) {
          ++probes;
          ok = !ell_has(ell, colval4(row, w, st.non[J][t], x), y);
        }
        if (!ok) continue;
      }
      x[J] = y;
      tot += dfs_ell<J + 1, NQ>(st, row, w, ws, bloom, x, ell, cand, probes);
    }
    return tot;
  }
}

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }
__host__ __device__ inline long long ntiles_of(const StepIO &io) {
  return (io.in_rows + kTileRows - 1) / kTileRows;
}

struct SmemLayout {
  int32_t *rows;     // [kTileRows][ws] the tile exactly as stored in global memory
  long long *pref;   // [kTileRows+1]  first-vertex candidate prefix (pref[nrows] = C0)
  long long *abeg;   // [kTileRows]    CSR start of the first-vertex anchor's list
  int32_t *acol;     // [kTileRows]    first-vertex anchor column
  int32_t *owner;    // [kStepThreads] candidate -> row / entry map of the current round
  long long *apref;  // [kStepThreads+1] second-vertex candidate prefix (per round)
  long long *aabeg;  // [kStepThreads] CSR start of the second-vertex anchor's list
  int32_t *ar;       // [kStepThreads] row of the accepted first vertex
  int32_t *ax0;      // [kStepThreads] accepted first vertex
  int32_t *aacol;    // [kStepThreads] second-vertex anchor column
  int32_t *sv_row;   // [kSurvBuf]
  int32_t *sv_x;     // [kSurvBuf][2]
};

__host__ __device__ inline size_t smem_bytes(int in_w, bool stage) {
  size_t b = align16(sizeof(int32_t) * (size_t)kTileRows * smem_stride(in_w));
  b += align16(sizeof(long long) * (kTileRows + 1));
  b += align16(sizeof(long long) * kTileRows);
  b += align16(sizeof(int32_t) * kTileRows);
  b += align16(sizeof(int32_t) * kStepThreads);
  b += align16(sizeof(long long) * (kStepThreads + 1));
  b += align16(sizeof(long long) * kStepThreads);
  b += 3 * align16(sizeof(int32_t) * kStepThreads);
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
  L.rows = reinterpret_cast<int32_t *>(take(sizeof(int32_t) * (size_t)kTileRows * smem_stride(in_w)));
  L.pref = reinterpret_cast<long long *>(take(sizeof(long long) * (kTileRows + 1)));
  L.abeg = reinterpret_cast<long long *>(take(sizeof(long long) * kTileRows));
  L.acol = reinterpret_cast<int32_t *>(take(sizeof(int32_t) * kTileRows));
  L.owner = reinterpret_cast<int32_t *>(take(sizeof(int32_t) * kStepThreads));
  L.apref = reinterpret_cast<long long *>(take(sizeof(long long) * (kStepThreads + 1)));
  L.aabeg = reinterpret_cast<long long *>(take(sizeof(long long) * kStepThreads));
  L.ar = reinterpret_cast<int32_t *>(take(sizeof(int32_t) * kStepThreads));
  L.ax0 = reinterpret_cast<int32_t *>(take(sizeof(int32_t) * kStepThreads));
  L.aacol = reinterpret_cast<int32_t *>(take(sizeof(int32_t) * kStepThreads));
  if (stage) {
    L.sv_row = reinterpret_cast<int32_t *>(take(sizeof(int32_t) * kSurvBuf));
    L.sv_x = reinterpret_cast<int32_t *>(take(sizeof(int32_t) * 2 * kSurvBuf));
  } else {
    L.sv_row = L.sv_x = nullptr;
  }
  return L;
}

// Write `fill` staged survivors as rows [base, base+fill) of out (row stride Wp = stride(W)).
// A row is Wp/4 int4 chunks; lpr lanes (power of two >= Wp/4) cover one row, so one warp
// store instruction writes 32/lpr consecutive rows = a contiguous, 16-byte aligned span.
// The new vertices are patched into the chunk that holds columns w, w+1.
// map == nullptr: staged entry o is (sv_row[o], sv_x[2o], sv_x[2o+1]); otherwise map[o] =
// (row << 4 | i) names slot row*S + i of the per-row slots (row-serial kernel).
__device__ __forceinline__ void flush_rows(const int32_t *rows, const int32_t *sv_row,
                                           const int32_t *sv_x, const int32_t *map, int S, int w,
                                           int n_new, int fill, int32_t *__restrict__ out,
                                           int64_t base) {
  const int ws = row_stride(w), ss = smem_stride(w), Wp = row_stride(w + n_new);
  const int nq = Wp >> 2, nqs = ws >> 2;
  int lpr = 1;
  while (lpr < nq) lpr <<= 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = kStepThreads / 32;
  const int q = lane & (lpr - 1);
  const int rpi = 32 / lpr;
  const int sub = lane / lpr;
  if (q >= nq) return;
  const int c0 = q << 2;
  const int k0 = w - c0, k1 = w + 1 - c0;  // component index of x0 / x1 in this chunk
  const bool has0 = k0 >= 0 && k0 < 4, has1 = n_new == 2 && k1 >= 0 && k1 < 4;
  int4 *out4 = reinterpret_cast<int4 *>(out);
  for (int o = warp * rpi + sub; o < fill; o += nwarps * rpi) {
    int s, r;
    if (map) {
      const int m = map[o];
      r = m >> 4;
      s = r * S + (m & 15);
    } else {
      s = o;
      r = sv_row[o];
    }
    int4 v = q < nqs ? reinterpret_cast<const int4 *>(rows + r * ss)[q] : make_int4(-1, -1, -1, -1);
    if (has0) {
      const int32_t x0 = sv_x[2 * s];
      v.x = k0 == 0 ? x0 : v.x;
      v.y = k0 == 1 ? x0 : v.y;
      v.z = k0 == 2 ? x0 : v.z;
      v.w = k0 == 3 ? x0 : v.w;
    }
    if (has1) {
      const int32_t x1 = sv_x[2 * s + 1];
      v.x = k1 == 0 ? x1 : v.x;
      v.y = k1 == 1 ? x1 : v.y;
      v.z = k1 == 2 ? x1 : v.z;
      v.w = k1 == 3 ? x1 : v.w;
    }
    out4[(base + o) * nq + q] = v;
  }
}


// 16-bit variant of the survivor flush: lanes -> (output row, 8-id chunk); each lane reads the
// parent ids from the int32 smem row, patches the new vertices, packs to uint16 and stores 16 B.
__device__ __forceinline__ int32_t pick8(const int4 &a, const int4 &b, int i) {
  return i < 4 ? (i == 0 ? a.x : i == 1 ? a.y : i == 2 ? a.z : a.w)
               : (i == 4 ? b.x : i == 5 ? b.y : i == 6 ? b.z : b.w);
}

__device__ __forceinline__ void flush_rows16(const int32_t *rows, const int32_t *sv_x,
                                             const int32_t *map, int S, int w, int n_new,
                                             int fill, int32_t *__restrict__ out, int64_t base) {
  const int ws = row_stride(w), ss = smem_stride(w);
  const int nq = row_stride16(w + n_new) >> 3;
  int lpr = 1;
  while (lpr < nq) lpr <<= 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = kStepThreads / 32;
  const int q = lane & (lpr - 1), rpi = 32 / lpr, sub = lane / lpr;
  if (q >= nq) return;
  uint4 *out16 = reinterpret_cast<uint4 *>(out);
  const int c0 = 8 * q;
  const bool tail = c0 + 8 > w;  // chunk holds column w or w+1 (or padding)
  for (int o = warp * rpi + sub; o < fill; o += nwarps * rpi) {
    const int m = map[o];
    const int r = m >> 4, sl = r * S + (m & 15);
    const int32_t *prow = rows + r * ss;
    const int4 neg = make_int4(-1, -1, -1, -1);
    const int4 a = c0 < ws ? reinterpret_cast<const int4 *>(prow + c0)[0] : neg;
    const int4 b = c0 + 4 < ws ? reinterpret_cast<const int4 *>(prow + c0 + 4)[0] : neg;
    int32_t x0 = -1, x1 = -1;
    if (tail) {
      x0 = sv_x[2 * sl];
      x1 = sv_x[2 * sl + 1];
    }
    uint32_t packed[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      int32_t lo = pick8(a, b, 2 * t), hi = pick8(a, b, 2 * t + 1);
      const int cl = c0 + 2 * t, ch = cl + 1;
      if (tail) {
        lo = cl == w ? x0 : ((cl == w + 1 && n_new == 2) ? x1 : (cl >= w ? -1 : lo));
        hi = ch == w ? x0 : ((ch == w + 1 && n_new == 2) ? x1 : (ch >= w ? -1 : hi));
      }
      packed[t] = ((uint32_t)lo & 0xffffu) | ((uint32_t)hi << 16);
    }
    out16[(base + o) * nq + q] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
  }
}

__device__ __forceinline__ unsigned long long ld_volatile(const unsigned long long *p) {
  return *reinterpret_cast<const volatile unsigned long long *>(p);
}
__device__ __forceinline__ void st_volatile(unsigned long long *p, unsigned long long v) {
  *reinterpret_cast<volatile unsigned long long *>(p) = v;
}

// Decoupled look-back by warp 0: publish the tile aggregate, then scan 32 predecessors at a
// time (ballot for the nearest inclusive prefix); returns the exclusive prefix to all lanes.
__device__ unsigned long long lookback(unsigned long long *status, int64_t tile,
                                       unsigned long long agg) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) st_volatile(status, kFlagPrefix | agg);
    return 0;
  }
  if (lane == 0) st_volatile(status + tile, kFlagAgg | agg);
  unsigned long long excl = 0;
  int64_t hi = tile - 1;
  while (true) {
    const int64_t p = hi - lane;
    const unsigned long long v = p >= 0 ? ld_volatile(status + p) : kFlagPrefix;
    const unsigned pm = __ballot_sync(0xffffffffu, (v & kFlagPrefix) != 0);
    const unsigned zm = __ballot_sync(0xffffffffu, v == 0);
    const int fp = pm ? __ffs(pm) - 1 : 31;  // lanes 0..fp are needed
    const unsigned need = fp >= 31 ? 0xffffffffu : ((1u << (fp + 1)) - 1u);
    if (zm & need) continue;  // a needed predecessor has not published yet: re-read
    unsigned long long val = lane <= fp ? (v & kValueMask) : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
    excl += val;
    if (pm) break;
    hi -= 32;
  }
  if (lane == 0) st_volatile(status + tile, kFlagPrefix | (excl + agg));
  return excl;
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
  const int ws = row_stride(w);
  const int ss = smem_stride(w);
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

  // ---- 1. tile -> shared memory
  load_tile(L.rows, ss, ws, io, r0, nrows, &s_bar);

  // ---- 2. per-row join key for the first new vertex; tile candidate space
  long long cnt = 0;
  if (tid < nrows) {
    int32_t av;
    int64_t ad;
    L.acol[tid] = pick_anchor(st, 0, L.rows + tid * ss, w, 0, off, av, ad);
    L.abeg[tid] = __ldg(off + av);
    cnt = ad;
  }
  long long pref, C0;
  ScanLL(tmp.ll).ExclusiveSum(cnt, pref, C0);
  L.pref[tid] = pref;
  if (tid == 0) L.pref[nrows] = C0;
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
      flush_rows(L.rows, L.sv_row, L.sv_x, nullptr, 0, w, st.n_new, fill, io.out, base);
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

  // owner[t] = index i of the segment [pref[i], pref[i+1]) that holds candidate j0 + t:
  // segment starts are scattered, then an inclusive max-scan fills the gaps.
  auto map_round = [&](const long long *pf, int nseg, long long j0) {
    L.owner[tid] = -1;
    __syncthreads();
    if (tid < nseg) {
      const long long b = pf[tid], e = pf[tid + 1];
      if (e > b && e > j0 && b < j0 + kStepThreads) L.owner[(b > j0 ? b : j0) - j0] = tid;
    }
    __syncthreads();
    int o = L.owner[tid];
    ScanI(tmp.i).InclusiveScan(o, o, cub::Max());
    __syncthreads();
    return o;
  };

  // ---- 3. candidate rounds
  for (long long j0 = 0; j0 < C0; j0 += kStepThreads) {
    const long long j = j0 + tid;
    const int r = map_round(L.pref, nrows, j0);
    int32_t x0 = -1;
    bool ok = false;
    if (j < C0) {
      x0 = __ldg(adj + L.abeg[r] + (j - L.pref[r]));
      ++my_cand;
      ok = accept(st, 0, L.rows + r * ss, w, ws, 0, x0, L.acol[r], off, adj, my_probe);
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
      L.aacol[tid] = pick_anchor(st, 1, L.rows + r * ss, w, x0, off, av, ad);
      L.aabeg[tid] = __ldg(off + av);
      L.ar[tid] = r;
      L.ax0[tid] = x0;
      d1 = ad;
    }
    long long p1, C1;
    ScanLL(tmp.ll).ExclusiveSum(d1, p1, C1);
    L.apref[tid] = p1;
    if (tid == 0) L.apref[kStepThreads] = C1;
    __syncthreads();
    for (long long q0 = 0; q0 < C1; q0 += kStepThreads) {
      const long long q = q0 + tid;
      const int t = map_round(L.apref, kStepThreads, q0);
      int ra = 0;
      int32_t xa = -1, x1 = -1;
      bool ok1 = false;
      if (q < C1) {
        ra = L.ar[t];
        xa = L.ax0[t];
        x1 = __ldg(adj + L.aabeg[t] + (q - L.apref[t]));
        ++my_cand;
        ok1 = accept(st, 1, L.rows + ra * ss, w, ws, xa, x1, L.aacol[t], off, adj, my_probe);
      }
      emit(ok1, ra, xa, x1);
    }
    __syncthreads();  // second-vertex arrays are rewritten next round
  }

  // ---- 4. finish
  if (MODE == kModeWrite) {
    __syncthreads();
    flush_rows(L.rows, L.sv_row, L.sv_x, nullptr, 0, w, st.n_new, fill, io.out, base);
    return;
  }
  if (io.stats || MODE == kModeCount) {
    unsigned long long v3[3] = {my_cand, my_probe, my_surv};
    block_sum3(v3);
    if (tid == 0) {
      const int slot = (int)(tile & (kAccSlots - 1));
      if (io.stats) {
        atomicAdd(io.stats + slot, v3[0]);
        atomicAdd(io.stats + kAccSlots + slot, v3[1]);
      }
      if (MODE == kModeCount) {
        if (io.block_cnt) io.block_cnt[tile] = v3[2];
        if (io.total && v3[2]) atomicAdd(io.total + slot, v3[2]);
      }
    }
  }
  if (MODE == kModeCount) return;
  // kModeSingle: decoupled look-back for the tile's exclusive prefix, then write
  if (tid < 32) {
    const unsigned long long excl = lookback(io.status, tile, (unsigned long long)agg);
    if (tid == 0) {
      atomicAdd(io.ctrl + 2, (unsigned long long)agg);
      const bool fits = !ovf && excl + (unsigned long long)agg <= io.cap;
      if (!fits) atomicMax(io.ctrl + 1, (unsigned long long)(ntiles_of(io) - tile));
      s_bc = fits ? excl : ~0ull;
    }
  }
  __syncthreads();
  if (s_bc != ~0ull) flush_rows(L.rows, L.sv_row, L.sv_x, nullptr, 0, w, st.n_new, fill, io.out, (int64_t)s_bc);
}


// ---------------------------------------------------------------------------------------
// Row-serial variant for low-degree data graphs (lattices: max degree <= kRowSerialDeg):
// thread = frontier row; the thread walks its join candidates (CSR range of the anchor key,
// then of the second new vertex's key) serially, so a tile needs one CTA scan instead of
// per-round scans and barriers.  Survivors go to per-thread slots (kRowSlots each); a thread
// that overflows its slots marks the tile unwritten and the host re-runs it with the general
// kernel (kModeWrite).  Output order is identical to k_step (row, then candidate order).
template <int MODE, int NQ, bool ELL>
__global__ void __launch_bounds__(kStepThreads) __maxnreg__(MODE == kModeCount ? 64 : 48)
    k_rows(const DevStep st, const StepIO io, const int64_t *__restrict__ off,
           const int32_t *__restrict__ adj) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  typedef cub::BlockScan<int, kStepThreads> ScanI;
  __shared__ typename ScanI::TempStorage tmp;
  __shared__ unsigned long long s_bc;
  __shared__ __align__(8) uint64_t s_bar;
  constexpr bool kStage = MODE != kModeCount;

  const int w = st.in_w;
  const int ws = row_stride(w);
  const int ss = smem_stride(w);
  const int S = io.slots;
  const int tid = threadIdx.x, lane = tid & 31;
  int64_t tile;
  if (MODE == kModeSingle) {
    if (tid == 0) s_bc = atomicAdd(io.ctrl + 0, 1ull);
    __syncthreads();
    tile = (int64_t)s_bc;
  } else {
    tile = io.block_begin + blockIdx.x;
  }
  const int64_t r0 = tile * kTileRows;
  if (r0 >= io.in_rows) return;
  const int nrows = (int)(io.in_rows - r0 < kTileRows ? io.in_rows - r0 : kTileRows);
  int32_t *rows = reinterpret_cast<int32_t *>(smem_raw);
  int32_t *sv_x = rows + kTileRows * ss;         // [kTileRows * S][2]
  int32_t *map = sv_x + 2 * kTileRows * S;       // [kTileRows * S]

  load_tile(rows, ss, ws, io, r0, nrows, &s_bar);

  int ns = 0;
  bool ovf = false;
  uint32_t my_cand = 0, my_probe = 0;
  auto record = [&](int32_t x0, int32_t x1) {
    if (kStage) {
      if (ns < S) {
        const int sl = tid * S + ns;
        sv_x[2 * sl] = x0;
        sv_x[2 * sl + 1] = x1;
      } else {
        ovf = true;
      }
    }
    ++ns;
  };
  // all survivors of this thread's row, in candidate order
  auto enumerate = [&](auto &&on_survivor, uint32_t &n_cand, uint32_t &n_probe) {
    const int32_t *row = rows + tid * ss;
    if (ELL) {
      // max degree <= 4: candidate lists are single int4 loads (sorted, -1 padded)
      const int4 *ell = reinterpret_cast<const int4 *>(io.ell);
      unsigned long long bloom = 0;
      for (int c = 0; c < w; ++c) bloom |= bloom_bit(row[c]);
      int4 na;
      const int ac = pick_anchor_ell(st, 0, row, w, 0, ell, na);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int32_t x0 = ell_at(na, i);
        if (x0 < 0) break;
        ++n_cand;
        if (!accept_ell<NQ>(st, 0, row, w, ws, bloom, 0, x0, ac, ell, n_probe)) continue;
        if (st.n_new == 1) {
          on_survivor(x0, -1);
          continue;
        }
        int4 nb;
        const int bc = pick_anchor_ell(st, 1, row, w, x0, ell, nb);
#pragma unroll
        for (int i1 = 0; i1 < 4; ++i1) {
          const int32_t x1 = ell_at(nb, i1);
          if (x1 < 0) break;
          ++n_cand;
          if (accept_ell<NQ>(st, 1, row, w, ws, bloom, x0, x1, bc, ell, n_probe)) on_survivor(x0, x1);
        }
      }
    } else {
      int32_t av;
      int64_t ad;
      const int ac = pick_anchor(st, 0, row, w, 0, off, av, ad);
      const int64_t e0 = __ldg(off + av);
      for (int64_t e = e0; e < e0 + ad; ++e) {
        const int32_t x0 = __ldg(adj + e);
        ++n_cand;
        if (!accept<NQ>(st, 0, row, w, ws, 0, x0, ac, off, adj, n_probe)) continue;
        if (st.n_new == 1) {
          on_survivor(x0, -1);
          continue;
        }
        int32_t bv;
        int64_t bd;
        const int bc = pick_anchor(st, 1, row, w, x0, off, bv, bd);
        const int64_t f0 = __ldg(off + bv);
        for (int64_t f = f0; f < f0 + bd; ++f) {
          const int32_t x1 = __ldg(adj + f);
          ++n_cand;
          if (accept<NQ>(st, 1, row, w, ws, x0, x1, bc, off, adj, n_probe)) on_survivor(x0, x1);
        }
      }
    }
  };
  if (tid < nrows) enumerate(record, my_cand, my_probe);
  // statistics and count-mode totals: CTA reduction, one atomic per CTA on slot tile % 64
  if (io.stats || MODE == kModeCount) {
    unsigned long long v3[3] = {my_cand, my_probe, (unsigned long long)ns};
    block_sum3(v3);
    if (tid == 0) {
      const int slot = (int)(tile & (kAccSlots - 1));
      if (io.stats) {
        atomicAdd(io.stats + slot, v3[0]);
        atomicAdd(io.stats + kAccSlots + slot, v3[1]);
      }
      if (MODE == kModeCount) {
        if (io.block_cnt) io.block_cnt[tile] = v3[2];
        if (io.total && v3[2]) atomicAdd(io.total + slot, v3[2]);
      }
    }
  }
  if (MODE == kModeCount) return;
  int pos, agg;
  ScanI(tmp).ExclusiveSum(ns, pos, agg);
  const bool any_ovf = __syncthreads_or(ovf);
  if (!any_ovf)
    for (int i = 0; i < ns; ++i) map[pos + i] = (tid << 4) | i;
  if (MODE == kModeWrite) {  // re-run at an exact offset (no look-back)
    if (tid == 0) s_bc = io.block_off[tile] - io.out_base;
  } else if (tid < 32) {
    const unsigned long long excl = lookback(io.status, tile, (unsigned long long)agg);
    if (tid == 0) {
      atomicAdd(io.ctrl + 2, (unsigned long long)agg);
      const bool fits = excl + (unsigned long long)agg <= io.cap;
      if (!fits) atomicMax(io.ctrl + 1, (unsigned long long)(ntiles_of(io) - tile));
      s_bc = fits ? excl : ~0ull;
    }
  }
  __syncthreads();
  if (s_bc == ~0ull) return;
  if (!any_ovf) {
    if (io.out_elem == 2) flush_rows16(rows, sv_x, map, S, w, st.n_new, agg, io.out, (int64_t)s_bc);
    else flush_rows(rows, nullptr, sv_x, map, S, w, st.n_new, agg, io.out, (int64_t)s_bc);
    return;
  }
  // a row overflowed its slots: every thread re-enumerates its row and writes its survivors
  // directly at their final positions (same order, uncoalesced; rare)
  if (tid < nrows && ns > 0 && io.out_elem == 2) {
    const int32_t *row = rows + tid * ss;
    const int W = w + st.n_new, s16 = row_stride16(W);
    uint16_t *dst = reinterpret_cast<uint16_t *>(io.out) + ((int64_t)s_bc + pos) * s16;
    uint32_t dc = 0, dp = 0;
    enumerate(
        [&](int32_t x0, int32_t x1) {
          for (int c = 0; c < s16; ++c) {
            const int32_t v = c < w ? row[c] : (c == w ? x0 : ((c == w + 1 && st.n_new == 2) ? x1 : -1));
            dst[c] = (uint16_t)(v & 0xffff);
          }
          dst += s16;
        },
        dc, dp);
  } else if (tid < nrows && ns > 0) {
    const int32_t *row = rows + tid * ss;
    const int nq = row_stride(w + st.n_new) >> 2, nqs = ws >> 2, qw = w >> 2;
    int4 *dst = reinterpret_cast<int4 *>(io.out) + ((int64_t)s_bc + pos) * nq;
    uint32_t dc = 0, dp = 0;
    enumerate(
        [&](int32_t x0, int32_t x1) {
          for (int q = 0; q < nq; ++q) {
            int4 v = q < nqs ? reinterpret_cast<const int4 *>(row)[q] : make_int4(-1, -1, -1, -1);
            if (q == qw || q == qw + 1) {
              int32_t t4[4] = {v.x, v.y, v.z, v.w};
              for (int c = 0; c < 4; ++c) {
                const int col = 4 * q + c;
                if (col == w) t4[c] = x0;
                if (col == w + 1 && st.n_new == 2) t4[c] = x1;
              }
              v = make_int4(t4[0], t4[1], t4[2], t4[3]);
            }
            dst[q] = v;
          }
          dst += nq;
        },
        dc, dp);
  }
}


// Deep count-only last step (3-4 new vertices, ELL graphs): tile -> smem, one thread per row,
// depth-first enumeration (dfs_ell), CTA-reduced counters.
template <int NQ>
__global__ void __launch_bounds__(kStepThreads)
    k_deep(const DevStep st, const StepIO io, const int64_t *__restrict__ off,
           const int32_t *__restrict__ adj) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t s_bar;
  const int w = st.in_w, ws = row_stride(w), ss = smem_stride(w);
  const int tid = threadIdx.x;
  const int64_t tile = io.block_begin + blockIdx.x;
  const int64_t r0 = tile * kTileRows;
  if (r0 >= io.in_rows) return;
  const int nrows = (int)(io.in_rows - r0 < kTileRows ? io.in_rows - r0 : kTileRows);
  int32_t *rows = reinterpret_cast<int32_t *>(smem_raw);
  load_tile(rows, ss, ws, io, r0, nrows, &s_bar);
  uint32_t my_cand = 0, my_probe = 0;
  unsigned ns = 0;
  if (tid < nrows) {
    int32_t x[kMaxNew] = {-1, -1, -1, -1};
    const int32_t *row = rows + tid * ss;
    unsigned long long bloom = 0;
    for (int c = 0; c < w; ++c) bloom |= bloom_bit(row[c]);
    ns = dfs_ell<0, NQ>(st, row, w, ws, bloom, x, reinterpret_cast<const int4 *>(io.ell), my_cand,
                        my_probe);
  }
  unsigned long long v3[3] = {my_cand, my_probe, ns};
  block_sum3(v3);
  if (tid == 0) {
    const int slot = (int)(tile & (kAccSlots - 1));
    if (io.stats) {
      atomicAdd(io.stats + slot, v3[0]);
      atomicAdd(io.stats + kAccSlots + slot, v3[1]);
    }
    if (io.block_cnt) io.block_cnt[tile] = v3[2];
    if (io.total && v3[2]) atomicAdd(io.total + slot, v3[2]);
  }
}

size_t rows_smem_bytes(int in_w, bool stage, int slots) {
  size_t b = sizeof(int32_t) * (size_t)kTileRows * smem_stride(in_w);
  if (stage) b += sizeof(int32_t) * (size_t)kTileRows * slots * 3;
  return b;
}

// survivor slots per row for the row-serial kernel: min(max_degree^n_new, kRowSlotsMax); a row
// with more survivors makes its tile fall back to direct writes
int row_slots(const DevStep &st, const dm_graph &g) {
  int64_t d = g.max_deg < 1 ? 1 : g.max_deg;
  int64_t s = st.n_new == 1 ? d : d * d;
  return (int)(s < kRowSlotsMax ? s : kRowSlotsMax);
}


// ---------------------------------------------------------------------------------------
// Shared-key pair step (count-only last step): both new vertices have the same join keys
// (e.g. the two apexes of a diamond on an edge, or the last two vertices of a 4-clique whose
// second also keys on the first).  Per frontier row the warp computes the candidate list S of
// the first new vertex once -- the equi-join of the row with Res(M2) on every key (the anchor's
// sorted list, filtered by injectivity, the other keys' probes and induced non-edges) -- and
// then inspects every ordered pair (x0, x1) of S: x1 != x0 (all-distinct) and, when the second
// vertex also keys on the first, the closing-edge probe (x0, x1) (pair_mode 1) or the induced
// non-edge probe (pair_mode 2).  Every candidate pair is inspected (no |S|(|S|-1) shortcut).
// Persistent grid; warps claim rows in batches; S lives in shared memory (kPairSmem entries)
// or, for longer anchor lists, in a per-warp global slab of max_degree entries.
template <int NQ>
__global__ void __launch_bounds__(kStepThreads)
    k_pairs(const DevStep st, const StepIO io, const int64_t *__restrict__ off,
            const int32_t *__restrict__ adj, int32_t *__restrict__ slab, int64_t slab_cap,
            int pair_mode, unsigned long long *__restrict__ row_counter) {
  constexpr int kWarps = kStepThreads / 32;
  __shared__ __align__(16) int32_t s_row[kWarps][64];
  __shared__ int32_t s_list[kWarps][kPairSmem];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int64_t wg = (int64_t)blockIdx.x * kWarps + wl;
  int32_t *gslab = slab + wg * slab_cap;
  const int w = st.in_w, ws = row_stride(w);
  const unsigned lt = (1u << lane) - 1u;
  unsigned long long cnt = 0, cand = 0, probes = 0;
  int32_t *row = s_row[wl];
  for (;;) {
    unsigned long long b0 = 0;
    if (lane == 0) b0 = atomicAdd(row_counter, (unsigned long long)kPairBatch);
    b0 = __shfl_sync(0xffffffffu, b0, 0);
    if ((int64_t)b0 >= io.in_rows) break;
    const int64_t b1 = (int64_t)b0 + kPairBatch < io.in_rows ? (int64_t)b0 + kPairBatch : io.in_rows;
    for (int64_t r = (int64_t)b0; r < b1; ++r) {
      // row -> shared (padded with -1 to ws words)
      for (int c = lane; c < ws; c += 32)
        row[c] = io.in ? __ldg(io.in + r * ws + c) : (c == 0 ? (int32_t)(io.seed_base + r) : -1);
      __syncwarp();
      int32_t av;
      int64_t ad;
      const int ac = pick_anchor(st, 0, row, w, 0, off, av, ad);
      const int64_t e0 = __ldg(off + av);
      int32_t *S = ad <= kPairSmem ? s_list[wl] : gslab;
      // ---- S: accepted first-vertex candidates, in anchor-list (ascending) order
      int ns = 0;
      uint32_t pr = 0;
      for (int64_t i0 = 0; i0 < ad; i0 += 32) {
        const int64_t i = i0 + lane;
        bool ok = false;
        int32_t x = -1;
        if (i < ad) {
          x = __ldg(adj + e0 + i);
          ok = accept<NQ>(st, 0, row, w, ws, 0, x, ac, off, adj, pr);
        }
        const unsigned m = __ballot_sync(0xffffffffu, ok);
        if (ok) S[ns + __popc(m & lt)] = x;
        ns += __popc(m);
      }
      probes += pr;
      cand += (lane == 0) ? (unsigned long long)ad : 0ull;
      __syncwarp();
      // ---- every ordered pair of S
      const int64_t np = (int64_t)ns * ns;
      if (lane == 0 && pair_mode != 1) cand += (unsigned long long)np;
      for (int i = 0; i < ns; ++i) {
        const int32_t x0 = S[i];
        if (pair_mode == 1 && ns > 1) {
          // x1 in S with (x0, x1) in E: join S with N(x0) restricted to [S[0], S[ns-1]],
          // iterating the smaller side and binary-searching the other (S is sorted)
          const int64_t b = __ldg(off + x0), e = __ldg(off + x0 + 1);
          int64_t lo = b, hi = e;
          {
            const int32_t smin = S[0];
            int64_t l = b, h = e;
            while (l < h) {
              const int64_t m = (l + h) >> 1;
              if (__ldg(adj + m) < smin) l = m + 1;
              else h = m;
            }
            lo = l;
            const int32_t smax = S[ns - 1];
            l = lo;
            h = e;
            while (l < h) {
              const int64_t m = (l + h) >> 1;
              if (__ldg(adj + m) <= smax) l = m + 1;
              else h = m;
            }
            hi = l;
          }
          const int64_t m = hi - lo;
          if (lane == 0) cand += (unsigned long long)(m <= 2 * (int64_t)ns ? m : ns);
          if (m <= 2 * (int64_t)ns) {
            for (int64_t t = lo + lane; t < hi; t += 32) {  // N(x0) side, probe S
              const int32_t y = __ldg(adj + t);
              int l = 0, h = ns;
              while (l < h) {
                const int mid = (l + h) >> 1;
                if (S[mid] < y) l = mid + 1;
                else h = mid;
              }
              ++probes;
              cnt += (l < ns && S[l] == y);
            }
          } else {
            for (int j = lane; j < ns; j += 32) {  // S side, probe N(x0)
              const int32_t x1 = S[j];
              if (j == i) continue;
              int64_t l = lo, h = hi;
              while (l < h) {
                const int64_t mid = (l + h) >> 1;
                if (__ldg(adj + mid) < x1) l = mid + 1;
                else h = mid;
              }
              ++probes;
              cnt += (l < hi && __ldg(adj + l) == x1);
            }
          }
          continue;
        }
        for (int j = lane; j < ns; j += 32) {
          const int32_t x1 = S[j];
          bool ok = j != i;
          if (ok && pair_mode != 0) {
            ++probes;
            const bool e = has_edge(off, adj, x0, x1);
            ok = pair_mode == 1 ? e : !e;
          }
          cnt += ok;
        }
      }
      __syncwarp();
    }
  }
  unsigned long long v3[3] = {cand, probes, cnt};
  block_sum3(v3);
  if (threadIdx.x == 0) {
    const int slot = (int)(blockIdx.x & (kAccSlots - 1));
    if (io.stats) {
      atomicAdd(io.stats + slot, v3[0]);
      atomicAdd(io.stats + kAccSlots + slot, v3[1]);
    }
    if (io.total && v3[2]) atomicAdd(io.total + slot, v3[2]);
  }
}

// exclusive prefix over tiles from the look-back status words: excl[t] = inclusive[t-1]
__global__ void k_status_to_excl(const unsigned long long *__restrict__ status, int64_t tiles,
                                 uint64_t *__restrict__ excl) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t <= tiles;
       t += (int64_t)gridDim.x * blockDim.x)
    excl[t] = t == 0 ? 0 : (status[t - 1] & kValueMask);
}

// Raise the dynamic shared-memory limit (and prefer the maximum carveout) of a kernel once per
// (device, kernel) growth.  `which` is unused (kept for call-site readability).
cudaError_t prep(const void *fn, int which, size_t smem) {
  (void)which;
  static std::mutex mu;
  static std::map<std::pair<int, const void *>, size_t> configured;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_pair(dev, fn);
  auto it = configured.find(key);
  if (it != configured.end() && it->second >= smem) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e == cudaSuccess) configured[key] = smem;
  return e;
}

template <int MODE, int NQ>
cudaError_t launch_rows_nq(const DevStep &st, const StepIO &io, const dm_graph &g, int64_t tiles,
                           size_t smem, cudaStream_t s) {
  if (MODE == kModeCount && g.d_ell && st.n_new > 2) {
    StepIO io2 = io;
    io2.ell = g.d_ell;
    cudaError_t e = prep((const void *)k_deep<NQ>, 90 + NQ % 6, smem);
    if (e != cudaSuccess) return e;
    k_deep<NQ><<<(unsigned)tiles, kStepThreads, smem, s>>>(st, io2, g.d_off, g.d_adj);
    return cudaGetLastError();
  }
  if (g.d_ell) {
    StepIO io2 = io;
    io2.ell = g.d_ell;
    cudaError_t e = prep((const void *)k_rows<MODE, NQ, true>, 48 + 3 * (NQ + 1) + MODE, smem);
    if (e != cudaSuccess) return e;
    k_rows<MODE, NQ, true><<<(unsigned)tiles, kStepThreads, smem, s>>>(st, io2, g.d_off, g.d_adj);
    return cudaGetLastError();
  }
  cudaError_t e = prep((const void *)k_rows<MODE, NQ, false>, 3 * (NQ + 1) + MODE, smem);
  if (e != cudaSuccess) return e;
  k_rows<MODE, NQ, false><<<(unsigned)tiles, kStepThreads, smem, s>>>(st, io, g.d_off, g.d_adj);
  return cudaGetLastError();
}

// row-serial kernel specialised on the row width (16-byte chunks per row)
template <int MODE>
cudaError_t launch_rows(int nq, const DevStep &st, const StepIO &io, const dm_graph &g,
                        int64_t tiles, size_t smem, cudaStream_t s) {
  switch (nq) {
    case 1: return launch_rows_nq<MODE, 1>(st, io, g, tiles, smem, s);
    case 2: return launch_rows_nq<MODE, 2>(st, io, g, tiles, smem, s);
    case 3: return launch_rows_nq<MODE, 3>(st, io, g, tiles, smem, s);
    case 4: return launch_rows_nq<MODE, 4>(st, io, g, tiles, smem, s);
    case 5: return launch_rows_nq<MODE, 5>(st, io, g, tiles, smem, s);
    case 6: return launch_rows_nq<MODE, 6>(st, io, g, tiles, smem, s);
    case 7: return launch_rows_nq<MODE, 7>(st, io, g, tiles, smem, s);
    case 8: return launch_rows_nq<MODE, 8>(st, io, g, tiles, smem, s);
    default: return launch_rows_nq<MODE, 0>(st, io, g, tiles, smem, s);
  }
}

// Low-degree graphs take the row-serial kernel (count and single-pass launches); re-runs at
// exact offsets (kModeWrite) and skewed graphs take the candidate-partitioned kernel.
bool use_row_serial(const DevStep &st, const dm_graph &g) {
  return st.n_new == 1 ? g.max_deg <= kRowSerialDeg1 : g.max_deg <= kRowSerialDeg2;
}

template <int MODE>
cudaError_t launch(const DevStep &st, const StepIO &io, const dm_graph &g, int64_t num_tiles,
                   cudaStream_t s) {
  if (num_tiles <= 0) return cudaSuccess;
  if ((MODE != kModeWrite || io.elem == 2 || io.out_elem == 2) && use_row_serial(st, g)) {
    StepIO io2 = io;
    io2.slots = row_slots(st, g);
    size_t smem = rows_smem_bytes(st.in_w, MODE != kModeCount, io2.slots);
    return launch_rows<MODE>(row_stride(st.in_w) >> 2, st, io2, g, num_tiles, smem, s);
  }
  size_t smem = smem_bytes(st.in_w, MODE != kModeCount);
  cudaError_t e = prep((const void *)k_step<MODE>, MODE, smem);
  if (e != cudaSuccess) return e;
  k_step<MODE><<<(unsigned)num_tiles, kStepThreads, smem, s>>>(st, io, g.d_off, g.d_adj);
  return cudaGetLastError();
}

}  // namespace

size_t step_smem_bytes(int in_w, bool write_pass) { return smem_bytes(in_w, write_pass); }

bool row_serial_step(const DevStep &st, const dm_graph &g) { return use_row_serial(st, g); }

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

// Shared-key pair step?  Second new vertex keys on exactly the first one's keys (plus, maybe,
// the first vertex itself); returns the pair probe mode (0 none, 1 edge, 2 non-edge) or -1.
int pair_mode_of(const DevStep &st) {
  if (st.n_new != 2) return -1;
  const int w = st.in_w;
  auto same = [&](const uint8_t *a, int na, const uint8_t *b, int nb) {
    if (na != nb) return false;
    for (int i = 0; i < na; ++i) {
      bool f = false;
      for (int j = 0; j < nb; ++j) f |= a[i] == b[j];
      if (!f) return false;
    }
    return true;
  };
  uint8_t nb1[DM_MAX_PATTERN], nn1[DM_MAX_PATTERN];
  int c1 = 0, d1 = 0, mode = 0;
  for (int t = 0; t < st.n_nbr[1]; ++t) {
    if (st.nbr[1][t] == w) mode = 1;
    else nb1[c1++] = st.nbr[1][t];
  }
  for (int t = 0; t < st.n_non[1]; ++t) {
    if (st.non[1][t] == w) mode = 2;
    else nn1[d1++] = st.non[1][t];
  }
  if (!same(st.nbr[0], st.n_nbr[0], nb1, c1) || !same(st.non[0], st.n_non[0], nn1, d1)) return -1;
  return mode;
}

cudaError_t launch_pairs(const DevStep &st, const StepIO &io, const dm_graph &g, int pair_mode,
                         cudaStream_t s) {
  if (io.in_rows <= 0) return cudaSuccess;
  auto kern = k_pairs<0>;
  switch (row_stride(st.in_w) >> 2) {
    case 1: kern = k_pairs<1>; break;
    case 2: kern = k_pairs<2>; break;
    case 3: kern = k_pairs<3>; break;
    case 4: kern = k_pairs<4>; break;
    default: break;
  }
  int per_sm = 0, sms = 0, dev = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kStepThreads, 0);
  if (e != cudaSuccess) return e;
  cudaGetDevice(&dev);
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  const int64_t grid = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
  const int64_t warps = grid * (kStepThreads / 32);
  const int64_t cap = g.max_deg > kPairSmem ? g.max_deg : 1;
  int32_t *slab = nullptr;
  unsigned long long *counter = nullptr;
  e = cudaMallocAsync((void **)&slab, sizeof(int32_t) * (size_t)(warps * cap), s);
  if (e != cudaSuccess) return e;
  e = cudaMallocAsync((void **)&counter, sizeof(unsigned long long), s);
  if (e != cudaSuccess) {
    cudaFreeAsync(slab, s);
    return e;
  }
  cudaMemsetAsync(counter, 0, sizeof(unsigned long long), s);
  kern<<<(unsigned)grid, kStepThreads, 0, s>>>(st, io, g.d_off, g.d_adj, slab, cap, pair_mode, counter);
  e = cudaGetLastError();
  cudaFreeAsync(slab, s);
  cudaFreeAsync(counter, s);
  return e;
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
