// extend_common.cuh -- device helpers shared by the join-step kernels (extend.cu, tail.cu,
// pairs.cu): key lookups and closing-edge probes on the sorted CSR / ELL adjacency, the
// all-distinct row test, tile loads (TMA bulk copy / cp.async / 16-bit widening), CTA counters.
#pragma once
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
// NQ > 0: ws == 4*NQ known at compile time (the 16-bit widening then divides by a constant)
template <int NQ = 0>
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
    const int nq8 = NQ > 0 ? (NQ + 1) / 2 : s16 >> 3;
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

// tail2 = the row's last two columns: compared before the Bloom test because the anchor's
// predecessors (always in its list) sit there for path-like joins -- a certain Bloom hit and
// exact scan otherwise
template <int NQ>
__device__ __forceinline__ bool accept_ell(const DevStep &st, int j, const int32_t *row, int w,
                                           int ws, unsigned long long bloom, int2 tail2,
                                           int32_t x0, int32_t x, int acol,
                                           const int4 *__restrict__ ell, uint32_t &probes) {
  if (j == 1 && x == x0) return false;
  if (x == tail2.x || x == tail2.y) return false;
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


__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }
__host__ __device__ inline long long ntiles_of(const StepIO &io) {
  return (io.in_rows + kTileRows - 1) / kTileRows;
}

// Raise the dynamic shared-memory limit (and prefer the maximum carveout) of a kernel once per
// (device, kernel) growth.  `which` is unused (kept for call-site readability).
// carveout: preferred shared-memory share of the unified L1/shared array in percent (100 = as
// much shared memory as possible; lower leaves the rest to L1).
cudaError_t prep(const void *fn, int which, size_t smem, int carveout = 100) {
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
  if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
  if (e == cudaSuccess) configured[key] = smem;
  return e;
}

}  // namespace
}  // namespace dm
