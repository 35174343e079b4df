// tail.cu -- the deep count-only last step ("tail", 3-4 new vertices) of a join program on
// ELL graphs (max degree <= 4): the last joins of the program are executed per frontier row
// without materializing their levels -- the larger-motif joins of PAPER.md §3.5
// applied row by row.  Every candidate is still inspected: the all-distinct rule (P:237,
// S:213), the closing-edge probes of multi-key joins (Fig. 2 C1/C2) and, in induced
// mode, the non-edge probes.  CTA = tile of 256 rows in shared memory; thread = row; the
// recursion is unrolled at compile time (static indices into the assigned new vertices).  For a
// 3-4 vertex tail the CTA splits the recursion in two phases (k_deep_split): the first two levels
// per row, their surviving partial rows queued in shared memory, the last two levels per queue
// entry spread evenly over the threads (P30: 5.62 -> 5.16 ms).
//
// Measured alternatives (config 5, P30 on heavy-hex w=31, B200, r01): deeper tails (5-8 new
// vertices, which would skip materializing the last levels) lose -- a warp-cooperative
// breadth-first tail in shared memory ran 12.2 ms, an iterative lockstep per-thread DFS with
// row stealing 11.7 ms and an unrolled 8-deep recursion 24 ms, against 5.4 ms for this 4-deep
// tail plus 4.7 ms for materializing the two extra levels; see DESIGN.md §5.
#include <cmath>

#include "extend_common.cuh"

namespace dm {
namespace {

// ---- depth-first enumeration of a 3-4 vertex count-only last step (ELL graphs): the larger
// motif joins of PAPER.md §3.5 executed per row without materializing the levels
__device__ __forceinline__ int32_t colval4(const int32_t *row, int w, int c, const int32_t (&x)[kMaxNew]) {
  const int k = c - w;
  return k < 0 ? row[c] : (k == 0 ? x[0] : (k == 1 ? x[1] : (k == 2 ? x[2] : x[3])));
}

// Shared-memory queue of partial rows (row in tile, x_0, x_1) handed from the first two tail
// levels to the rest (split tail, n_new 3-4).
struct TailQueue {
  int *n;           // entries claimed (may exceed cap)
  int cap;
  int32_t *x0, *x1;
  uint8_t *r;
};

template <int J, int NQ, bool PUSH = false>
__device__ __forceinline__ unsigned dfs_ell(const DevStep &st, const int32_t *row, int w, int ws,
                                            unsigned long long bloom, int2 tail2,
                                            int32_t (&x)[kMaxNew],
                                            const int4 *__restrict__ ell, uint32_t &cand,
                                            uint32_t &probes, const TailQueue *q = nullptr) {
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
      // ... and from the row: the two most recent columns first (for the first two new
      // vertices they hold the anchor's own predecessors, which every list contains), then
      // the Bloom filter and the exact scan
      if constexpr (J < 2) {
        if (y == tail2.x || y == tail2.y) continue;
      }
      if ((bloom & bloom_bit(y)) && in_row_q<NQ>(row, ws, y)) continue;
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
      if constexpr (PUSH && J == 1) {  // hand (row, x_0, x_1) to the second phase
        const int slot = atomicAdd(q->n, 1);
        if (slot < q->cap) {
          q->x0[slot] = x[0];
          q->x1[slot] = y;
          q->r[slot] = (uint8_t)(threadIdx.x);
          continue;
        }
      }
      tot += dfs_ell<J + 1, NQ, PUSH>(st, row, w, ws, bloom, tail2, x, ell, cand, probes, q);
    }
    return tot;
  }
}

// Split tail (n_new 3-4): phase 1 (thread = row) enumerates x_0, x_1 and queues the
// surviving partial rows in shared memory; phase 2 spreads the queue evenly over the CTA's
// threads, each finishing x_2, x_3 of its entries.  The per-row 4-deep recursion left 17 of 32
// lanes idle (rows' subtrees differ); the queue rebalances the second half within the tile.
constexpr int kTailQueuePerRow = 4;
static_assert(kTileRows <= 256, "TailQueue stores the row of an entry in a uint8");

template <int NQ>
__global__ void __launch_bounds__(kStepThreads, 4)
    k_deep_split(const DevStep st, const StepIO io_, const int64_t *__restrict__ off,
                 const int32_t *__restrict__ adj) {
  StepIO io = io_;  // device-written input size (sync-free chaining)
  if (!resolve_in_rows(io)) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t s_bar;
  __shared__ int s_qn;
  __shared__ unsigned long long s_bloom[kTileRows];
  const int w = st.in_w, ws = row_stride(w), ss = smem_stride(w);
  const int tid = threadIdx.x;
  const int64_t tile = io.block_begin + blockIdx.x;
  const int64_t r0 = tile * kTileRows;
  if (r0 >= io.in_rows) return;
  const int nrows = (int)(io.in_rows - r0 < kTileRows ? io.in_rows - r0 : kTileRows);
  int32_t *rows = reinterpret_cast<int32_t *>(smem_raw);
  constexpr int kCap = kTileRows * kTailQueuePerRow;
  int32_t *qx0 = rows + kTileRows * ss;
  int32_t *qx1 = qx0 + kCap;
  uint8_t *qr = reinterpret_cast<uint8_t *>(qx1 + kCap);
  if (tid == 0) s_qn = 0;
  load_tile<NQ>(rows, ss, ws, io, r0, nrows, &s_bar);  // ends with a CTA barrier
  const int4 *ell = reinterpret_cast<const int4 *>(io.ell);
  TailQueue q{&s_qn, kCap, qx0, qx1, qr};
  uint32_t my_cand = 0, my_probe = 0;
  unsigned ns = 0;
  if (tid < nrows) {
    int32_t x[kMaxNew] = {-1, -1, -1, -1};
    const int32_t *row = rows + tid * ss;
    unsigned long long bloom = 0;
    for (int c = 0; c < w; ++c) bloom |= bloom_bit(row[c]);
    s_bloom[tid] = bloom;
    ns = dfs_ell<0, NQ, true>(st, row, w, ws, bloom, make_int2(row[w - 1], w >= 2 ? row[w - 2] : -1),
                              x, ell, my_cand, my_probe, &q);
  }
  __syncthreads();
  const int nq = s_qn < kCap ? s_qn : kCap;
  for (int e = tid; e < nq; e += kStepThreads) {
    const int r = qr[e];
    const int32_t *row = rows + r * ss;
    int32_t x[kMaxNew] = {qx0[e], qx1[e], -1, -1};
    ns += dfs_ell<2, NQ>(st, row, w, ws, s_bloom[r], make_int2(row[w - 1], w >= 2 ? row[w - 2] : -1), x,
                         ell, my_cand, my_probe);
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

}  // namespace

cudaError_t launch_tail(const DevStep &st, const StepIO &io, const dm_graph &g, int64_t tiles,
                        cudaStream_t s) {
  if ((io.in_rows <= 0 && !io.d_in_rows) || tiles <= 0) return cudaSuccess;
  StepIO io2 = io;
  io2.ell = g.d_ell;
  size_t smem = sizeof(int32_t) * (size_t)kTileRows * smem_stride(st.in_w) +
                (size_t)kTileRows * kTailQueuePerRow * (2 * sizeof(int32_t) + 1);
  auto kern = k_deep_split<0>;
  switch (row_stride(st.in_w) >> 2) {
    case 1: kern = k_deep_split<1>; break;
    case 2: kern = k_deep_split<2>; break;
    case 3: kern = k_deep_split<3>; break;
    case 4: kern = k_deep_split<4>; break;
    case 5: kern = k_deep_split<5>; break;
    case 6: kern = k_deep_split<6>; break;
    case 7: kern = k_deep_split<7>; break;
    case 8: kern = k_deep_split<8>; break;
    default: break;
  }
  // Shared memory only for the register-limited number of resident CTAs; the rest of the
  // unified array stays L1 for the ELL lists (160 KB on heavy-hex w=31): with the maximal
  // carveout the ELL loads hit L1 70% of the time, the tile rows need only ~120 KB per SM.
  // Configured per (device, kernel) whenever a launch needs more dynamic shared memory than
  // the kernel was configured for (k_deep_split<0> serves every row width > 32 columns).
  {
    static std::mutex mu;
    static std::map<std::pair<int, const void *>, size_t> configured;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_pair(dev, (const void *)kern);
    auto it = configured.find(key);
    if (it == configured.end() || it->second < smem) {
      e = cudaFuncSetAttribute((const void *)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      int nb = 0;
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, kStepThreads, smem);
      if (e != cudaSuccess) return e;
      cudaFuncAttributes fa{};
      e = cudaFuncGetAttributes(&fa, (const void *)kern);
      if (e != cudaSuccess) return e;
      const double need = (double)nb * (double)(smem + fa.sharedSizeBytes + 1024);
      int cv = (int)std::ceil(100.0 * need / (228.0 * 1024.0));
      cv = cv < 1 ? 1 : (cv > 100 ? 100 : cv);
      e = cudaFuncSetAttribute((const void *)kern, cudaFuncAttributePreferredSharedMemoryCarveout, cv);
      if (e != cudaSuccess) return e;
      configured[key] = smem;
    }
  }
  kern<<<(unsigned)tiles, kStepThreads, smem, s>>>(st, io2, g.d_off, g.d_adj);
  return cudaGetLastError();
}

}  // namespace dm
