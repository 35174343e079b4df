// pairs.cu -- shared-key pair count-only last step (diamond / 4-clique style patterns).
#include "extend_common.cuh"

namespace dm {
namespace {


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
// or, for longer anchor lists, in a per-warp global slab of max_degree entries.  With the
// triangle-apex table (atoff / aapex) and rows that are exactly one arc whose two
// columns are both keys, S is read from the table (apex(u, v), u the lower-degree endpoint)
// instead of being intersected per row; the pairs are inspected the same way.
template <int NQ>
__global__ void __launch_bounds__(kStepThreads)
    k_pairs(const DevStep st, const StepIO io_, const int64_t *__restrict__ off,
            const int32_t *__restrict__ adj, int32_t *__restrict__ slab, int64_t slab_cap,
            int pair_mode, unsigned long long *__restrict__ row_counter, const int64_t *__restrict__ atoff,
            const int32_t *__restrict__ aapex) {
  StepIO io = io_;  // device-written input size (sync-free chaining)
  if (!resolve_in_rows(io)) return;
  constexpr int kWarps = kStepThreads / 32;
  __shared__ __align__(16) int32_t s_row[kWarps][DM_MAX_PATTERN];
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
      int32_t *S;
      int ns = 0;
      if (aapex) {  // S = apex(u, v): one lookup instead of a per-row intersection
        const int64_t d0 = degree(off, row[0]), d1 = degree(off, row[1]);
        const int32_t u = d0 <= d1 ? row[0] : row[1], v = d0 <= d1 ? row[1] : row[0];
        int64_t lo = __ldg(off + u), hi = __ldg(off + u + 1);
        while (lo < hi) {
          const int64_t m = (lo + hi) >> 1;
          if (__ldg(adj + m) < v) lo = m + 1;
          else hi = m;
        }
        const int64_t s0 = __ldg(atoff + lo);
        ns = (int)(__ldg(atoff + lo + 1) - s0);
        S = ns <= kPairSmem ? s_list[wl] : gslab;
        DM_DCHECK(lo < __ldg(off + u + 1) && __ldg(adj + lo) == v && (ns <= kPairSmem || ns <= slab_cap));
        for (int i = lane; i < ns; i += 32) S[i] = __ldg(adj + __ldg(aapex + s0 + i));
        cand += (lane == 0) ? (unsigned long long)ns : 0ull;
      } else {
        int32_t av;
        int64_t ad;
        const int ac = pick_anchor(st, 0, row, w, 0, off, av, ad);
        const int64_t e0 = __ldg(off + av);
        S = ad <= kPairSmem ? s_list[wl] : gslab;
        // ---- S: accepted first-vertex candidates, in anchor-list (ascending) order
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
      }
      __syncwarp();
      // ---- every ordered pair of S
      const int64_t np = (int64_t)ns * ns;
      if (lane == 0 && pair_mode != 1) cand += (unsigned long long)np;
      // 32 splitters of S in registers (lane k: S[ns*k/32]) for the bisections into S
      const int32_t ssp = (pair_mode == 1 && ns > 1) ? S[(ns * lane) >> 5] : 0;
      // 4-clique closing probe: the ranges of N(x0) inside [min S, max S] are found for 32
      // first vertices at once (one bisection chain per lane, in parallel) and broadcast
      int64_t my_lo = 0, my_hi = 0;
      for (int i = 0; i < ns; ++i) {
        const int32_t x0 = S[i];
        if (pair_mode == 1 && ns > 1) {
          if ((i & 31) == 0) {
            const int ii = i + lane;
            if (ii < ns) {
              const int32_t xx = S[ii];
              const int64_t b = __ldg(off + xx), e = __ldg(off + xx + 1);
              const int32_t smin = S[0], smax = S[ns - 1];
              int64_t l = b, h = e;
              while (l < h) {
                const int64_t m = (l + h) >> 1;
                if (__ldg(adj + m) < smin) l = m + 1;
                else h = m;
              }
              my_lo = l;
              h = e;
              while (l < h) {
                const int64_t m = (l + h) >> 1;
                if (__ldg(adj + m) <= smax) l = m + 1;
                else h = m;
              }
              my_hi = l;
            }
          }
          const int64_t lo = __shfl_sync(0xffffffffu, my_lo, i & 31);
          const int64_t hi = __shfl_sync(0xffffffffu, my_hi, i & 31);
          const int64_t m = hi - lo;
          if (lane == 0) cand += (unsigned long long)(m <= 2 * (int64_t)ns ? m : ns);
          if (m <= 2 * (int64_t)ns) {
            for (int64_t t0 = lo; t0 < hi; t0 += 32) {  // N(x0) side, probe S
              const int64_t t = t0 + lane;
              const int32_t y = t < hi ? __ldg(adj + t) : 0;
              int c = 0;  // S splitters (registers, one per lane) below y
#pragma unroll
              for (int sft = 16; sft >= 1; sft >>= 1) {
                const int32_t v = __shfl_sync(0xffffffffu, ssp, c + sft - 1);
                if (v < y) c += sft;
              }
              if (__shfl_sync(0xffffffffu, ssp, c & 31) < y && c == 31) c = 32;
              if (t >= hi) continue;
              int l = c == 0 ? 0 : ((ns * (c - 1)) >> 5) + 1;
              int h = c == 32 ? ns : ((ns * c) >> 5);
              while (l < h) {
                const int mid = (l + h) >> 1;
                if (S[mid] < y) l = mid + 1;
                else h = mid;
              }
              ++probes;
              cnt += (l < ns && S[l] == y);
            }
          } else {
            // S side, probe N(x0): 32 splitters of N(x0)[lo, hi) (one load per lane) give
            // every probe its 1/32 bucket by register shuffles, so each bisection in global
            // memory starts 5 levels down
            const int32_t sp = __ldg(adj + lo + ((m * lane) >> 5));
            for (int j0 = 0; j0 < ns; j0 += 32) {
              const int j = j0 + lane;
              const bool valid = j < ns && j != i;
              const int32_t x1 = j < ns ? S[j] : 0;
              int c = 0;  // number of splitters < x1
#pragma unroll
              for (int sft = 16; sft >= 1; sft >>= 1) {
                const int32_t v = __shfl_sync(0xffffffffu, sp, c + sft - 1);
                if (v < x1) c += sft;
              }
              if (__shfl_sync(0xffffffffu, sp, c & 31) < x1 && c == 31) c = 32;
              if (!valid) continue;
              int64_t l = c == 0 ? lo : lo + ((m * (c - 1)) >> 5) + 1;
              int64_t h = c == 32 ? hi : lo + ((m * c) >> 5);
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

}  // namespace

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
                         cudaStream_t s, const ApexTable *apex) {
  if (io.in_rows <= 0 && !io.d_in_rows) return cudaSuccess;
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
  kern<<<(unsigned)grid, kStepThreads, 0, s>>>(st, io, g.d_off, g.d_adj, slab, cap, pair_mode, counter,
                                                apex ? apex->d_toff : nullptr, apex ? apex->d_apex : nullptr);
  e = cudaGetLastError();
  cudaFreeAsync(slab, s);
  cudaFreeAsync(counter, s);
  return e;
}

}  // namespace dm
