// apex.cu -- the triangle-apex table: Res(M3-O) keyed by directed edge.
//
// Res(M3-O) = Res(M2) ⋈ Res(M2) ⋈ Res(M2) on the three shared vertices of a triangle (P:262,
// §3.4; Alg. 2 builds it once per data graph).  Keyed by its first two template
// positions it is, for every CSR arc (a,b), the sorted list apex(a,b) = N(a) ∩ N(b): the
// candidates of a vertex joined on the two keys a and b.  Layout on the device:
//   toff  int64 [arcs + 1]   apex(a,b) of arc e = (a, adj[e]) is apex[toff[e] .. toff[e+1])
//   apex  int32 [toff[arcs]] each entry c is stored as the CSR arc index of (a, c), i.e. the
//                            position off[a] + p of c in N(a) (the "arc index payload" of
//                            SURVEY §8(a)); the vertex is adj[entry].  Ascending in c.
// Storing arc indices instead of vertex ids makes apex(a, c) of an entry one offset lookup
// (toff[entry]) and makes every apex list keyed by a a set of positions in N(a), so two of
// them intersect by a bitmap over N(a) (k_pairs_apex).  sum |apex| = 6T = tr(A^3).
//
// Build (two-pass, SURVEY a7 style): pass 1 counts |N(a) ∩ N(b)| per arc (warp per arc: lanes
// walk the shorter list, binary search in the longer one), an exclusive scan gives toff, pass 2
// re-runs the intersection and writes the positions in order (warp ballot compaction).
#include <chrono>

#include <cub/cub.cuh>

#include "extend_common.cuh"

namespace dm {
namespace {

constexpr int kApexThreads = 256;
constexpr int kApexBatch = 4;  // arc rows claimed per atomic by a warp of the 4-clique pair step

__global__ void k_arc_src(const int64_t *__restrict__ off, int32_t n, int32_t *__restrict__ src) {
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= n) return;
  for (int64_t e = off[v], e1 = off[v + 1]; e < e1; ++e) src[e] = (int32_t)v;
}

__device__ __forceinline__ int64_t lower_bound_g(const int32_t *__restrict__ adj, int64_t lo, int64_t hi,
                                                 int32_t key) {
  while (lo < hi) {
    const int64_t m = (lo + hi) >> 1;
    if (__ldg(adj + m) < key) lo = m + 1;
    else hi = m;
  }
  return lo;
}

// WRITE = false: cnt[e] = |N(a) ∩ N(b)|;  WRITE = true: apex[toff[e] ..] = arc indices of (a, c)
template <bool WRITE>
__global__ void __launch_bounds__(kApexThreads)
    k_apex(const int64_t *__restrict__ off, const int32_t *__restrict__ adj, const int32_t *__restrict__ src,
           int64_t arcs, int64_t *__restrict__ cnt_toff, int32_t *__restrict__ apex) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t e = warp0; e < arcs; e += nwarps) {
    const int32_t a = __ldg(src + e), b = __ldg(adj + e);
    const int64_t la = __ldg(off + a), ha = __ldg(off + a + 1);
    const int64_t lb = __ldg(off + b), hb = __ldg(off + b + 1);
    const bool a_small = (ha - la) <= (hb - lb);
    const int64_t ls = a_small ? la : lb, hs = a_small ? ha : hb;  // walked list
    const int64_t lL = a_small ? lb : la, hL = a_small ? hb : ha;  // searched list
    int64_t pos = WRITE ? cnt_toff[e] : 0;
    int64_t cnt = 0;
    for (int64_t i0 = ls; i0 < hs; i0 += 32) {
      const int64_t i = i0 + lane;
      bool hit = false;
      int64_t arc = 0;
      if (i < hs) {
        const int32_t x = __ldg(adj + i);
        const int64_t j = lower_bound_g(adj, lL, hL, x);
        hit = j < hL && __ldg(adj + j) == x;
        arc = a_small ? i : j;  // position of x in N(a)
      }
      const unsigned m = __ballot_sync(0xffffffffu, hit);
      if (WRITE) {
        DM_DCHECK(!hit || pos + __popc(m & lt) < cnt_toff[e + 1]);
        if (hit) apex[pos + __popc(m & lt)] = (int32_t)arc;
        pos += __popc(m);
      } else {
        cnt += __popc(m);
      }
    }
    if (!WRITE && lane == 0) cnt_toff[e] = cnt;
  }
}

// ---------------------------------------------------------------------------------------
// Shared-key pair count-only last step on the apex table (pairs.cu's step, SURVEY §8(a) a4-a7
// with a1b): rows are arcs (x_a, x_b) (in_w == 2), both new vertices are keyed on both
// columns, so the first new vertex's candidate set is exactly S = apex(u, v) (u = the endpoint
// of lower degree) -- the equi-join on two keys becomes one table lookup.  The pair
// (x0, x1), x0, x1 in S, passes injectivity iff x0 != x1 (S holds neither u nor v: no
// self-loops); with the closing edge (x0, x1) (4-clique) x1 must lie in
// S ∩ N(x0) = S ∩ apex(u, x0): both are position sets in N(u), so S is put in a per-warp
// bitmap over N(u) and every entry of apex(u, x0) is one bit test.  Entries of the apex lists of
// 32 consecutive x0 are spread over the lanes as one flat range (segment found by a shuffle
// bisection over the lanes' exclusive prefix), so short and long lists keep all lanes busy.
// This is the join of x1 on the keys {u, x0} (Res(M3-O) again) with the closing edge (x1, v) as
// the probe -- a re-association of the pair step, every candidate of that join is
// inspected, and injectivity holds by construction (x1 is in N(u) ∩ N(x0) ∩ N(v), no self-loops).
// Only the closing-edge pair step (4-clique) uses it: the distinct-pairs (diamond) and induced
// non-edge pair steps keep pairs.cu (with S read from this table), which inspects every pair of
// S (no count-mode shortcut that skips inspecting candidates).
__global__ void __launch_bounds__(kStepThreads)
    k_pairs_apex(const StepIO io_, const int64_t *__restrict__ off, const int32_t *__restrict__ adj,
                 const int64_t *__restrict__ toff, const int32_t *__restrict__ apex,
                 uint32_t *__restrict__ gbits, int bm_words, unsigned long long *__restrict__ row_counter) {
  StepIO io = io_;
  if (!resolve_in_rows(io)) return;
  extern __shared__ uint32_t s_bits[];
  constexpr int kWarps = kStepThreads / 32;
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int64_t wg = (int64_t)blockIdx.x * kWarps + wl;
  uint32_t *B = gbits ? gbits + wg * (int64_t)bm_words : s_bits + wl * bm_words;
  if (!gbits) {
    for (int i = lane; i < bm_words; i += 32) B[i] = 0u;
    __syncwarp();
  }
  unsigned long long cnt = 0, cand = 0, probes = 0;
  for (;;) {
    unsigned long long b0 = 0;
    if (lane == 0) b0 = atomicAdd(row_counter, (unsigned long long)kApexBatch);
    b0 = __shfl_sync(0xffffffffu, b0, 0);
    if ((int64_t)b0 >= io.in_rows) break;
    const int64_t b1 = (int64_t)b0 + kApexBatch < io.in_rows ? (int64_t)b0 + kApexBatch : io.in_rows;
    for (int64_t r = (int64_t)b0; r < b1; ++r) {
      const int2 ab = __ldg(reinterpret_cast<const int2 *>(io.in + r * 4));
      const int64_t da = degree(off, ab.x), db = degree(off, ab.y);
      const int32_t u = da <= db ? ab.x : ab.y, v = da <= db ? ab.y : ab.x;
      const int64_t lu = __ldg(off + u), hu = __ldg(off + u + 1);
      const int64_t e = lower_bound_g(adj, lu, hu, v);  // arc (u, v): every lane, broadcast loads
      DM_DCHECK(e < hu && __ldg(adj + e) == v);        // the rows are arcs
      const int64_t s0 = __ldg(toff + e), ns = __ldg(toff + e + 1) - s0;
      DM_DCHECK(ns >= 0 && ns <= hu - lu);
      if (lane == 0) cand += (unsigned long long)ns;
      if (ns < 2) continue;
      for (int64_t i = lane; i < ns; i += 32) {
        const int64_t p = __ldg(apex + s0 + i) - lu;
        DM_DCHECK(p >= 0 && p < hu - lu && (p >> 5) < bm_words);  // positions in N(u)
        atomicOr(B + (p >> 5), 1u << (p & 31));
      }
      __syncwarp();
      unsigned long long edges = 0;
      // chunks of 32 x0: the next chunk's arcs (u, x0) are loaded while this chunk is tested, and
      // two 32-entry rounds are in flight at a time (the apex lists are mostly L2/HBM reads)
      int32_t e_nxt = lane < ns ? __ldg(apex + s0 + lane) : -1;
      for (int64_t c0 = 0; c0 < ns; c0 += 32) {
        const int32_t e0 = e_nxt;  // arc (u, x0) of this lane's x0, -1 past the end
        int64_t t0 = 0;
        int len = 0;
        if (e0 >= 0) {
          t0 = __ldg(toff + e0);
          len = (int)(__ldg(toff + e0 + 1) - t0);
        }
        e_nxt = c0 + 32 + lane < ns ? __ldg(apex + s0 + c0 + 32 + lane) : -1;
        int incl = len;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, d);
          if (lane >= d) incl += y;
        }
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        const int excl = incl - len;
        if (lane == 0) probes += (unsigned long long)total;
        for (int j0 = 0; j0 < total; j0 += 64) {
          const int ja = j0 + lane, jb = j0 + 32 + lane;
          int ka = 0, kb = 0;  // last lane whose segment starts at or before ja / jb
#pragma unroll
          for (int sft = 16; sft >= 1; sft >>= 1) {
            if (__shfl_sync(0xffffffffu, excl, ka + sft) <= ja) ka += sft;
            if (__shfl_sync(0xffffffffu, excl, kb + sft) <= jb) kb += sft;
          }
          const int64_t tka = __shfl_sync(0xffffffffu, t0, ka), tkb = __shfl_sync(0xffffffffu, t0, kb);
          const int eka = __shfl_sync(0xffffffffu, excl, ka), ekb = __shfl_sync(0xffffffffu, excl, kb);
          const bool va = ja < total, vb = jb < total;
          const int64_t qa = (va ? __ldg(apex + tka + (ja - eka)) : lu) - lu;
          const int64_t qb = (vb ? __ldg(apex + tkb + (jb - ekb)) : lu) - lu;
          DM_DCHECK(qa >= 0 && qa < hu - lu && qb >= 0 && qb < hu - lu);  // apex(u, x0) ⊆ N(u)
          edges += va & ((B[qa >> 5] >> (qa & 31)) & 1u);
          edges += vb & ((B[qb >> 5] >> (qb & 31)) & 1u);
        }
      }
      __syncwarp();
      for (int64_t i = lane; i < ns; i += 32) {  // clear S's bits
        const int64_t p = __ldg(apex + s0 + i) - lu;
        B[p >> 5] = 0u;
      }
      __syncwarp();
      cnt += edges;
    }
  }
  cand += probes;  // second-level candidates: the apex entries inspected
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

dm_status build_apex_table(const dm_graph *g, cudaStream_t s, ApexTable &t) {
  NvtxRange nvtx("triangle-apex table");
  const int64_t arcs = g->arcs;
  if (arcs >= (int64_t)INT32_MAX) return fail(DM_ERR_UNSUPPORTED, "apex table needs < 2^31 arcs");
  const auto t_start = std::chrono::steady_clock::now();
  int64_t *d_toff = nullptr;
  int32_t *d_src = nullptr, *d_apex = nullptr;
  void *d_tmp = nullptr;
  auto cleanup = [&]() {
    if (d_src) cudaFreeAsync(d_src, s);
    if (d_tmp) cudaFreeAsync(d_tmp, s);
  };
  auto cfail = [&](cudaError_t e, const char *what) {
    cleanup();
    if (d_toff) cudaFreeAsync(d_toff, s);
    if (d_apex) cudaFreeAsync(d_apex, s);
    return fail(e == cudaErrorMemoryAllocation ? DM_ERR_OOM : DM_ERR_CUDA,
                std::string("apex table: ") + what + ": " + cudaGetErrorString(e));
  };
#define AK(call, what)                      \
  do {                                      \
    cudaError_t _e = (call);                \
    if (_e != cudaSuccess) return cfail(_e, what); \
  } while (0)
  AK(cudaMallocAsync((void **)&d_toff, sizeof(int64_t) * (size_t)(arcs + 1), s), "alloc");
  AK(cudaMallocAsync((void **)&d_src, sizeof(int32_t) * (size_t)std::max<int64_t>(arcs, 1), s), "alloc");
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (g->n > 0) k_arc_src<<<(unsigned)((g->n + 255) / 256), 256, 0, s>>>(g->d_off, g->n, d_src);
  AK(cudaGetLastError(), "arc sources");
  const int64_t want = (arcs * 32 + kApexThreads - 1) / kApexThreads;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * 16));
  AK(cudaMemsetAsync(d_toff + arcs, 0, sizeof(int64_t), s), "memset");
  if (arcs > 0) k_apex<false><<<grid, kApexThreads, 0, s>>>(g->d_off, g->d_adj, d_src, arcs, d_toff, nullptr);
  AK(cudaGetLastError(), "count pass");
  size_t tmp_bytes = 0;
  AK(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, d_toff, d_toff, arcs + 1, s), "scan");
  AK(cudaMallocAsync(&d_tmp, tmp_bytes, s), "alloc");
  AK(cub::DeviceScan::ExclusiveSum(d_tmp, tmp_bytes, d_toff, d_toff, arcs + 1, s), "scan");
  int64_t total = 0;
  AK(cudaMemcpyAsync(&total, d_toff + arcs, sizeof(int64_t), cudaMemcpyDeviceToHost, s), "readback");
  AK(cudaStreamSynchronize(s), "sync");
  AK(cudaMallocAsync((void **)&d_apex, sizeof(int32_t) * (size_t)std::max<int64_t>(total, 1), s), "alloc");
  if (arcs > 0 && total > 0)
    k_apex<true><<<grid, kApexThreads, 0, s>>>(g->d_off, g->d_adj, d_src, arcs, d_toff, d_apex);
  AK(cudaGetLastError(), "write pass");
  AK(cudaStreamSynchronize(s), "sync");
#undef AK
  cleanup();
  t.d_toff = d_toff;
  t.d_apex = d_apex;
  t.entries = total;
  t.build_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
  return DM_OK;
}

// The apex table serves a shared-key pair step (pair_mode_of >= 0) on rows that are exactly one
// arc (in_w == 2) when both new vertices key on both columns, with no other filter on the first
// one (induced non-edges to other columns do not exist at w == 2): the closing-edge (4-clique)
// step runs k_pairs_apex, the others take S from the table in k_pairs.
bool apex_arc_rows(const DevStep &st, int elem) {
  if (st.in_w != 2 || st.n_new != 2 || elem != 4) return false;
  if (st.n_nbr[0] != 2 || st.n_non[0] != 0) return false;
  const bool keys = (st.nbr[0][0] == 0 && st.nbr[0][1] == 1) || (st.nbr[0][0] == 1 && st.nbr[0][1] == 0);
  return keys && pair_mode_of(st) >= 0;
}

cudaError_t launch_pairs_apex(const DevStep &st, const StepIO &io, const dm_graph &g, const ApexTable &t,
                              cudaStream_t s) {
  if (io.in_rows <= 0 && !io.d_in_rows) return cudaSuccess;
  const int bm_words = (g.max_deg + 31) / 32 + 1;
  const size_t smem = sizeof(uint32_t) * (size_t)bm_words * (kStepThreads / 32);
  const bool use_smem = smem <= 160 * 1024;
  auto kern = k_pairs_apex;
  const size_t dyn = use_smem ? smem : 0;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  if (e != cudaSuccess) return e;
  int per_sm = 0, sms = 0, dev = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kStepThreads, dyn);
  if (e != cudaSuccess) return e;
  cudaGetDevice(&dev);
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  const int64_t grid = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
  uint32_t *gbits = nullptr;
  unsigned long long *counter = nullptr;
  if (!use_smem) {
    const size_t gb = sizeof(uint32_t) * (size_t)bm_words * (size_t)(grid * (kStepThreads / 32));
    e = cudaMallocAsync((void **)&gbits, gb, s);
    if (e != cudaSuccess) return e;
    cudaMemsetAsync(gbits, 0, gb, s);
  }
  e = cudaMallocAsync((void **)&counter, sizeof(unsigned long long), s);
  if (e != cudaSuccess) {
    if (gbits) cudaFreeAsync(gbits, s);
    return e;
  }
  cudaMemsetAsync(counter, 0, sizeof(unsigned long long), s);
  kern<<<(unsigned)grid, kStepThreads, dyn, s>>>(io, g.d_off, g.d_adj, t.d_toff, t.d_apex, gbits, bm_words, counter);
  e = cudaGetLastError();
  if (gbits) cudaFreeAsync(gbits, s);
  cudaFreeAsync(counter, s);
  return e;
}

}  // namespace dm
