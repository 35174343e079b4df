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

#include "extend_common.cuh"

namespace dm {

namespace {
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
    k_step(const DevStep st, const StepIO io_, const int64_t *__restrict__ off,
           const int32_t *__restrict__ adj) {
  StepIO io = io_;  // device-written input size (sync-free chaining)
  if (!resolve_in_rows(io)) return;
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
      io.agg[tile] = (unsigned long long)agg;
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
    k_rows(const DevStep st, const StepIO io_, const int64_t *__restrict__ off,
           const int32_t *__restrict__ adj) {
  StepIO io = io_;  // device-written input size (sync-free chaining)
  if (!resolve_in_rows(io)) return;
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
  const int tid = threadIdx.x;
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

  load_tile<NQ>(rows, ss, ws, io, r0, nrows, &s_bar);

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
      const int2 tail2 = make_int2(row[w - 1], w >= 2 ? row[w - 2] : -1);
      int4 na;
      const int ac = pick_anchor_ell(st, 0, row, w, 0, ell, na);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int32_t x0 = ell_at(na, i);
        if (x0 < 0) break;
        ++n_cand;
        if (!accept_ell<NQ>(st, 0, row, w, ws, bloom, tail2, 0, x0, ac, ell, n_probe)) continue;
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
          if (accept_ell<NQ>(st, 1, row, w, ws, bloom, tail2, x0, x1, bc, ell, n_probe)) on_survivor(x0, x1);
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
  auto reduce_stats = [&]() {
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
  };
  if (MODE == kModeCount) {
    reduce_stats();
    return;
  }
  int pos, agg;
  ScanI(tmp).ExclusiveSum(ns, pos, agg);
  // Output space by atomic reservation: no tile waits for its predecessors (a decoupled
  // look-back here stalled the CTA at the barrier for ~25% of the step).  The rows of a level
  // are then in tile-completion order; counts do not depend on it and tables are sorted at the
  // end (a9).  A tile that does not fit makes the host re-run the whole step at exact offsets
  // (kModeWrite, tile order) from the per-tile counts.  The reservation is issued as soon as
  // the tile total is known; its round trip overlaps the statistics reduction and the map.
  unsigned long long base = 0;
  if (MODE == kModeSingle && tid == 0 && agg) base = atomicAdd(io.ctrl + 2, (unsigned long long)agg);
  if (io.stats) reduce_stats();
  const bool any_ovf = __syncthreads_or(ovf);
  if (!any_ovf)
    for (int i = 0; i < ns; ++i) map[pos + i] = (tid << 4) | i;
  if (MODE == kModeWrite) {  // re-run at an exact offset
    if (tid == 0) s_bc = io.block_off[tile] - io.out_base;
  } else if (tid == 0) {
    io.agg[tile] = (unsigned long long)agg;
    const bool fits = base + (unsigned long long)agg <= io.cap;
    if (!fits) atomicMax(io.ctrl + 1, (unsigned long long)ntiles_of(io));
    s_bc = fits ? base : ~0ull;
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

template <int MODE, int NQ>
cudaError_t launch_rows_nq(const DevStep &st, const StepIO &io, const dm_graph &g, int64_t tiles,
                           size_t smem, cudaStream_t s) {
  if (MODE == kModeCount && g.d_ell && st.n_new > 2) return launch_tail(st, io, g, tiles, s);
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

cudaError_t launch_agg_to_excl(const unsigned long long *agg, int64_t tiles, uint64_t *excl,
                               cudaStream_t s) {
  const unsigned long long *in = agg;
  unsigned long long *out = reinterpret_cast<unsigned long long *>(excl);
  size_t tmp_bytes = 0;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, in, out, (int64_t)(tiles + 1), s);
  if (e != cudaSuccess) return e;
  void *tmp = nullptr;
  e = cudaMallocAsync(&tmp, tmp_bytes, s);
  if (e != cudaSuccess) return e;
  e = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, in, out, (int64_t)(tiles + 1), s);
  cudaFreeAsync(tmp, s);
  return e;
}

DevStep make_dev_step(const Step &st) {
  DevStep d{};
  d.in_w = st.in_w;
  d.n_new = st.n_new;
  if (st.tab_motif) {  // table step: widths + the key (per-row work estimate of k_row_work)
    d.n_nbr[0] = 1;
    d.nbr[0][0] = (uint8_t)st.key0;
    return d;
  }
  for (int j = 0; j < st.n_new; ++j) {
    d.n_nbr[j] = st.nv[j].n_nbr;
    d.n_non[j] = st.nv[j].n_non;
    for (int t = 0; t < st.nv[j].n_nbr; ++t) d.nbr[j][t] = (uint8_t)st.nv[j].nbr[t];
    for (int t = 0; t < st.nv[j].n_non; ++t) d.non[j][t] = (uint8_t)st.nv[j].non[t];

  }
  return d;
}

}  // namespace dm
