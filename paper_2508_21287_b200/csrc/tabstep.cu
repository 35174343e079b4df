// tabstep.cu -- table steps: the join of a frontier level with a materialized motif table
// Res(M) (Alg. 1 l.6 InnerJoin; the larger motifs of §3.4-3.5), fused
// with the overlapping-node filter and the closing-edge probes of the remaining
// pattern edges.
//
// Res(M) rows are sorted lexicographically and indexed by the CSR arc of their first two
// template positions (MotifTable::d_toff), so the equi-join of a row on its key column(s) is an
// index range: one key (template position 0 bound) -> the rows of the key's vertex, minus the
// sub-range whose position 1 is the image of a pattern neighbour of the key (a known duplicate
// the all-distinct filter would reject: skipping it is the same selection, evaluated on the
// index); two keys (positions 0 and 1 bound) -> the rows of that arc.
//
// CTA = tile of 256 frontier rows in shared memory.  Per row the index range(s) are looked up
// and the tile's entries are laid out by an exclusive scan, so every thread inspects one entry
// per round wherever it comes from (hub keys spread over the CTA; no per-row divergence).  An
// entry is accepted when every further bound template position equals its row column
// (equality filters = the remaining join constraints), its new vertices are not in the row
// (Bloom filter, then the exact LDS.128 scan) and every closing-edge probe holds (non-edge
// probes fail, induced mode).  Survivors are staged (row, entry) in shared memory with warp
// ballots and flushed in chunks: single-pass launches reserve output rows with one atomicAdd per
// flush (rows land in completion order, as in k_rows), the exact re-run (kModeWrite) writes at
// its tile's exclusive offset, count launches only reduce.
#include <cub/cub.cuh>

#include "extend_common.cuh"

namespace dm {
namespace {


// position of b in N(a) as a CSR arc index, -1 if (a, b) is not an arc
template <bool ELL>
__device__ __forceinline__ int64_t arc_index(const int64_t *__restrict__ off, const int32_t *__restrict__ adj,
                                             const int4 *__restrict__ ell, int32_t a, int32_t b) {
  const int64_t lo0 = __ldg(off + a);
  if (ELL) {
    const int4 e = __ldg(ell + a);
    const int i = e.x == b ? 0 : (e.y == b ? 1 : (e.z == b ? 2 : (e.w == b ? 3 : -1)));
    return i < 0 ? -1 : lo0 + i;
  }
  int64_t lo = lo0, hi = __ldg(off + a + 1);
  const int64_t end = hi;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(adj + mid) < b) lo = mid + 1;
    else hi = mid;
  }
  return (lo < end && __ldg(adj + lo) == b) ? lo : -1;
}

// template position p of an entry held in up to three int4 registers
__device__ __forceinline__ int32_t tsel(const int4 (&E)[3], int p) {
  const int4 v = p < 4 ? E[0] : (p < 8 ? E[1] : E[2]);
  const int c = p & 3;
  return c == 0 ? v.x : (c == 1 ? v.y : (c == 2 ? v.z : v.w));
}

template <bool ELL>
__device__ __forceinline__ bool edge_probe(const int64_t *__restrict__ off, const int32_t *__restrict__ adj,
                                           const int4 *__restrict__ ell, int32_t u, int32_t x) {
  if (ELL) return ell_has(ell, u, x);
  return has_edge(off, adj, u, x);
}

// entry component p (compile-time p after unrolling)
__device__ __forceinline__ int32_t tcomp(const int4 (&E)[3], int p) {
  const int4 &v = E[p >> 2];
  return (p & 3) == 0 ? v.x : ((p & 3) == 1 ? v.y : ((p & 3) == 2 ? v.z : v.w));
}

constexpr int kWarpStage = 64;  // survivors staged per warp before a warp-level flush
// per-row 512-bit membership filter of the row's vertex set (one hash; ~5% false positives for
// 24-column rows, against ~17% for a 128-bit filter; 1024 bits measured slower: the larger
// shared-memory footprint costs a CTA per SM); stride 17 words (bank spread)
constexpr int kFiltWords = 16, kFiltStride = 17;
__device__ __forceinline__ uint32_t filt_hash(int32_t v) { return ((uint32_t)v * 0x9E3779B1u) >> 23; }

// 16-bit levels (R16): the tile is kept in shared memory as the stored uint16 ids (half the bytes
// of widened rows: more CTAs per SM), rows padded to an odd number of 16-byte chunks
// (conflict-free LDS.128 across lanes); the exact all-distinct scan tests two ids per 32-bit
// word: t = word ^ (x | x << 16) has a zero half iff x is one of them, detected branch-free by
// (t - 0x00010001) & ~t & 0x80008000 (a borrow from a zero low half can only add a report when a
// zero half exists already); padding 0xFFFF is never an id since n <= 65535.  __vcmpeq2 is
// emulated on sm_100 (~6 instructions per word).
__host__ __device__ inline int smem_stride16(int w) {
  const int rs = row_stride16(w);
  return ((rs >> 3) & 1) ? rs : rs + 8;
}
__device__ __forceinline__ bool in_row16(const uint16_t *row, int nq8, int32_t x) {
  const uint32_t xx = (uint32_t)x * 0x10001u;
  const uint4 *r4 = reinterpret_cast<const uint4 *>(row);
  uint32_t hit = 0;
  auto zero_half = [](uint32_t t) { return (t - 0x00010001u) & ~t & 0x80008000u; };
  for (int q = 0; q < nq8; ++q) {
    const uint4 v = r4[q];
    hit |= zero_half(v.x ^ xx) | zero_half(v.y ^ xx) | zero_half(v.z ^ xx) | zero_half(v.w ^ xx);
  }
  return hit != 0u;
}
// tile of 16-bit rows -> shared memory (no widening): one TMA bulk copy when the smem stride
// equals the stored stride, else 16-byte chunks.  Ends with a CTA barrier.
__device__ __forceinline__ void load_tile16(uint16_t *rows, int ss16, int rs16, const StepIO &io, int64_t r0,
                                            int nrows, uint64_t *bar) {
  const uint16_t *src = reinterpret_cast<const uint16_t *>(io.in) + r0 * rs16;
  if (ss16 == rs16) {
    if (threadIdx.x == 0) {
      mbar_init(bar, 1);
      const unsigned bytes = (unsigned)(nrows * rs16) * 2u;
      mbar_expect_tx(bar, bytes);
      tma_bulk_g2s(rows, src, bytes, bar);
    }
    __syncthreads();
    mbar_wait(bar, 0);
    return;
  }
  const int nq8 = rs16 >> 3, total = nrows * nq8;
  const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
  for (int i = threadIdx.x; i < total; i += kStepThreads) {
    const int r = i / nq8, q = i - r * nq8;
    reinterpret_cast<uint4 *>(rows + r * ss16)[q] = __ldcs(s4 + i);
  }
  __syncthreads();
}

// Warp-level join: warp w owns the tile rows [32w, 32w+32) (lane = row for the index lookups);
// the warp's entries are laid out by a warp scan of the per-row entry counts and inspected 32 per
// round, lane -> entry, the entry's row found by a 5-step shuffle bisection of the row offsets.
// No CTA barrier between the tile load and the epilogue.  TS = table row stride (4, 8 or 12 ids).
// Occupancy targets (registers capped by the launch bounds): the count launch fits 6 CTAs per SM
// in shared memory on 16-bit tiles, the materializing launches 4.
template <int MODE, bool ELL, int TS, bool R16>
__global__ void __launch_bounds__(kStepThreads, MODE == kModeCount ? 6 : 4)
    k_table(const DevTabStep st, const StepIO io_, const int64_t *__restrict__ off,
            const int32_t *__restrict__ adj, const int32_t *__restrict__ tab,
            const int64_t *__restrict__ toff) {
  StepIO io = io_;
  if (!resolve_in_rows(io)) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int4 s_meta[kTileRows];  // per row: {first index range start, its length, second range
                                      //  start, last column}; table indices < 2^31
  __shared__ unsigned long long s_tile;
  __shared__ unsigned long long s_wtot[kStepThreads / 32];
  __shared__ __align__(8) uint64_t s_bar;
  constexpr int kWarps = kStepThreads / 32;
  constexpr int NE = TS / 4;  // int4 loads per table row

  // ss: smem row stride in elements (int32, or uint16 for R16); ws: int32 words of a widened row
  const int w = st.in_w, ws = row_stride(w), ss = R16 ? smem_stride16(w) : smem_stride(w);
  const int nq8 = row_stride16(w) >> 3;  // R16: 16-byte chunks of a stored row
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int64_t tile;
  if (MODE == kModeSingle) {
    if (tid == 0) s_tile = atomicAdd(io.ctrl + 0, 1ull);
    __syncthreads();
    tile = (int64_t)s_tile;
  } else {
    tile = io.block_begin + blockIdx.x;
  }
  const int64_t r0 = tile * kTileRows;
  if (r0 >= io.in_rows) return;
  const int nrows = (int)(io.in_rows - r0 < kTileRows ? io.in_rows - r0 : kTileRows);
  int32_t *rows = reinterpret_cast<int32_t *>(smem_raw);
  uint16_t *rows16 = reinterpret_cast<uint16_t *>(smem_raw);
  uint32_t *filt = reinterpret_cast<uint32_t *>(smem_raw + (size_t)kTileRows * ss * (R16 ? 2 : 4));  // [kTileRows][kFiltStride]
  int32_t *sv_new = reinterpret_cast<int32_t *>(filt + kTileRows * kFiltStride) + warp * kWarpStage * TS;
  int32_t *stage_r = reinterpret_cast<int32_t *>(filt + kTileRows * kFiltStride) + kWarps * kWarpStage * TS +
                     warp * kWarpStage;
  if constexpr (R16) load_tile16(rows16, ss, row_stride16(w), io, r0, nrows, &s_bar);  // ends with a CTA barrier
  else load_tile(rows, ss, ws, io, r0, nrows, &s_bar);
  const int4 *ell = reinterpret_cast<const int4 *>(io.ell);
  // column c (< w) of tile row r
  auto RV = [&](int r, int c) -> int32_t {
    if constexpr (R16) return (int32_t)rows16[r * ss + c];
    else return rows[r * ss + c];
  };
  auto IN_ROW = [&](int r, int32_t x) -> bool {
    if constexpr (R16) return in_row16(rows16 + r * ss, nq8, x);
    else return in_row(rows + r * ss, ws, x);
  };

  // ---- lane = row: index range(s) of the join and the row's membership filter
  long long cnt = 0;
  if (tid < nrows) {
    uint32_t *f = filt + tid * kFiltStride;
#pragma unroll
    for (int i = 0; i < kFiltWords; ++i) f[i] = 0u;
    for (int c = 0; c < w; ++c) {
      const uint32_t h = filt_hash(RV(tid, c));
      f[h >> 5] |= 1u << (h & 31);
    }
    const int32_t a = RV(tid, st.key0);
    long long lo = 0, seg1 = 0, seg2 = 0, tot = 0;
    if (st.key1 >= 0) {
      const int64_t ai = arc_index<ELL>(off, adj, ell, a, RV(tid, st.key1));
      if (ai >= 0) {
        lo = __ldg(toff + ai);
        seg1 = tot = __ldg(toff + ai + 1) - lo;
      }
    } else {
      lo = __ldg(toff + __ldg(off + a));
      const long long hi = __ldg(toff + __ldg(off + a + 1));
      seg1 = tot = hi - lo;
      seg2 = hi;
      if (st.skip >= 0) {
        const int64_t ai = arc_index<ELL>(off, adj, ell, a, RV(tid, st.skip));
        if (ai >= 0) {
          const long long slo = __ldg(toff + ai), shi = __ldg(toff + ai + 1);
          seg1 = slo - lo;
          seg2 = shi;
          tot = (hi - lo) - (shi - slo);
        }
      }
    }
    s_meta[tid] = make_int4((int)lo, (int)seg1, (int)seg2, 0);
    cnt = tot;
  }
  long long incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const long long ex = incl - cnt;                        // first entry of this lane's row
  const long long T = __shfl_sync(0xffffffffu, incl, 31);  // entries of the warp's rows
  const bool small = T < (1ll << 30);                     // 32-bit offsets for the bisection
  const int ex32 = (int)ex;
  __syncwarp();

  uint32_t my_cand = 0, my_probe = 0;
  unsigned long long my_surv = 0;
  const uint32_t newmask = st.newmask, eqmask = st.eqmask;

  // one round: lane -> entry j of the warp; returns acceptance, the entry's row and its ids
  auto eval = [&](long long j, int &r, int4 (&E)[3]) -> bool {
    int c = 0;  // largest lane i with ex_i <= j (binary lifting over the warp's row offsets)
    long long exr;
    if (small) {
      const int j32 = (int)j;
#pragma unroll
      for (int sft = 16; sft >= 1; sft >>= 1)
        if (__shfl_sync(0xffffffffu, ex32, c + sft) <= j32) c += sft;
      exr = __shfl_sync(0xffffffffu, ex32, c);
    } else {
#pragma unroll
      for (int sft = 16; sft >= 1; sft >>= 1)
        if (__shfl_sync(0xffffffffu, ex, c + sft) <= j) c += sft;
      exr = __shfl_sync(0xffffffffu, ex, c);
    }
    if (j >= T) return false;
    r = warp * 32 + c;
    const int loc = (int)(j - exr);
    const int4 meta = s_meta[r];
    const int ei = loc < meta.y ? meta.x + loc : meta.z + (loc - meta.y);
    DM_DCHECK(r < nrows && ei >= 0 && ei < st.trows);
    ++my_cand;
    const int4 *ent = reinterpret_cast<const int4 *>(tab + (int64_t)ei * TS);
#pragma unroll
    for (int i = 0; i < 3; ++i) E[i] = i < NE ? __ldg(ent + i) : make_int4(-1, -1, -1, -1);
    const uint32_t *f = filt + r * kFiltStride;
    bool ok = true;
    if (eqmask) {  // further bound template positions: the remaining join constraints
#pragma unroll
      for (int p = 0; p < TS; ++p)
        if ((eqmask >> p) & 1u) ok = ok && tcomp(E, p) == RV(r, st.eq_colp[p]);
    }
    uint32_t hits = 0;  // new positions whose filter bit is set: exact scan needed
#pragma unroll
    for (int p = 0; p < TS; ++p) {
      if ((newmask >> p) & 1u) {
        // all-distinct: the row filter sends the few possible duplicates to the exact
        // scan below
        const uint32_t h = filt_hash(tcomp(E, p));
        hits |= ((f[h >> 5] >> (h & 31)) & 1u) << p;
      }
    }
    while (ok && hits) {  // deferred exact scans: only the filter hits
      const int p = __ffs(hits) - 1;
      hits &= hits - 1;
      if (IN_ROW(r, tsel(E, p))) ok = false;
    }
    for (int p = 0; p < st.n_pr && ok; ++p) {
      const int cc = st.pr_c[p];
      const int32_t u = cc < w ? RV(r, cc) : tsel(E, st.newpos[cc - w]);
      const int32_t x = tsel(E, st.newpos[st.pr_j[p]]);
      ++my_probe;
      ok = edge_probe<ELL>(off, adj, ell, u, x) != (st.pr_neg[p] != 0);
    }
    return ok;
  };

  if (MODE == kModeCount) {
    for (long long jb = 0; jb < T; jb += 32) {
      int r;
      int4 E[3];
      my_surv += eval(jb + lane, r, E);
    }
  } else {
    // output chunk of this lane in a warp flush: 8 (16-bit) or 4 (int32) consecutive columns;
    // per column a source code: new column index j (< 0xFE), 0xFE = the parent row, 0xFF = pad
    const int Wn = w + st.n_new;
    const int nq = io.out_elem == 2 ? (row_stride16(Wn) >> 3) : (row_stride(Wn) >> 2);
    int lpr = 1;
    while (lpr < nq) lpr <<= 1;
    const int rpi = 32 / lpr, q = lane & (lpr - 1), sub = lane / lpr;
    const int per = io.out_elem == 2 ? 8 : 4;
    const int c0 = per * q;
    const bool all_parent = c0 + per <= w;
    // aligned tail: when the output columns from the last chunk boundary before w (w_al) to the
    // row end fit the TS staged words, a survivor is staged as exactly those columns (parent
    // columns [w_al, w), then the new vertices in output order), so a flush lane whose chunk
    // reaches past w reads its chunk with 16-byte loads -- no per-column source selection
    const int w_al = (w / per) * per;
    const bool tail_fast = Wn - w_al <= TS;
    unsigned long long codes = 0;
    for (int i = 0; i < per; ++i) {
      const int c = c0 + i;
      const unsigned code = c < w ? 0xFEu : (c < Wn ? (unsigned)(c - w) : 0xFFu);
      codes |= (unsigned long long)code << (8 * i);
    }
    unsigned long long wbase = 0;  // kModeWrite: this warp's first output row
    if (MODE == kModeWrite) {      // exact re-run: survivors per warp first, then a CTA prefix
      unsigned long long mine = 0;
      for (long long jb = 0; jb < T; jb += 32) {
        int r;
        int4 E[3];
        mine += eval(jb + lane, r, E);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
      if (lane == 0) s_wtot[warp] = mine;
      __syncthreads();
      wbase = io.block_off[tile] - io.out_base;
      for (int i = 0; i < warp; ++i) wbase += s_wtot[i];
      my_cand = my_probe = 0;
    }
    unsigned long long written = 0;
    auto warp_flush = [&](int fill) {
      unsigned long long base;
      if (MODE == kModeSingle) {
        unsigned long long b = 0;
        if (lane == 0) {
          b = atomicAdd(io.ctrl + 2, (unsigned long long)fill);
          if (b + (unsigned long long)fill > io.cap) {
            atomicMax(io.ctrl + 1, (unsigned long long)ntiles_of(io));
            b = ~0ull;
          }
        }
        base = __shfl_sync(0xffffffffu, b, 0);
      } else {
        base = wbase + written;
      }
      __syncwarp();
      if (R16 && io.out_elem == 2 && tail_fast) {
        // 16-bit rows with an aligned tail: two converged passes instead of one divergent one --
        // the parent-only chunks copied as stored, then the tail chunks packed from the stage
        if (base != ~0ull) {
          const int npar = w_al >> 3, ntail = nq - npar;
          if (npar > 0) {
            const int rpi_p = 32 / npar, my_o = lane / npar, my_q = lane - my_o * npar;
            for (int o = my_o; my_o < rpi_p && o < fill; o += rpi_p)
              reinterpret_cast<uint4 *>(io.out)[(int64_t)(base + o) * nq + my_q] =
                  *reinterpret_cast<const uint4 *>(rows16 + stage_r[o] * ss + 8 * my_q);
          }
          if (ntail > 0) {
            const int rpi_t = 32 / ntail, my_o = lane / ntail, my_t = lane - my_o * ntail;
            const int tq = npar + my_t, tc0 = 8 * tq;  // output chunk and its first column
            for (int o = my_o; my_o < rpi_t && o < fill; o += rpi_t) {
              const int32_t *nv = sv_new + o * TS + 8 * my_t;
              uint32_t u[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const uint32_t lo = tc0 + 2 * i < Wn ? (uint32_t)nv[2 * i] & 0xffffu : 0xffffu;
                const uint32_t hi = tc0 + 2 * i + 1 < Wn ? (uint32_t)nv[2 * i + 1] & 0xffffu : 0xffffu;
                u[i] = lo | (hi << 16);
              }
              reinterpret_cast<uint4 *>(io.out)[(int64_t)(base + o) * nq + tq] = make_uint4(u[0], u[1], u[2], u[3]);
            }
          }
        }
      } else if (base != ~0ull && q < nq) {
        for (int o = sub; o < fill; o += rpi) {
          const int pr = stage_r[o];
          const int4 neg = make_int4(-1, -1, -1, -1);
          if (R16 && io.out_elem == 2 && all_parent) {  // 16 parent bytes copied as they are stored
            reinterpret_cast<uint4 *>(io.out)[(int64_t)(base + o) * nq + q] =
                *reinterpret_cast<const uint4 *>(rows16 + pr * ss + c0);
            continue;
          }
          int32_t v[8];
          if (!all_parent && tail_fast) {
            // every column of this chunk is in the staged tail (nothing from the parent row)
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = -1;
          } else if constexpr (R16) {
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = (i < per && c0 + i < w) ? RV(pr, c0 + i) : -1;
          } else {
            const int32_t *prow = rows + pr * ss;
            const int4 pa = c0 < ws ? *reinterpret_cast<const int4 *>(prow + c0) : neg;
            const int4 pb = (per == 8 && c0 + 4 < ws) ? *reinterpret_cast<const int4 *>(prow + c0 + 4) : neg;
            v[0] = pa.x; v[1] = pa.y; v[2] = pa.z; v[3] = pa.w;
            v[4] = pb.x; v[5] = pb.y; v[6] = pb.z; v[7] = pb.w;
          }
          if (!all_parent) {
            const int32_t *nv = sv_new + o * TS;
            if (tail_fast) {  // the staged tail holds this chunk's columns at offset c0 - w_al
              const int4 ta = *reinterpret_cast<const int4 *>(nv + (c0 - w_al));
              const int4 tb = per == 8 ? *reinterpret_cast<const int4 *>(nv + (c0 - w_al) + 4) : neg;
              const int32_t t[8] = {ta.x, ta.y, ta.z, ta.w, tb.x, tb.y, tb.z, tb.w};
#pragma unroll
              for (int i = 0; i < 8; ++i) v[i] = c0 + i < Wn ? t[i] : -1;
            } else {
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const unsigned code = (unsigned)(codes >> (8 * i)) & 0xFFu;
                if (code != 0xFEu) v[i] = code == 0xFFu ? -1 : nv[code];
              }
            }
          }
          if (io.out_elem == 2) {
            reinterpret_cast<uint4 *>(io.out)[(int64_t)(base + o) * nq + q] =
                make_uint4(((uint32_t)v[0] & 0xffffu) | ((uint32_t)v[1] << 16),
                           ((uint32_t)v[2] & 0xffffu) | ((uint32_t)v[3] << 16),
                           ((uint32_t)v[4] & 0xffffu) | ((uint32_t)v[5] << 16),
                           ((uint32_t)v[6] & 0xffffu) | ((uint32_t)v[7] << 16));
          } else {
            reinterpret_cast<int4 *>(io.out)[(int64_t)(base + o) * nq + q] = make_int4(v[0], v[1], v[2], v[3]);
          }
        }
      }
      __syncwarp();
      written += (unsigned long long)fill;
    };
    const unsigned lt = (1u << lane) - 1u;
    int fill = 0;
    for (long long jb = 0; jb < T; jb += 32) {
      int r = 0;
      int4 E[3];
      const bool ok = eval(jb + lane, r, E);
      const unsigned m = __ballot_sync(0xffffffffu, ok);
      if (ok) {  // stage the row and the new vertices in output column order
        const int slot = fill + __popc(m & lt);
        stage_r[slot] = r;
        int32_t *nv = sv_new + slot * TS;
        const int nb = tail_fast ? w - w_al : 0;  // aligned tail: parent columns [w_al, w) first
        for (int c = 0; c < nb; ++c) nv[c] = RV(r, w_al + c);
#pragma unroll
        for (int p = 0; p < TS; ++p)
          if ((newmask >> p) & 1u) nv[nb + st.colpos[p]] = tcomp(E, p);
      }
      fill += __popc(m);
      if (fill > kWarpStage - 32) {
        warp_flush(fill);
        fill = 0;
      }
    }
    if (fill > 0) warp_flush(fill);
    my_surv = written;
  }
  unsigned long long v3[3] = {my_cand, my_probe, MODE == kModeCount ? my_surv : (lane == 0 ? my_surv : 0ull)};
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
    if (MODE == kModeSingle) io.agg[tile] = v3[2];
  }
}

// ---- table construction
__global__ void k_repack(const int32_t *__restrict__ packed, int64_t rows, int L, int stride,
                         int32_t *__restrict__ out) {
  const int64_t total = rows * stride;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / stride;
    const int c = (int)(t - i * stride);
    out[t] = c < L ? packed[i * L + c] : -1;
  }
}

__global__ void k_arc_count(const int32_t *__restrict__ t, int64_t rows, int stride, const int64_t *__restrict__ off,
                            const int32_t *__restrict__ adj, unsigned long long *__restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ai = arc_index<false>(off, adj, nullptr, t[i * stride], t[i * stride + 1]);
    if (ai >= 0) atomicAdd(cnt + ai, 1ull);
  }
}

int grid_n(int64_t work) {
  int64_t b = (work + 255) / 256;
  return (int)(b < 1 ? 1 : (b > 148 * 16 ? 148 * 16 : b));
}

}  // namespace

int motif_bit(int id) {
  int b = 0;
  while (b < 31 && (1 << b) != id) ++b;
  return b;
}

DevTabStep make_dev_tab_step(const Step &s, const MotifTable &t) {
  DevTabStep d{};
  d.in_w = s.in_w;
  d.n_new = s.n_new;
  d.key0 = s.key0;
  d.key1 = s.key1;
  d.skip = s.skip;
  d.L = t.L;
  d.tstride = t.stride;
  d.trows = t.rows;
  d.n_eq = s.n_eq;
  for (int i = 0; i < s.n_eq; ++i) {
    d.eq_pos[i] = (int8_t)s.eq_pos[i];
    d.eq_col[i] = (uint8_t)s.eq_col[i];
  }
  for (int j = 0; j < s.n_new; ++j) {
    d.newpos[j] = (int8_t)s.newpos[j];
    d.newmask |= 1u << s.newpos[j];
    d.colpos[s.newpos[j]] = (uint8_t)j;
  }
  for (int i = 0; i < s.n_eq; ++i) {
    d.eqmask |= 1u << s.eq_pos[i];
    d.eq_colp[s.eq_pos[i]] = (uint8_t)s.eq_col[i];
  }
  d.n_pr = (int32_t)s.probes.size();
  for (size_t p = 0; p < s.probes.size(); ++p) {
    d.pr_j[p] = (uint8_t)s.probes[p].j;
    d.pr_c[p] = (uint8_t)s.probes[p].col;
    d.pr_neg[p] = (uint8_t)s.probes[p].neg;
  }
  return d;
}

template <int MODE, bool ELL, bool R16>
cudaError_t launch_table_ts(const DevTabStep &st, const StepIO &io, const dm_graph &g, const MotifTable &t,
                            int64_t num_tiles, cudaStream_t s) {
  void (*kern)(const DevTabStep, const StepIO, const int64_t *, const int32_t *, const int32_t *, const int64_t *);
  switch (t.stride) {
    case 4: kern = k_table<MODE, ELL, 4, R16>; break;
    case 8: kern = k_table<MODE, ELL, 8, R16>; break;
    default: kern = k_table<MODE, ELL, 12, R16>; break;
  }
  const int TS = t.stride <= 4 ? 4 : (t.stride <= 8 ? 8 : 12);
  const size_t row_bytes = R16 ? sizeof(uint16_t) * (size_t)smem_stride16(st.in_w)
                               : sizeof(int32_t) * (size_t)smem_stride(st.in_w);
  const size_t smem = row_bytes * (size_t)kTileRows +
                      sizeof(uint32_t) * (size_t)kTileRows * kFiltStride +
                      (MODE != kModeCount ? sizeof(int32_t) * (size_t)(kStepThreads / 32) * kWarpStage * (TS + 1) : 0);
  cudaError_t e = prep((const void *)kern, 0, smem);
  if (e != cudaSuccess) return e;
  kern<<<(unsigned)num_tiles, kStepThreads, smem, s>>>(st, io, g.d_off, g.d_adj, t.d_rows, t.d_toff);
  return cudaGetLastError();
}

cudaError_t launch_table(int mode, const DevTabStep &st, const StepIO &io, const dm_graph &g, const MotifTable &t,
                         int64_t num_tiles, cudaStream_t s) {
  if (num_tiles <= 0 || (io.in_rows <= 0 && !io.d_in_rows)) return cudaSuccess;
  StepIO io2 = io;
  io2.ell = g.d_ell;
  const bool ell = g.d_ell != nullptr;
  const bool r16 = io.elem == 2 && io.in != nullptr;  // 16-bit level kept 16-bit in shared memory
#define DM_TABLE_LAUNCH(M)                                                                   \
  return ell ? (r16 ? launch_table_ts<M, true, true>(st, io2, g, t, num_tiles, s)           \
                    : launch_table_ts<M, true, false>(st, io2, g, t, num_tiles, s))         \
             : (r16 ? launch_table_ts<M, false, true>(st, io2, g, t, num_tiles, s)          \
                    : launch_table_ts<M, false, false>(st, io2, g, t, num_tiles, s))
  if (mode == kModeCount) DM_TABLE_LAUNCH(kModeCount);
  if (mode == kModeSingle) DM_TABLE_LAUNCH(kModeSingle);
  DM_TABLE_LAUNCH(kModeWrite);
#undef DM_TABLE_LAUNCH
}

dm_status finish_motif_table(const dm_graph &g, int32_t *packed, int64_t rows, MotifTable &t, cudaStream_t s) {
  t.stride = row_stride(t.L);
  t.rows = rows;
  // graph-owned buffers come from the stream-ordered pool (released by dm_graph_destroy)
  cudaError_t e = cudaMallocAsync((void **)&t.d_rows, sizeof(int32_t) * (size_t)std::max<int64_t>(rows, 1) * t.stride, s);
  if (e == cudaSuccess) e = cudaMallocAsync((void **)&t.d_toff, sizeof(int64_t) * ((size_t)g.arcs + 1), s);
  unsigned long long *cnt = nullptr;
  void *tmp = nullptr;
  size_t tb = 0;
  if (e == cudaSuccess) e = cudaMallocAsync((void **)&cnt, sizeof(unsigned long long) * ((size_t)g.arcs + 1), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * ((size_t)g.arcs + 1), s);
  if (e == cudaSuccess && rows > 0) {
    k_repack<<<grid_n(rows * t.stride), 256, 0, s>>>(packed, rows, t.L, t.stride, t.d_rows);
    k_arc_count<<<grid_n(rows), 256, 0, s>>>(t.d_rows, rows, t.stride, g.d_off, g.d_adj, cnt);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess)
    e = cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, reinterpret_cast<unsigned long long *>(t.d_toff),
                                      g.arcs + 1, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&tmp, tb, s);
  if (e == cudaSuccess)
    e = cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, reinterpret_cast<unsigned long long *>(t.d_toff),
                                      g.arcs + 1, s);
  if (tmp) cudaFreeAsync(tmp, s);
  if (cnt) cudaFreeAsync(cnt, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    if (t.d_rows) cudaFreeAsync(t.d_rows, s);
    if (t.d_toff) cudaFreeAsync(t.d_toff, s);
    cudaStreamSynchronize(s);
    t.d_rows = nullptr;
    t.d_toff = nullptr;
    return fail(e == cudaErrorMemoryAllocation ? DM_ERR_OOM : DM_ERR_CUDA,
                std::string("motif table: ") + cudaGetErrorString(e));
  }
  return DM_OK;
}

}  // namespace dm
