// dm_device.cuh -- internal device-side declarations shared by the .cu files of
// libdeltamotif.so (graph builder, join-step kernels, match driver).
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdint>
#include <mutex>
#include <string>

#include "dm_internal.h"

namespace dm {
// A materialized motif table Res(M) (Alg. 2) on the device: every embedding of the
// template (rows = labelled embeddings, columns = template positions), rows in ascending
// lexicographic order, 16-byte row stride (padding -1); the arc index toff[arc] = first row whose
// (position 0, position 1) pair is >= that CSR arc, so the rows keyed by a vertex a are
// [toff[off[a]], toff[off[a+1]]) and those keyed by an arc (a,b) [toff[arc], toff[arc+1]).
struct MotifTable {
  int motif = 0;            // DM_MOTIF_* bit
  int L = 0;                // template vertices
  int stride = 0;           // int32 words per row (round_up(L, 4))
  int64_t rows = 0;
  int32_t *d_rows = nullptr;
  int64_t *d_toff = nullptr;  // [arcs + 1]
  double build_ms = 0.0;
};
// The triangle-apex table (apex.cu): Res(M3-O) keyed by directed edge --
// apex(a,b) = N(a) ∩ N(b) of CSR arc e = (a,b) is d_apex[d_toff[e] .. d_toff[e+1]), each entry
// the arc index of (a, c) (its vertex is adj[entry]), ascending.
struct ApexTable {
  int64_t *d_toff = nullptr;  // [arcs + 1]
  int32_t *d_apex = nullptr;  // [entries]
  int64_t entries = -1;       // -1: not built
  double build_ms = 0.0;
};
struct TabStore {
  std::mutex mu;
  MotifTable t[32];  // by motif bit index
  ApexTable apex;
};
int motif_bit(int id);  // bit index of a DM_MOTIF_* id
}  // namespace dm

struct dm_graph {
  int device = 0;
  int32_t n = 0;
  int64_t arcs = 0;     // 2|E| after dedup
  int32_t max_deg = 0;
  int64_t *d_off = nullptr;  // [n+1]
  int32_t *d_adj = nullptr;  // [arcs], each list sorted ascending
  int32_t *d_ell = nullptr;  // max degree <= 4: [n][4] adjacency (ELL, sorted, -1 padded)
  double sum_d2 = 0.0;       // sum of squared degrees (size-biased degree = sum_d2 / arcs)
  double closure = 0.0;      // sampled P[c in N(a) | a-b-c wedge] (triangle closure)
  uint64_t gen = 0;          // process-unique creation id (keys host-side caches)
  dm::TabStore *tabs = nullptr;  // motif database (Alg. 2), built on demand
};

namespace dm {

#define DM_CUDA(call)                                                                     \
  do {                                                                                    \
    cudaError_t _e = (call);                                                              \
    if (_e != cudaSuccess)                                                                \
      return ::dm::fail(DM_ERR_CUDA, std::string(#call " failed: ") + cudaGetErrorString(_e)); \
  } while (0)

// Restores the caller's current device on scope exit.
struct DeviceGuard {
  int prev = -1;
  bool ok = false;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    ok = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// Device-side bounds checks of the checked build (libdeltamotif_checked.so, -DDM_CHECKED): a
// failed check traps the kernel (the launch then reports an error); compiled out otherwise.
#ifdef DM_CHECKED
#define DM_DCHECK(cond) \
  do {              \
    if (!(cond)) __trap(); \
  } while (0)
#else
#define DM_DCHECK(cond) \
  do {              \
  } while (0)
#endif

// The device's default stream-ordered memory pool keeps freed memory (release threshold = max):
// frontier levels, motif tables and the graph itself are allocated from it, so repeated queries and
// graph create / destroy cycles do not return memory to the driver (graph.cu).
void configure_pool(int device);

// NVTX range for profilers (header-only NVTX v3: free when no tool is attached)
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange &) = delete;
  NvtxRange &operator=(const NvtxRange &) = delete;
};

// ------------------------------------------------------------- join-step kernel interface
constexpr int kStepThreads = 256;   // threads per CTA
constexpr int kTileRows = 256;      // frontier rows per CTA tile
constexpr int kSurvBuf = 1024;      // survivors staged in shared memory per CTA
constexpr int kRowSlotsMax = 4;     // row-serial kernel: max survivor slots per frontier row
constexpr int kRowSerialDeg1 = 16;  // row-serial kernel for 1-vertex steps if max degree <= 16
constexpr int kRowSerialDeg2 = 4;   //   ... and for 2-vertex steps if max degree <= 4
constexpr int kPairSmem = 1024;     // shared-key pair kernel: per-warp list in shared memory
constexpr int kPairBatch = 16;      //   rows claimed per atomic
constexpr int kAccSlots = 64;       // counters are spread over 64 slots (atomic contention)
constexpr int kModeCount = 0;       // join-step kernel launch modes (see extend.cu)
constexpr int kModeWrite = 1;
constexpr int kModeSingle = 2;

// Frontier rows are stored with a 16-byte aligned stride: row_stride(w) int32 words, the
// padding words hold -1 (never a vertex id).
__host__ __device__ inline int row_stride(int w) { return (w + 3) & ~3; }
// 16-bit storage (graphs with n <= 65535, count-only ELL plans): rows of round_up(w, 8) uint16
// ids (16-byte rows, padding 0xFFFF = -1 when widened).  row_words = int32 words per stored row.
__host__ __device__ inline int row_stride16(int w) { return (w + 7) & ~7; }
__host__ __device__ inline int row_words(int w, int elem) {
  return elem == 2 ? row_stride16(w) / 2 : row_stride(w);
}

// Device copy of one executed step (passed by value as a kernel parameter).
struct DevStep {
  int32_t in_w;
  int32_t n_new;
  int32_t n_nbr[kMaxNew];
  int32_t n_non[kMaxNew];
  uint8_t nbr[kMaxNew][DM_MAX_PATTERN];
  uint8_t non[kMaxNew][DM_MAX_PATTERN];
};

struct StepIO {
  const int32_t *in;          // [in_rows][row_stride(in_w)], or nullptr for the implicit seed
  int64_t in_rows;            // rows of this launch's input (chunk)
  int64_t seed_base;          // implicit seed: row r is vertex seed_base + r
  int64_t block_begin;        // first tile index of this launch (chunked write passes)
  int32_t *out;               // write pass: [*][row_stride(in_w + n_new)]
  const uint64_t *block_off;  // write pass: exclusive prefix of survivors per tile (global)
  uint64_t out_base;          // write pass: block_off value that maps to out row 0
  uint64_t *block_cnt;        // count pass: survivors per tile (nullptr -> only total)
  unsigned long long *total;  // count pass: [tile % kAccSlots] += survivors (nullptr -> skip)
  unsigned long long *stats;  // [slot] += candidates, [kAccSlots + slot] += probes (or nullptr)
  unsigned long long *status; // single pass (k_step): look-back status word per tile (zeroed)
  unsigned long long *agg;    // single pass: survivors per tile ([tiles] = 0; exact re-run prefix)
  unsigned long long *ctrl;   // single pass: [0] tile counter, [1] max(#tiles - first tile that
                              //   must be re-run), [2] += survivors / output reservation (zeroed)
  uint64_t cap;               // single pass: output capacity in rows
  const unsigned long long *d_in_rows;  // if set: the input row count, written on the device by
                                        // the previous step (in_rows is then the capacity bound)
  const unsigned long long *d_in_ovf;   // if set: the previous step's overflow flag (its ctrl[1]);
                                        // non-zero -> the input level is incomplete, do nothing
  int32_t slots;              // row-serial kernel: survivor slots per row (set by launch)
  const int32_t *ell;         // row-serial kernel: ELL adjacency (max degree <= 4) or nullptr
  int32_t elem;               // bytes per stored vertex id in `in`: 4 (int32) or 2 (uint16)
  int32_t out_elem;           // bytes per stored vertex id in `out`
};

// Sync-free chaining: resolve the device-written input size.  Returns false when the previous
// level overflowed its capacity (its rows are incomplete: the host re-runs the match on the
// synchronising path); the size is clamped to the capacity the buffer was allocated with.
__device__ __forceinline__ bool resolve_in_rows(StepIO &io) {
  if (!io.d_in_rows) return true;
  if (io.d_in_ovf && *io.d_in_ovf) return false;
  const long long v = (long long)*io.d_in_rows;
  io.in_rows = v < io.in_rows ? v : io.in_rows;
  return true;
}

size_t step_smem_bytes(int in_w, bool write_pass);
cudaError_t launch_step_count(const DevStep &st, const StepIO &io, const dm_graph &g,
                              int64_t num_tiles, cudaStream_t s);
cudaError_t launch_step_write(const DevStep &st, const StepIO &io, const dm_graph &g,
                              int64_t num_tiles, cudaStream_t s);
cudaError_t launch_step_single(const DevStep &st, const StepIO &io, const dm_graph &g,
                               int64_t num_tiles, cudaStream_t s);
int pair_mode_of(const DevStep &st);
bool row_serial_step(const DevStep &st, const dm_graph &g);
// apex: optional triangle-apex table; S is then read from it (rows must satisfy apex_arc_rows)
cudaError_t launch_pairs(const DevStep &st, const StepIO &io, const dm_graph &g, int pair_mode,
                         cudaStream_t s, const ApexTable *apex = nullptr);
// shared-key pair step on the triangle-apex table (apex.cu)
dm_status build_apex_table(const dm_graph *g, cudaStream_t s, ApexTable &t);
bool apex_arc_rows(const DevStep &st, int elem);  // pair step on arc rows keyed on both columns
cudaError_t launch_pairs_apex(const DevStep &st, const StepIO &io, const dm_graph &g, const ApexTable &t,
                              cudaStream_t s);
// deep count-only last step (3..kMaxNew new vertices) on ELL graphs (tail.cu: k_deep)
cudaError_t launch_tail(const DevStep &st, const StepIO &io, const dm_graph &g, int64_t tiles,
                        cudaStream_t s);
// excl[t] = sum of agg[0..t) for t in [0, tiles] (agg[tiles] must be 0)
cudaError_t launch_agg_to_excl(const unsigned long long *agg, int64_t tiles, uint64_t *excl,
                               cudaStream_t s);

DevStep make_dev_step(const Step &st);

// canonical match table [count][k] on the device (match.cu); *d_table is allocated with
// cudaMallocAsync on opt's stream (free it with cudaFreeAsync / cudaFree), NULL when count == 0
dm_status match_device_table(const dm_graph *g, int32_t k, const int32_t *p_edges, int64_t pm,
                             const dm_match_opts *opt, int32_t **d_table, uint64_t *count);

// ---- table steps (tabstep.cu): one slice's fresh vertices joined with Res(M) (Step::tab_motif)
struct DevTabStep {
  int32_t in_w, n_new;
  int32_t key0, key1, skip;  // row columns bound to template positions 0 / 1; known-duplicate column
  int32_t L, tstride;        // template vertices, table row stride (words)
  int64_t trows;             // |Res(M)| (bounds of the checked build)
  int32_t n_eq, n_pr;
  uint32_t newmask;          // bit p: template position p is a new vertex
  uint32_t eqmask;           // bit p: template position p must equal row[eq_colp[p]]
  int8_t newpos[kMaxMotifV];
  int8_t eq_pos[kMaxMotifV];
  uint8_t eq_col[kMaxMotifV];
  uint8_t eq_colp[kMaxMotifV];
  uint8_t colpos[kMaxMotifV];  // new template position p -> new column index (w + colpos[p])
  uint8_t pr_j[kMaxTabProbes], pr_c[kMaxTabProbes], pr_neg[kMaxTabProbes];
};
DevTabStep make_dev_tab_step(const Step &st, const MotifTable &t);
cudaError_t launch_table(int mode, const DevTabStep &st, const StepIO &io, const dm_graph &g,
                         const MotifTable &t, int64_t num_tiles, cudaStream_t s);
// table construction helpers: repack a canonical [rows][L] table to the 16-byte stride and build
// the arc index (tabstep.cu)
dm_status finish_motif_table(const dm_graph &g, int32_t *packed, int64_t rows, MotifTable &t, cudaStream_t s);

}  // namespace dm
