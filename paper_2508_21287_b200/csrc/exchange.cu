// exchange.cu -- device helpers for the multi-GPU frontier exchange and the canonical table
// ("each row ... is an independent candidate",
// so any row partition of a level is valid and results are the union of the parts).
//
//   dm_rows_partition_by_work : pack the rows of a level by destination rank, the rank being
//       the row's position in the GLOBAL work prefix (equal-work cut; C2 all-to-all payload);
//   dm_rows_partition_by_key  : pack table rows by the range of one column (the range
//       partition of the canonical table by its first column, C4);
//   dm_table_sort             : lexicographic row order of a [n][k] table,
//       LSD radix sort over the columns (last column first), in place.
// All three are stream-ordered device work; the per-destination counts are read back to the
// host (the collectives that follow need them as split sizes).
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "dm_device.cuh"
#include "exchange.cuh"

namespace dm {
namespace {

int grid_of(int64_t work) {
  int64_t b = (work + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 16));
}

__global__ void k_iota32(uint32_t *p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = (uint32_t)i;
}

// keys[i] = table[perm[i] * stride + col]
__global__ void k_col(const int32_t *__restrict__ t, int64_t stride, int col, const uint32_t *__restrict__ perm,
                      uint32_t *__restrict__ keys, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    keys[i] = (uint32_t)t[(int64_t)perm[i] * stride + col];
}

// out[i][p] = in[perm[i]][cm[p]]  (out packed, k columns)
__global__ void k_rows_gather(const int32_t *__restrict__ in, int64_t in_stride, ColMap cm, int k,
                              const uint32_t *__restrict__ perm, int32_t *__restrict__ out, int64_t n) {
  const int64_t total = n * k;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / k;
    const int p = (int)(t - i * k);
    out[t] = in[(int64_t)perm[i] * in_stride + cm.c[p]];
  }
}

// dest = floor((base + exclusive work prefix) * parts / total), clamped (128-bit product)
__global__ void k_dest_work(const unsigned long long *__restrict__ excl, int64_t n, unsigned long long base,
                            unsigned long long total, int parts, uint32_t *__restrict__ dest,
                            unsigned long long *__restrict__ counts) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    unsigned d = 0;
    if (total) {
      const unsigned __int128 pos = (unsigned __int128)(base + excl[i]) * (unsigned)parts;
      const unsigned __int128 q = pos / total;
      d = q >= (unsigned)parts ? (unsigned)parts - 1 : (unsigned)q;
    }
    dest[i] = d;
    atomicAdd(counts + d, 1ull);
  }
}

// dest = number of splitters <= row[col]   (splitters ascending, parts - 1 of them)
__global__ void k_dest_key(const int32_t *__restrict__ rows, int64_t n, int64_t stride, int col,
                           const int32_t *__restrict__ split, int parts, uint32_t *__restrict__ dest,
                           unsigned long long *__restrict__ counts) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = rows[i * stride + col];
    int lo = 0, hi = parts - 1;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (split[mid] <= v) lo = mid + 1;
      else hi = mid;
    }
    dest[i] = (unsigned)lo;
    atomicAdd(counts + lo, 1ull);
  }
}

// out[i] = rows[perm[i]] (stride words per row)
__global__ void k_row_copy(const int32_t *__restrict__ rows, int64_t stride, const uint32_t *__restrict__ perm,
                           int32_t *__restrict__ out, int64_t n) {
  const int64_t total = n * stride;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / stride, c = t - i * stride;
    out[t] = rows[(int64_t)perm[i] * stride + c];
  }
}

template <typename T>
struct Buf {
  T *p = nullptr;
  cudaStream_t s = nullptr;
  cudaError_t alloc(size_t n, cudaStream_t st) {
    s = st;
    return cudaMallocAsync((void **)&p, sizeof(T) * std::max<size_t>(n, 1), st);
  }
  ~Buf() {
    if (p) cudaFreeAsync(p, s);
  }
};

#define XK(call, what)                                                                  \
  do {                                                                                  \
    cudaError_t _e = (call);                                                            \
    if (_e != cudaSuccess)                                                              \
      return ::dm::fail(_e == cudaErrorMemoryAllocation ? DM_ERR_OOM : DM_ERR_CUDA,           \
                  std::string(what) + ": " + cudaGetErrorString(_e));                   \
  } while (0)

// stable partition of rows by dest (radix sort of (dest, index) pairs), counts to the host
dm_status pack_by_dest(const int32_t *rows, int64_t n, int64_t stride, Buf<uint32_t> &dest,
                       Buf<unsigned long long> &dcnt, int parts, int32_t *out, int64_t *counts,
                       cudaStream_t s) {
  int bits = 1;
  while (bits < 31 && (1ll << bits) < parts) ++bits;
  Buf<uint32_t> dest2, idx, idx2;
  XK(dest2.alloc((size_t)n, s), "partition keys");
  XK(idx.alloc((size_t)n, s), "partition index");
  XK(idx2.alloc((size_t)n, s), "partition index");
  k_iota32<<<grid_of(n), 256, 0, s>>>(idx.p, n);
  XK(cudaGetLastError(), "iota");
  cub::DoubleBuffer<uint32_t> dk(dest.p, dest2.p), dv(idx.p, idx2.p);
  size_t tb = 0;
  XK(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, n, 0, bits, s), "partition sort");
  Buf<unsigned char> tmp;
  XK(tmp.alloc(tb, s), "partition temp");
  XK(cub::DeviceRadixSort::SortPairs(tmp.p, tb, dk, dv, n, 0, bits, s), "partition sort");
  k_row_copy<<<grid_of(n * stride), 256, 0, s>>>(rows, stride, dv.Current(), out, n);
  XK(cudaGetLastError(), "row copy");
  std::vector<unsigned long long> h((size_t)parts);
  XK(cudaMemcpyAsync(h.data(), dcnt.p, sizeof(unsigned long long) * (size_t)parts, cudaMemcpyDeviceToHost, s),
     "D2H counts");
  XK(cudaStreamSynchronize(s), "sync");
  for (int r = 0; r < parts; ++r) counts[r] = (int64_t)h[(size_t)r];
  return DM_OK;
}

// device of a device pointer (the helpers run where the data lives)
bool pointer_device(const void *p, int *dev) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged) return false;
  *dev = a.device;
  return true;
}

}  // namespace

dm_status lex_sort_rows(const int32_t *in, int64_t n, int64_t in_stride, const int32_t *colmap, int k,
                        int end_bit, int32_t *out, cudaStream_t s) {
  if (n <= 0) return DM_OK;
  if (n >= (int64_t)UINT32_MAX) return fail(DM_ERR_ROW_BUDGET, "table too large to sort");
  if (k < 1 || k > DM_MAX_PATTERN) return fail(DM_ERR_ARG, "bad table width");
  Buf<uint32_t> keys, keys2, perm, perm2;
  XK(keys.alloc((size_t)n, s), "sort keys");
  XK(keys2.alloc((size_t)n, s), "sort keys");
  XK(perm.alloc((size_t)n, s), "sort perm");
  XK(perm2.alloc((size_t)n, s), "sort perm");
  k_iota32<<<grid_of(n), 256, 0, s>>>(perm.p, n);
  XK(cudaGetLastError(), "iota");
  cub::DoubleBuffer<uint32_t> dk(keys.p, keys2.p), dv(perm.p, perm2.p);
  size_t tb = 0;
  XK(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, n, 0, end_bit, s), "sort");
  Buf<unsigned char> tmp;
  XK(tmp.alloc(tb, s), "sort temp");
  for (int p = k - 1; p >= 0; --p) {  // LSD: least significant column first, stable passes
    k_col<<<grid_of(n), 256, 0, s>>>(in, in_stride, colmap[p], dv.Current(), dk.Current(), n);
    XK(cudaGetLastError(), "gather");
    XK(cub::DeviceRadixSort::SortPairs(tmp.p, tb, dk, dv, n, 0, end_bit, s), "sort");
  }
  ColMap cm{};
  for (int p = 0; p < k; ++p) cm.c[p] = colmap[p];
  k_rows_gather<<<grid_of(n * k), 256, 0, s>>>(in, in_stride, cm, k, dv.Current(), out, n);
  XK(cudaGetLastError(), "gather rows");
  return DM_OK;
}

int id_bits(int64_t n_vertices) {
  int b = 1;
  while (b < 32 && ((uint64_t)n_vertices >> b) != 0) ++b;
  return b;
}

}  // namespace dm

extern "C" {

dm_status dm_rows_partition_by_work(const int32_t *d_rows, const uint64_t *d_work, int64_t n, int32_t stride,
                                    uint64_t work_base, uint64_t work_total, int32_t parts, int32_t *d_out,
                                    int64_t *counts, void *stream) {
  dm::clear_error();
  if (n < 0 || stride < 1 || parts < 1 || !counts || (n > 0 && (!d_rows || !d_work || !d_out)))
    return dm::fail(DM_ERR_ARG, "bad partition arguments");
  for (int r = 0; r < parts; ++r) counts[r] = 0;
  if (n == 0) return DM_OK;
  int dev = 0;
  if (!dm::pointer_device(d_rows, &dev)) return dm::fail(DM_ERR_ARG, "d_rows is not device memory");
  dm::DeviceGuard dg(dev);
  if (!dg.ok) return dm::fail(DM_ERR_CUDA, "cudaSetDevice failed");
  cudaStream_t s = (cudaStream_t)stream;
  dm::Buf<unsigned long long> excl, dcnt;
  dm::Buf<uint32_t> dest;
  XK(excl.alloc((size_t)n, s), "work prefix");
  XK(dcnt.alloc((size_t)parts, s), "counts");
  XK(dest.alloc((size_t)n, s), "dest");
  XK(cudaMemsetAsync(dcnt.p, 0, sizeof(unsigned long long) * (size_t)parts, s), "memset");
  size_t tb = 0;
  const unsigned long long *w = reinterpret_cast<const unsigned long long *>(d_work);
  XK(cub::DeviceScan::ExclusiveSum(nullptr, tb, w, excl.p, n, s), "scan");
  dm::Buf<unsigned char> tmp;
  XK(tmp.alloc(tb, s), "scan temp");
  XK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, w, excl.p, n, s), "scan");
  dm::k_dest_work<<<dm::grid_of(n), 256, 0, s>>>(excl.p, n, work_base, work_total, parts, dest.p, dcnt.p);
  XK(cudaGetLastError(), "dest kernel");
  return dm::pack_by_dest(d_rows, n, stride, dest, dcnt, parts, d_out, counts, s);
}

dm_status dm_rows_partition_by_key(const int32_t *d_rows, int64_t n, int32_t stride, int32_t col,
                                   const int32_t *splitters, int32_t parts, int32_t *d_out, int64_t *counts,
                                   void *stream) {
  dm::clear_error();
  if (n < 0 || stride < 1 || col < 0 || col >= stride || parts < 1 || !counts ||
      (parts > 1 && !splitters) || (n > 0 && (!d_rows || !d_out)))
    return dm::fail(DM_ERR_ARG, "bad partition arguments");
  for (int r = 1; r + 1 < parts; ++r)
    if (splitters[r] < splitters[r - 1]) return dm::fail(DM_ERR_ARG, "splitters must be ascending");
  for (int r = 0; r < parts; ++r) counts[r] = 0;
  if (n == 0) return DM_OK;
  int dev = 0;
  if (!dm::pointer_device(d_rows, &dev)) return dm::fail(DM_ERR_ARG, "d_rows is not device memory");
  dm::DeviceGuard dg(dev);
  if (!dg.ok) return dm::fail(DM_ERR_CUDA, "cudaSetDevice failed");
  cudaStream_t s = (cudaStream_t)stream;
  dm::Buf<unsigned long long> dcnt;
  dm::Buf<uint32_t> dest;
  dm::Buf<int32_t> dsplit;
  XK(dcnt.alloc((size_t)parts, s), "counts");
  XK(dest.alloc((size_t)n, s), "dest");
  XK(dsplit.alloc((size_t)parts, s), "splitters");
  XK(cudaMemsetAsync(dcnt.p, 0, sizeof(unsigned long long) * (size_t)parts, s), "memset");
  if (parts > 1)
    XK(cudaMemcpyAsync(dsplit.p, splitters, sizeof(int32_t) * (size_t)(parts - 1), cudaMemcpyHostToDevice, s),
       "H2D splitters");
  dm::k_dest_key<<<dm::grid_of(n), 256, 0, s>>>(d_rows, n, stride, col, dsplit.p, parts, dest.p, dcnt.p);
  XK(cudaGetLastError(), "dest kernel");
  return dm::pack_by_dest(d_rows, n, stride, dest, dcnt, parts, d_out, counts, s);
}

dm_status dm_table_sort(int32_t *d_rows, int64_t n, int32_t k, int32_t n_vertices, void *stream) {
  dm::clear_error();
  if (n < 0 || k < 1 || k > DM_MAX_PATTERN || n_vertices < 0 || (n > 0 && !d_rows))
    return dm::fail(DM_ERR_ARG, "bad table arguments");
  if (n <= 1) return DM_OK;
  int dev = 0;
  if (!dm::pointer_device(d_rows, &dev)) return dm::fail(DM_ERR_ARG, "d_rows is not device memory");
  dm::DeviceGuard dg(dev);
  if (!dg.ok) return dm::fail(DM_ERR_CUDA, "cudaSetDevice failed");
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<int32_t> cm((size_t)k);
  for (int p = 0; p < k; ++p) cm[(size_t)p] = p;
  dm::Buf<int32_t> out;
  XK(out.alloc((size_t)n * k, s), "sorted table");
  dm_status st = dm::lex_sort_rows(d_rows, n, k, cm.data(), k, dm::id_bits(n_vertices), out.p, s);
  if (st != DM_OK) return st;
  XK(cudaMemcpyAsync(d_rows, out.p, sizeof(int32_t) * (size_t)n * k, cudaMemcpyDeviceToDevice, s), "copy");
  XK(cudaStreamSynchronize(s), "sync");
  return DM_OK;
}

}  // extern "C"
