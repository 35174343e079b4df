// exchange.cuh -- internal declarations of exchange.cu (canonical row sort, partitions).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "dm_internal.h"

namespace dm {

// column map of a gather: out column p = in column c[p]
struct ColMap {
  int32_t c[DM_MAX_PATTERN];
};

// out = the n rows of `in` (in_stride words per row), columns permuted by colmap[0..k), in
// ascending lexicographic order (LSD radix sort over the k columns, stable passes; ids are
// non-negative and < 2^end_bit).  out is packed [n][k]; in and out must not alias.
dm_status lex_sort_rows(const int32_t *in, int64_t n, int64_t in_stride, const int32_t *colmap, int k,
                        int end_bit, int32_t *out, cudaStream_t s);
// bits needed for vertex ids in [0, n_vertices)
int id_bits(int64_t n_vertices);

}  // namespace dm
