// motifdb.cu -- persistence of the motif database: the Res(M) tables that
// Alg. 2 builds once per data graph are "performed once, cached, and reused"
// (the GPU* protocol), so they can be saved to a file and loaded into a later
// process, bound to the graph by a fingerprint.
//
// File layout (little-endian):
//   header : magic "DMMOTDB1" | uint32 version (1) | uint32 table count
//            | int64 n | int64 arcs | uint64 graph fingerprint
//   table  : int32 motif id | int32 L | int64 rows | int32[rows][L] rows (template order,
//            lexicographic) | int64[arcs + 1] arc index | uint64 FNV-1a of the table payload
//            (the triangle-apex table, id DM_MOTIF_APEX: L = 1, rows = entries, the payload is the
//            entry array (arc indices) and toff)
// The graph fingerprint is FNV-1a over (n, the CSR offsets, the sorted adjacency), i.e. a hash
// of the sorted, deduplicated edge list plus the vertex count (order independent in the input).
#include <cstdio>
#include <cstring>
#include <vector>

#include "dm_device.cuh"

namespace dm {
namespace {

constexpr char kMagic[8] = {'D', 'M', 'M', 'O', 'T', 'D', 'B', '1'};
constexpr uint32_t kVersion = 1;

struct Fnv {
  uint64_t h = 1469598103934665603ull;
  void add(const void *p, size_t n) {
    const unsigned char *c = static_cast<const unsigned char *>(p);
    for (size_t i = 0; i < n; ++i) {
      h ^= c[i];
      h *= 1099511628211ull;
    }
  }
};

dm_status graph_fingerprint(const dm_graph *g, uint64_t &out) {
  std::vector<int64_t> off((size_t)g->n + 1);
  std::vector<int32_t> adj((size_t)std::max<int64_t>(g->arcs, 1));
  DeviceGuard dg(g->device);
  if (!dg.ok) return fail(DM_ERR_CUDA, "cudaSetDevice failed");
  DM_CUDA(cudaMemcpy(off.data(), g->d_off, sizeof(int64_t) * off.size(), cudaMemcpyDeviceToHost));
  if (g->arcs > 0) DM_CUDA(cudaMemcpy(adj.data(), g->d_adj, sizeof(int32_t) * (size_t)g->arcs, cudaMemcpyDeviceToHost));
  Fnv f;
  const int64_t n = g->n;
  f.add(&n, sizeof(n));
  f.add(off.data(), sizeof(int64_t) * off.size());
  f.add(adj.data(), sizeof(int32_t) * (size_t)g->arcs);
  out = f.h;
  return DM_OK;
}

struct File {
  FILE *f = nullptr;
  ~File() {
    if (f) std::fclose(f);
  }
};

bool rd(FILE *f, void *p, size_t n, Fnv *h = nullptr) {
  if (n == 0) return true;
  if (std::fread(p, 1, n, f) != n) return false;
  if (h) h->add(p, n);
  return true;
}
bool wr(FILE *f, const void *p, size_t n, Fnv *h = nullptr) {
  if (n == 0) return true;
  if (h) h->add(p, n);
  return std::fwrite(p, 1, n, f) == n;
}

}  // namespace
}  // namespace dm

extern "C" {

dm_status dm_graph_save_motifs(const dm_graph *g, const char *path) {
  dm::clear_error();
  if (!g || !path) return dm::fail(DM_ERR_ARG, "NULL argument");
  uint64_t fp = 0;
  dm_status st = dm::graph_fingerprint(g, fp);
  if (st != DM_OK) return st;
  std::vector<dm::MotifTable> tabs;
  {
    std::lock_guard<std::mutex> lk(g->tabs->mu);
    for (auto &t : g->tabs->t)
      if (t.d_toff) tabs.push_back(t);
    const dm::ApexTable &ap = g->tabs->apex;
    if (ap.entries >= 0) {  // written like a one-column table: rows = entries
      dm::MotifTable t;
      t.motif = DM_MOTIF_APEX;
      t.L = 1;
      t.stride = 1;
      t.rows = ap.entries;
      t.d_rows = ap.d_apex;
      t.d_toff = ap.d_toff;
      tabs.push_back(t);
    }
  }
  const std::string tmp = std::string(path) + ".tmp";
  dm::File F;
  F.f = std::fopen(tmp.c_str(), "wb");
  if (!F.f) return dm::fail(DM_ERR_IO, std::string("cannot open ") + tmp + " for writing");
  const uint32_t ntab = (uint32_t)tabs.size();
  const int64_t n = g->n, arcs = g->arcs;
  bool ok = dm::wr(F.f, dm::kMagic, 8) && dm::wr(F.f, &dm::kVersion, 4) && dm::wr(F.f, &ntab, 4) &&
            dm::wr(F.f, &n, 8) && dm::wr(F.f, &arcs, 8) && dm::wr(F.f, &fp, 8);
  dm::DeviceGuard dg(g->device);
  for (const auto &t : tabs) {
    if (!ok) break;
    std::vector<int32_t> rows((size_t)t.rows * t.stride);
    std::vector<int64_t> toff((size_t)arcs + 1);
    if (t.rows > 0 && cudaMemcpy(rows.data(), t.d_rows, sizeof(int32_t) * rows.size(), cudaMemcpyDeviceToHost) != cudaSuccess)
      return dm::fail(DM_ERR_CUDA, "D2H motif table");
    if (cudaMemcpy(toff.data(), t.d_toff, sizeof(int64_t) * toff.size(), cudaMemcpyDeviceToHost) != cudaSuccess)
      return dm::fail(DM_ERR_CUDA, "D2H motif index");
    std::vector<int32_t> packed;
    if (t.stride == t.L) {
      packed.swap(rows);
    } else {
      packed.resize((size_t)t.rows * t.L);
      for (int64_t i = 0; i < t.rows; ++i)
        std::memcpy(packed.data() + i * t.L, rows.data() + i * t.stride, sizeof(int32_t) * (size_t)t.L);
    }
    dm::Fnv h;
    const int32_t id = t.motif, L = t.L;
    const int64_t R = t.rows;
    ok = dm::wr(F.f, &id, 4, &h) && dm::wr(F.f, &L, 4, &h) && dm::wr(F.f, &R, 8, &h) &&
         dm::wr(F.f, packed.data(), sizeof(int32_t) * packed.size(), &h) &&
         dm::wr(F.f, toff.data(), sizeof(int64_t) * toff.size(), &h);
    ok = ok && dm::wr(F.f, &h.h, 8);
  }
  if (!ok) return dm::fail(DM_ERR_IO, std::string("write failed: ") + tmp);
  std::fclose(F.f);
  F.f = nullptr;
  if (std::rename(tmp.c_str(), path) != 0) return dm::fail(DM_ERR_IO, std::string("cannot rename to ") + path);
  return DM_OK;
}

dm_status dm_graph_load_motifs(dm_graph *g, const char *path) {
  dm::clear_error();
  if (!g || !path) return dm::fail(DM_ERR_ARG, "NULL argument");
  dm::File F;
  F.f = std::fopen(path, "rb");
  if (!F.f) return dm::fail(DM_ERR_IO, std::string("cannot open ") + path);
  char magic[8];
  uint32_t ver = 0, ntab = 0;
  int64_t n = 0, arcs = 0;
  uint64_t fp = 0;
  if (!dm::rd(F.f, magic, 8) || std::memcmp(magic, dm::kMagic, 8) != 0 || !dm::rd(F.f, &ver, 4) ||
      ver != dm::kVersion || !dm::rd(F.f, &ntab, 4) || !dm::rd(F.f, &n, 8) || !dm::rd(F.f, &arcs, 8) ||
      !dm::rd(F.f, &fp, 8) || ntab > 32)
    return dm::fail(DM_ERR_IO, "corrupt motif database file (header)");
  uint64_t mine = 0;
  dm_status st = dm::graph_fingerprint(g, mine);
  if (st != DM_OK) return st;
  if (n != g->n || arcs != g->arcs || fp != mine)
    return dm::fail(DM_ERR_ARG, "motif database fingerprint mismatch: it was built for another graph (stale cache)");
  std::vector<dm::MotifTable> loaded;
  auto drop = [&]() {
    for (auto &t : loaded) {
      if (t.d_rows) cudaFreeAsync(t.d_rows, nullptr);
      if (t.d_toff) cudaFreeAsync(t.d_toff, nullptr);
    }
  };
  dm::DeviceGuard dg(g->device);
  for (uint32_t i = 0; i < ntab; ++i) {
    dm::Fnv h;
    int32_t id = 0, L = 0;
    int64_t R = 0;
    if (!dm::rd(F.f, &id, 4, &h) || !dm::rd(F.f, &L, 4, &h) || !dm::rd(F.f, &R, 8, &h) ||
        !(id == DM_MOTIF_APEX ? L == 1 && R >= 0
                              : (dm::motif_def(id) && dm::motif_is_table(id) && dm::motif_def(id)->nv == L && R >= 0 &&
                                 R <= (int64_t)INT32_MAX))) {
      drop();
      return dm::fail(DM_ERR_IO, "corrupt motif database file (table header)");
    }
    std::vector<int32_t> packed((size_t)R * L);
    std::vector<int64_t> toff((size_t)arcs + 1);
    uint64_t sum = 0;
    if (!dm::rd(F.f, packed.data(), sizeof(int32_t) * packed.size(), &h) ||
        !dm::rd(F.f, toff.data(), sizeof(int64_t) * toff.size(), &h) || !dm::rd(F.f, &sum, 8) || sum != h.h ||
        toff.back() != R) {
      drop();
      return dm::fail(DM_ERR_IO, "corrupt motif database file (truncated or checksum mismatch)");
    }
    dm::MotifTable t;
    t.motif = id;
    t.L = L;
    t.stride = id == DM_MOTIF_APEX ? 1 : dm::row_stride(L);
    t.rows = R;
    std::vector<int32_t> rows;
    if (t.stride == L) {
      rows.swap(packed);
    } else {
      rows.assign((size_t)R * t.stride, -1);
      for (int64_t r = 0; r < R; ++r)
        std::memcpy(rows.data() + r * t.stride, packed.data() + r * L, sizeof(int32_t) * (size_t)L);
    }
    // graph-owned buffers come from the stream-ordered pool (legacy stream: ordered before the
    // synchronous copies below; released by dm_graph_destroy)
    if (cudaMallocAsync((void **)&t.d_rows, sizeof(int32_t) * std::max<size_t>(rows.size(), 1), nullptr) != cudaSuccess ||
        cudaMallocAsync((void **)&t.d_toff, sizeof(int64_t) * toff.size(), nullptr) != cudaSuccess ||
        (R > 0 && cudaMemcpy(t.d_rows, rows.data(), sizeof(int32_t) * rows.size(), cudaMemcpyHostToDevice) != cudaSuccess) ||
        cudaMemcpy(t.d_toff, toff.data(), sizeof(int64_t) * toff.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
      if (t.d_rows) cudaFreeAsync(t.d_rows, nullptr);
      if (t.d_toff) cudaFreeAsync(t.d_toff, nullptr);
      drop();
      return dm::fail(DM_ERR_OOM, "device allocation for a loaded motif table failed");
    }
    loaded.push_back(t);
  }
  std::lock_guard<std::mutex> lk(g->tabs->mu);
  for (auto &t : loaded) {
    if (t.motif == DM_MOTIF_APEX) {
      dm::ApexTable &ap = g->tabs->apex;
      if (ap.entries >= 0) {  // already built: keep the resident one
        if (t.d_rows) cudaFreeAsync(t.d_rows, nullptr);
        if (t.d_toff) cudaFreeAsync(t.d_toff, nullptr);
        continue;
      }
      ap.d_apex = t.d_rows;
      ap.d_toff = t.d_toff;
      ap.entries = t.rows;
      ap.build_ms = 0.0;
      continue;
    }
    dm::MotifTable &slot = g->tabs->t[dm::motif_bit(t.motif)];
    if (slot.d_toff) {  // already built: keep the resident one
      if (t.d_rows) cudaFreeAsync(t.d_rows, nullptr);
      if (t.d_toff) cudaFreeAsync(t.d_toff, nullptr);
      continue;
    }
    t.build_ms = 0.0;
    slot = t;
  }
  return DM_OK;
}

}  // extern "C"
