"""paper_2508_21287_b200 -- B200-native hot path of Delta-Motif (arXiv 2508.21287).

Thin ctypes binding over ``libdeltamotif.so`` (C ABI declared in ``include/deltamotif.h``).
This module only marshals arguments: graph construction, planning, every join step, the
filters and the canonical sort all run inside the library (CUDA kernels for sm_100a plus the
host planner).  There is no CPU fallback: if the library is missing or no CUDA device is
present, the calls raise.

    import paper_2508_21287_b200 as dm
    g = dm.Graph(n, edges)                       # dm_graph_create  (device CSR, Res(M2))
    r = g.match(k, pattern_edges, output="table")   # dm_match
    r.count, r.rows, r.stats
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# DM_LIBRARY_VARIANT=checked loads the bounds-checked build (device asserts trap on a bad index)
LIB_PATH = os.path.join(_HERE, "libdeltamotif_checked.so" if os.environ.get("DM_LIBRARY_VARIANT") == "checked"
                        else "libdeltamotif.so")

DM_OK = 0
ERRORS = {-1: "DM_ERR_ARG", -2: "DM_ERR_VERTEX_RANGE", -3: "DM_ERR_SELF_LOOP",
          -4: "DM_ERR_PATTERN_DISCONNECTED", -5: "DM_ERR_OOM", -6: "DM_ERR_ROW_BUDGET",
          -7: "DM_ERR_CUDA", -8: "DM_ERR_UNSUPPORTED", -9: "DM_ERR_IO"}
DM_MONO, DM_INDUCED = 0, 1
DM_OUT_COUNT, DM_OUT_TABLE = 1, 2
DM_MOTIF_M2, DM_MOTIF_M3, DM_MOTIF_M3O = 1, 2, 4
MOTIF_BITS = {"M2": 1, "M3": 2, "M3-O": 4, "M4": 8, "M5": 16, "M6": 32, "M7": 64, "M8": 128,
              "M4-O": 256, "M6-O": 512, "M12-O": 1024, "apex": 2048}
MOTIF_NAMES = {v: k for k, v in MOTIF_BITS.items()}
DM_MAX_MOTIF_VERTICES = 12
DM_GRAPH_DROP_SELF_LOOPS = 1
DM_MATCH_PROFILE = 1
DM_MAX_PATTERN = 128
DM_MAX_STEPS = 128
ABI_VERSION = 4
DM_MOTIF_APEX = 2048

MOTIF_SETS = {
    "all": DM_MOTIF_M2 | DM_MOTIF_M3 | DM_MOTIF_M3O,   # the implicit (CSR-joined) motifs
    "M2": DM_MOTIF_M2,
    "M3": DM_MOTIF_M2 | DM_MOTIF_M3,
    "M3O": DM_MOTIF_M2 | DM_MOTIF_M3O,
    # the paper's topology-aware sets: heavy-hex {M2, M4}, square grid {M2, M4-O, M6-O}
    "heavy-hex": DM_MOTIF_M2 | 8,
    "grid": DM_MOTIF_M2 | 256 | 512,
    # implicit motifs + the triangle-apex table (Res(M3-O) keyed by arc) for pair steps
    "apex": DM_MOTIF_M2 | DM_MOTIF_M3 | DM_MOTIF_M3O | 2048,
}


class DMError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


class _Opts(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("output", ctypes.c_int32), ("motifs", ctypes.c_int32),
                ("flags", ctypes.c_int32), ("row_budget", ctypes.c_uint64),
                ("mem_budget", ctypes.c_uint64), ("seed_begin", ctypes.c_int64),
                ("seed_end", ctypes.c_int64), ("cuda_stream", ctypes.c_void_p)]


class _Stats(ctypes.Structure):
    _fields_ = [("num_steps", ctypes.c_int32), ("num_launches", ctypes.c_int32),
                ("num_chunks", ctypes.c_int32), ("elem_bytes", ctypes.c_int32),
                ("rows_in", ctypes.c_uint64 * DM_MAX_STEPS),
                ("rows_out", ctypes.c_uint64 * DM_MAX_STEPS),
                ("candidates", ctypes.c_uint64 * DM_MAX_STEPS),
                ("probes", ctypes.c_uint64 * DM_MAX_STEPS),
                ("width_in", ctypes.c_int32 * DM_MAX_STEPS),
                ("width_out", ctypes.c_int32 * DM_MAX_STEPS),
                ("bytes_model", ctypes.c_double * DM_MAX_STEPS),
                ("bytes_stored", ctypes.c_double * DM_MAX_STEPS),
                ("ms_count", ctypes.c_double * DM_MAX_STEPS),
                ("ms_write", ctypes.c_double * DM_MAX_STEPS),
                ("ms_other", ctypes.c_double), ("ms_total", ctypes.c_double),
                ("pipelined", ctypes.c_int32), ("reserved", ctypes.c_int32)]


_lib = None

# every symbol include/deltamotif.h declares (checked by tests/test_abi.py)
EXPORTS = ["dm_match_opts_init", "dm_abi_version", "dm_graph_create", "dm_graph_destroy",
           "dm_graph_num_vertices", "dm_graph_num_arcs", "dm_graph_max_degree",
           "dm_graph_device", "dm_graph_stats", "dm_graph_device_csr", "dm_graph_copy_csr", "dm_match",
           "dm_result_count", "dm_result_width", "dm_result_rows", "dm_result_stats",
           "dm_result_free", "dm_last_error", "dm_plan_create", "dm_plan_create_ex", "dm_plan_destroy",
           "dm_plan_num_slices", "dm_plan_slice", "dm_plan_num_steps", "dm_plan_first_vertex",
           "dm_plan_describe", "dm_match_prefix", "dm_frontier_rows", "dm_frontier_width",
           "dm_frontier_stride", "dm_frontier_device_rows", "dm_frontier_device_work",
           "dm_frontier_free", "dm_match_resume", "dm_frontier_work_total", "dm_plan_create_for",
           "dm_plan_width", "dm_plan_stride", "dm_plan_column_vertex", "dm_plan_seed_work",
           "dm_plan_seed_cuts", "dm_plan_seed", "dm_plan_step", "dm_plan_finish_table", "dm_plan_run",
           "dm_rows_partition_by_work", "dm_rows_partition_by_key", "dm_table_sort",
           "dm_graph_build_motifs", "dm_graph_motif_rows", "dm_graph_motif_build_ms", "dm_graph_motif_table",
           "dm_graph_save_motifs", "dm_graph_load_motifs", "dm_score_layouts",
           "dm_graph_apex_entries", "dm_graph_apex_build_ms", "dm_graph_apex_table"]


def lib():
    """Load libdeltamotif.so (raises loudly when it is missing: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
                          " (paper_2508_21287_b200 has no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    c = ctypes
    P = c.c_void_p
    sig = {
        "dm_match_opts_init": (None, [c.POINTER(_Opts)]),
        "dm_abi_version": (c.c_int32, []),
        "dm_graph_create": (c.c_int, [c.c_int32, P, c.c_int64, c.c_int32, c.c_int32, c.POINTER(P)]),
        "dm_graph_destroy": (None, [P]),
        "dm_graph_num_vertices": (c.c_int32, [P]),
        "dm_graph_num_arcs": (c.c_int64, [P]),
        "dm_graph_max_degree": (c.c_int32, [P]),
        "dm_graph_device": (c.c_int32, [P]),
        "dm_graph_stats": (c.c_int, [P, c.POINTER(c.c_double), c.POINTER(c.c_double)]),
        "dm_graph_device_csr": (c.c_int, [P, c.POINTER(P), c.POINTER(P)]),
        "dm_graph_copy_csr": (c.c_int, [P, P, P]),
        "dm_match": (c.c_int, [P, c.c_int32, P, c.c_int64, c.POINTER(_Opts), c.POINTER(P)]),
        "dm_result_count": (c.c_uint64, [P]),
        "dm_result_width": (c.c_int32, [P]),
        "dm_result_rows": (P, [P]),
        "dm_result_stats": (c.c_int, [P, c.POINTER(_Stats)]),
        "dm_result_free": (None, [P]),
        "dm_last_error": (c.c_char_p, []),
        "dm_plan_create": (c.c_int, [c.c_int32, P, c.c_int64, c.c_int32, c.c_int32, c.POINTER(P)]),
        "dm_plan_create_ex": (c.c_int, [c.c_int32, P, c.c_int64, c.c_int32, c.c_int32, c.c_double,
                                        c.c_double, c.c_double, c.c_double, c.c_int32, c.c_int32,
                                        c.POINTER(P)]),
        "dm_plan_destroy": (None, [P]),
        "dm_plan_num_slices": (c.c_int32, [P]),
        "dm_plan_slice": (c.c_int, [P, c.c_int32, c.POINTER(c.c_int32), c.POINTER(c.c_int32),
                                    c.POINTER(c.c_int32), c.POINTER(c.c_int32),
                                    c.POINTER(c.c_int32)]),
        "dm_plan_num_steps": (c.c_int32, [P]),
        "dm_plan_first_vertex": (c.c_int32, [P]),
        "dm_plan_describe": (c.c_int64, [P, c.c_char_p, c.c_int64]),
        "dm_match_prefix": (c.c_int, [P, c.c_int32, P, c.c_int64, c.POINTER(_Opts), c.c_int32,
                                      c.POINTER(P)]),
        "dm_frontier_rows": (c.c_int64, [P]),
        "dm_frontier_width": (c.c_int32, [P]),
        "dm_frontier_stride": (c.c_int32, [P]),
        "dm_frontier_device_rows": (P, [P]),
        "dm_frontier_device_work": (P, [P]),
        "dm_frontier_free": (None, [P]),
        "dm_match_resume": (c.c_int, [P, c.c_int32, P, c.c_int64, c.POINTER(_Opts), c.c_int32, P,
                                      c.c_int64, c.POINTER(P)]),
        "dm_frontier_work_total": (c.c_uint64, [P]),
        "dm_plan_create_for": (c.c_int, [P, c.c_int32, P, c.c_int64, c.POINTER(_Opts), c.POINTER(P)]),
        "dm_plan_width": (c.c_int32, [P, c.c_int32]),
        "dm_plan_stride": (c.c_int32, [P, c.c_int32]),
        "dm_plan_column_vertex": (c.c_int32, [P, c.c_int32]),
        "dm_plan_seed_work": (c.c_int, [P, P, c.c_int64, c.c_int64, P]),
        "dm_plan_seed_cuts": (c.c_int, [P, P, c.c_int32, P]),
        "dm_plan_seed": (c.c_int, [P, P, c.POINTER(_Opts), c.POINTER(P)]),
        "dm_plan_step": (c.c_int, [P, P, c.POINTER(_Opts), c.c_int32, P, c.c_int64, c.POINTER(P),
                                   c.POINTER(c.c_uint64)]),
        "dm_plan_finish_table": (c.c_int, [P, P, c.POINTER(_Opts), P, c.c_int64, P]),
        "dm_plan_run": (c.c_int, [P, P, c.POINTER(_Opts), c.POINTER(P)]),
        "dm_rows_partition_by_work": (c.c_int, [P, P, c.c_int64, c.c_int32, c.c_uint64, c.c_uint64,
                                                c.c_int32, P, P, P]),
        "dm_rows_partition_by_key": (c.c_int, [P, c.c_int64, c.c_int32, c.c_int32, P, c.c_int32, P, P,
                                               P]),
        "dm_table_sort": (c.c_int, [P, c.c_int64, c.c_int32, c.c_int32, P]),
        "dm_graph_build_motifs": (c.c_int, [P, c.c_int32, c.POINTER(_Opts)]),
        "dm_graph_motif_rows": (c.c_int64, [P, c.c_int32]),
        "dm_graph_motif_build_ms": (c.c_double, [P, c.c_int32]),
        "dm_graph_motif_table": (c.c_int, [P, c.c_int32, P, P]),
        "dm_graph_save_motifs": (c.c_int, [P, c.c_char_p]),
        "dm_graph_apex_entries": (c.c_int64, [P]),
        "dm_graph_apex_build_ms": (c.c_double, [P]),
        "dm_graph_apex_table": (c.c_int, [P, P, P]),
        "dm_graph_load_motifs": (c.c_int, [P, c.c_char_p]),
        "dm_score_layouts": (c.c_int, [P, c.c_int32, P, c.c_int64, P, P, P, c.c_int64, c.POINTER(_Opts),
                                       c.c_int64, P, P, c.POINTER(c.c_int64), c.POINTER(c.c_uint64)]),
    }
    for name, (rt, args) in sig.items():
        f = getattr(L, name)
        f.restype = rt
        f.argtypes = args
    if L.dm_abi_version() != ABI_VERSION:
        raise ImportError("libdeltamotif.so ABI version mismatch; rebuild")
    _lib = L
    return L


def _check(rc: int):
    if rc != DM_OK:
        raise DMError(rc, (lib().dm_last_error() or b"").decode())


def _edges_arr(edges) -> np.ndarray:
    e = np.ascontiguousarray(np.asarray(edges, dtype=np.int32).reshape(-1, 2))
    return e


def _motifs(m) -> int:
    """Motif set: a MOTIF_SETS name, a comma list of motif names ("M2,M3,M5"), or a bitmask."""
    if isinstance(m, str):
        if m in MOTIF_SETS:
            return MOTIF_SETS[m]
        bits = 0
        for name in m.split(","):
            bits |= MOTIF_BITS[name.strip()]
        return bits
    return int(m)


def _check_rows(rows, graph, stride: int):
    """Device rows handed to the library: int32, contiguous, on the graph's device, [n][stride]."""
    import torch
    if not isinstance(rows, torch.Tensor):
        raise TypeError("rows must be a torch tensor")
    if rows.dtype != torch.int32 or not rows.is_cuda or not rows.is_contiguous():
        raise ValueError("rows must be a contiguous int32 CUDA tensor")
    if graph is not None and rows.device.index != lib().dm_graph_device(graph._h):
        raise ValueError("rows live on another device than the graph")
    if rows.dim() != 2 or int(rows.shape[1]) != int(stride):
        raise ValueError(f"rows must have shape [n, {stride}] (got {tuple(rows.shape)})")


def _stream_ptr(stream):
    if stream is None:
        return None
    return int(getattr(stream, "cuda_stream", stream))


# ------------------------------------------------------------------- exchange (§8(e))
def partition_by_work(rows, work, work_base: int, work_total: int, parts: int, *, stream=None):
    """dm_rows_partition_by_work: rows grouped by destination part (equal-work position in the
    global work order); returns (packed CUDA tensor, per-part row counts)."""
    import torch
    _check_rows(rows, None, int(rows.shape[1]) if rows.dim() == 2 else -1)
    n = int(rows.shape[0])
    out = torch.empty_like(rows)
    counts = np.zeros(int(parts), dtype=np.int64)
    if n:
        if work is None or work.dtype != torch.int64 or not work.is_cuda or work.shape != (n,):
            raise ValueError("work must be an int64 CUDA tensor [n]")
    _check(lib().dm_rows_partition_by_work(rows.data_ptr() if n else None, work.data_ptr() if n else None, n,
                                           int(rows.shape[1]), int(work_base), int(work_total), int(parts),
                                           out.data_ptr() if n else None, counts.ctypes.data, _stream_ptr(stream)))
    return out, [int(c) for c in counts]


def partition_by_key(rows, col: int, splitters, parts: int, *, stream=None):
    """dm_rows_partition_by_key: rows grouped by the range of column `col` (range partition)."""
    import torch
    _check_rows(rows, None, int(rows.shape[1]) if rows.dim() == 2 else -1)
    n = int(rows.shape[0])
    out = torch.empty_like(rows)
    sp = np.ascontiguousarray(np.asarray(splitters, dtype=np.int32).reshape(-1))
    if sp.size != int(parts) - 1:
        raise ValueError("need parts - 1 splitters")
    counts = np.zeros(int(parts), dtype=np.int64)
    _check(lib().dm_rows_partition_by_key(rows.data_ptr() if n else None, n, int(rows.shape[1]), int(col),
                                          sp.ctypes.data if sp.size else None, int(parts),
                                          out.data_ptr() if n else None, counts.ctypes.data, _stream_ptr(stream)))
    return out, [int(c) for c in counts]


def table_sort(rows, n_vertices: int, *, stream=None):
    """dm_table_sort: lexicographic row order of a CUDA int32 [n][k] table, in place."""
    _check_rows(rows, None, int(rows.shape[1]) if rows.dim() == 2 else -1)
    n = int(rows.shape[0])
    _check(lib().dm_table_sort(rows.data_ptr() if n else None, n, int(rows.shape[1]), int(n_vertices),
                               _stream_ptr(stream)))
    return rows


# ------------------------------------------------------------------------------- plans
class Plan:
    """Host join program (dm_plan_create): the §3.3 decomposition and the executed steps."""

    def __init__(self, k: int, p_edges, motifs="all", mode: str = "mono", stats=None):
        """stats: optional dict(n, arcs, sum_d2, closure, max_degree, count_only) for the cost
        model (dm_plan_create_ex); default = dm_plan_create's sparse-lattice defaults."""
        L = lib()
        pe = _edges_arr(p_edges)
        h = ctypes.c_void_p()
        md = DM_INDUCED if mode == "induced" else DM_MONO
        if stats is None:
            _check(L.dm_plan_create(k, pe.ctypes.data if pe.size else None, pe.shape[0],
                                    _motifs(motifs), md, ctypes.byref(h)))
        else:
            _check(L.dm_plan_create_ex(k, pe.ctypes.data if pe.size else None, pe.shape[0],
                                       _motifs(motifs), md, float(stats["n"]), float(stats["arcs"]),
                                       float(stats["sum_d2"]), float(stats.get("closure", 0.0)),
                                       int(stats.get("max_degree", 1 << 30)),
                                       int(bool(stats.get("count_only", False))), ctypes.byref(h)))
        self._h = h

    @classmethod
    def for_graph(cls, graph: "Graph", k: int, p_edges, *, mode: str = "mono", output: str = "count",
                  motifs="all") -> "Plan":
        """dm_plan_create_for: the plan dm_match executes for (graph, pattern, options)."""
        pe = _edges_arr(p_edges)
        o = graph._opts(mode, output, motifs, None, None, False, 0, 0)
        h = ctypes.c_void_p()
        _check(lib().dm_plan_create_for(graph._h, int(k), pe.ctypes.data if pe.size else None,
                                        pe.shape[0], ctypes.byref(o), ctypes.byref(h)))
        self = cls.__new__(cls)
        self._h = h
        self.k = int(k)
        self.mode, self.motifs = mode, motifs
        return self

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.dm_plan_destroy(self._h)
            self._h = None

    # ---- step-level execution (dm_plan_*)
    def width(self, level: int) -> int:
        return int(lib().dm_plan_width(self._h, int(level)))

    def stride(self, level: int) -> int:
        return int(lib().dm_plan_stride(self._h, int(level)))

    def column_vertex(self, column: int) -> int:
        return int(lib().dm_plan_column_vertex(self._h, int(column)))

    def seed_work(self, graph: "Graph", seed_begin: int = 0, seed_end: int = -1) -> np.ndarray:
        n = graph.n if seed_end < 0 else int(seed_end)
        out = np.zeros(n - int(seed_begin) + 1, dtype=np.uint64)
        _check(lib().dm_plan_seed_work(graph._h, self._h, int(seed_begin), int(seed_end), out.ctypes.data))
        return out

    def seed_cuts(self, graph: "Graph", parts: int) -> list:
        out = np.zeros(int(parts) + 1, dtype=np.int64)
        _check(lib().dm_plan_seed_cuts(graph._h, self._h, int(parts), out.ctypes.data))
        return [int(x) for x in out]

    def step(self, graph: "Graph", step: int, rows=None, *, seed_range=None, stream=None,
             materialize: bool = True):
        """dm_plan_step: level step+1 as a Frontier (materialize=True), or the count of the
        count-only last step (materialize=False).  rows: CUDA int32 [n][stride(step)] tensor
        (None for step 0: the implicit seed over seed_range)."""
        o = graph._opts("mono", "count", "all", seed_range, stream, False, 0, 0)
        ptr, n = None, 0
        if rows is not None:
            _check_rows(rows, graph, self.stride(step))
            n = int(rows.shape[0])
            ptr = rows.data_ptr() if n else None
        cnt = ctypes.c_uint64(0)
        if materialize:
            h = ctypes.c_void_p()
            _check(lib().dm_plan_step(graph._h, self._h, ctypes.byref(o), int(step), ptr, n, ctypes.byref(h),
                                      ctypes.byref(cnt)))
            return Frontier(h)
        _check(lib().dm_plan_step(graph._h, self._h, ctypes.byref(o), int(step), ptr, n, None, ctypes.byref(cnt)))
        return int(cnt.value)

    def seed(self, graph: "Graph", *, seed_range=None, stream=None) -> "Frontier":
        return self.step(graph, 0, None, seed_range=seed_range, stream=stream)

    def finish_table(self, graph: "Graph", rows, *, stream=None):
        """dm_plan_finish_table: final-level rows -> canonical CUDA tensor [n][k]."""
        import torch
        _check_rows(rows, graph, self.stride(self.num_steps))
        n = int(rows.shape[0])
        k = self.width(self.num_steps)
        out = torch.empty((n, k), dtype=torch.int32, device=rows.device)
        o = graph._opts("mono", "count", "all", None, stream, False, 0, 0)
        _check(lib().dm_plan_finish_table(graph._h, self._h, ctypes.byref(o), rows.data_ptr() if n else None, n,
                                          out.data_ptr() if n else None))
        return out

    def run(self, graph: "Graph", *, output: str = "count", seed_range=None, stream=None,
            profile: bool = False) -> "Result":
        """dm_plan_run: dm_match with this plan."""
        o = graph._opts(getattr(self, "mode", "mono"), output, "all", seed_range, stream, profile, 0, 0)
        r = ctypes.c_void_p()
        _check(lib().dm_plan_run(graph._h, self._h, ctypes.byref(o), ctypes.byref(r)))
        return graph._result(r, self.width(self.num_steps), output)

    @property
    def num_steps(self) -> int:
        return lib().dm_plan_num_steps(self._h)

    @property
    def first_vertex(self) -> int:
        return lib().dm_plan_first_vertex(self._h)

    def slices(self):
        L = lib()
        out = []
        names = MOTIF_NAMES
        for i in range(L.dm_plan_num_slices(self._h)):
            m, nv, nc = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
            vs = (ctypes.c_int32 * DM_MAX_MOTIF_VERTICES)()
            cs = (ctypes.c_int32 * DM_MAX_MOTIF_VERTICES)()
            _check(L.dm_plan_slice(self._h, i, ctypes.byref(m), ctypes.byref(nv), vs, ctypes.byref(nc), cs))
            out.append({"motif": names[m.value], "vertices": list(vs)[:nv.value],
                        "constraints": list(cs)[:nc.value]})
        return out

    def describe(self) -> dict:
        import json
        L = lib()
        n = L.dm_plan_describe(self._h, None, 0)
        buf = ctypes.create_string_buffer(int(n))
        L.dm_plan_describe(self._h, buf, n)
        return json.loads(buf.value.decode())


# ------------------------------------------------------------------------------ results
class Result:
    __slots__ = ("count", "rows", "stats")

    def __init__(self, count, rows, stats):
        self.count, self.rows, self.stats = count, rows, stats


def _stats_dict(s: _Stats) -> dict:
    n = s.num_steps
    return {
        "num_steps": n, "num_launches": s.num_launches, "num_chunks": s.num_chunks,
        "elem_bytes": s.elem_bytes,
        "rows_in": list(s.rows_in)[:n], "rows_out": list(s.rows_out)[:n],
        "candidates": list(s.candidates)[:n], "probes": list(s.probes)[:n],
        "width_in": list(s.width_in)[:n], "width_out": list(s.width_out)[:n],
        "bytes_model": list(s.bytes_model)[:n], "bytes_stored": list(s.bytes_stored)[:n],
        "ms_count": list(s.ms_count)[:n],
        "ms_write": list(s.ms_write)[:n], "ms_other": s.ms_other, "ms_total": s.ms_total,
        "pipelined": bool(s.pipelined),
    }


class _CudaArray:
    """Minimal __cuda_array_interface__ view of library-owned device memory (for torch.as_tensor)."""

    def __init__(self, ptr, shape, typestr, owner):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(ptr or 0), False), "version": 3,
                                         "strides": None}
        self._owner = owner


class Frontier:
    """A materialized level (dm_match_prefix): device rows [rows][stride] int32 in plan column
    order plus a per-row uint64 work estimate.  Owns the device buffers."""

    def __init__(self, h):
        L = lib()
        self._h = h
        self.rows = int(L.dm_frontier_rows(h))
        self.width = int(L.dm_frontier_width(h))
        self.stride = int(L.dm_frontier_stride(h))
        self.work_total = int(L.dm_frontier_work_total(h))

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.dm_frontier_free(self._h)
            self._h = None

    def rows_tensor(self, device=None):
        """torch view of the device rows (valid while this Frontier lives)."""
        import torch
        p = lib().dm_frontier_device_rows(self._h)
        return torch.as_tensor(_CudaArray(p, (self.rows, self.stride), "<i4", self), device=device)

    def work_tensor(self, device=None):
        """torch view of the per-row work estimates (None for the final level)."""
        import torch
        p = lib().dm_frontier_device_work(self._h)
        if not p:
            return None
        return torch.as_tensor(_CudaArray(p, (self.rows,), "<i8", self), device=device)


# ------------------------------------------------------------------------------- graphs
class Graph:
    """Device-resident data graph (dm_graph_create): Res(M2) as a sorted CSR on `device`."""

    def __init__(self, n: int, edges, *, drop_self_loops: bool = False, device: int = 0):
        L = lib()
        e = _edges_arr(edges)
        h = ctypes.c_void_p()
        _check(L.dm_graph_create(int(n), e.ctypes.data if e.size else None, e.shape[0],
                                 DM_GRAPH_DROP_SELF_LOOPS if drop_self_loops else 0, int(device),
                                 ctypes.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.dm_graph_destroy(self._h)
        self._h = None

    def __del__(self):
        self.close()

    @property
    def n(self) -> int:
        return lib().dm_graph_num_vertices(self._h)

    @property
    def num_arcs(self) -> int:
        return lib().dm_graph_num_arcs(self._h)

    @property
    def max_degree(self) -> int:
        return lib().dm_graph_max_degree(self._h)

    @property
    def device(self) -> int:
        return lib().dm_graph_device(self._h)

    def build_motifs(self, motifs, *, stream=None, row_budget: int = 0) -> dict:
        """dm_graph_build_motifs: the motif database (Alg. 2) for the table motifs of `motifs`;
        returns {name: (rows, build_ms)}."""
        bits = _motifs(motifs)
        o = self._opts("mono", "count", bits, None, stream, False, 0, row_budget)
        _check(lib().dm_graph_build_motifs(self._h, bits, ctypes.byref(o)))
        out = {MOTIF_NAMES[b]: (self.motif_rows(b), lib().dm_graph_motif_build_ms(self._h, b))
               for b in MOTIF_NAMES if 8 <= b < DM_MOTIF_APEX and bits & b}
        if bits & DM_MOTIF_APEX:
            out["apex"] = (int(lib().dm_graph_apex_entries(self._h)), lib().dm_graph_apex_build_ms(self._h))
        return out

    def apex_table(self):
        """(toff [num_arcs + 1] int64, apex [entries] int32 arc indices) of the built triangle-apex
        table (dm_graph_apex_table, host copies)."""
        ne = int(lib().dm_graph_apex_entries(self._h))
        if ne < 0:
            raise DMError(-1, "triangle-apex table not built")
        toff = np.empty(self.num_arcs + 1, dtype=np.int64)
        apex = np.empty(max(ne, 1), dtype=np.int32)
        _check(lib().dm_graph_apex_table(self._h, toff.ctypes.data, apex.ctypes.data))
        return toff, apex[:ne]

    def save_motifs(self, path: str):
        """dm_graph_save_motifs: persist the built motif tables (fingerprinted)."""
        _check(lib().dm_graph_save_motifs(self._h, os.fsencode(path)))

    def load_motifs(self, path: str):
        """dm_graph_load_motifs: add the tables of a saved database (fingerprint-checked)."""
        _check(lib().dm_graph_load_motifs(self._h, os.fsencode(path)))

    def motif_rows(self, motif) -> int:
        b = MOTIF_BITS[motif] if isinstance(motif, str) else int(motif)
        return int(lib().dm_graph_motif_rows(self._h, b))

    def motif_table(self, motif):
        """(rows [R][L] int32 canonical, toff [num_arcs + 1] int64) of a built table (host copies)."""
        b = MOTIF_BITS[motif] if isinstance(motif, str) else int(motif)
        R = self.motif_rows(b)
        if R < 0:
            raise DMError(-1, "motif table not built")
        Lv = {8: 4, 16: 5, 32: 6, 64: 7, 128: 8, 256: 4, 512: 6, 1024: 12}[b]
        rows = np.zeros((R, Lv), dtype=np.int32)
        toff = np.zeros(self.num_arcs + 1, dtype=np.int64)
        _check(lib().dm_graph_motif_table(self._h, b, rows.ctypes.data if R else None, toff.ctypes.data))
        return rows, toff

    def plan(self, k: int, p_edges, **kw) -> Plan:
        """dm_plan_create_for: the join program dm_match runs for this pattern."""
        return Plan.for_graph(self, k, p_edges, **kw)

    def stats(self, count_only: bool = True) -> dict:
        """Cost-model statistics (for Plan(..., stats=g.stats()) == the plan dm_match uses)."""
        a, b = ctypes.c_double(), ctypes.c_double()
        _check(lib().dm_graph_stats(self._h, ctypes.byref(a), ctypes.byref(b)))
        return dict(n=max(self.n, 2), arcs=self.num_arcs, sum_d2=a.value, closure=b.value,
                    max_degree=self.max_degree, count_only=count_only)

    def csr(self):
        """(off int64[n+1], adj int32[arcs]) copied to the host."""
        off = np.zeros(self.n + 1, dtype=np.int64)
        adj = np.zeros(max(self.num_arcs, 1), dtype=np.int32)
        _check(lib().dm_graph_copy_csr(self._h, off.ctypes.data, adj.ctypes.data))
        return off, adj[: self.num_arcs]

    def _opts(self, mode, output, motifs, seed_range, stream, profile, mem_budget, row_budget):
        L = lib()
        o = _Opts()
        L.dm_match_opts_init(ctypes.byref(o))
        o.mode = DM_INDUCED if mode == "induced" else DM_MONO
        o.output = {"count": DM_OUT_COUNT, "table": DM_OUT_TABLE, "both": DM_OUT_COUNT | DM_OUT_TABLE}[output]
        o.motifs = _motifs(motifs)
        o.flags = DM_MATCH_PROFILE if profile else 0
        o.mem_budget = int(mem_budget)
        o.row_budget = int(row_budget)
        if seed_range is not None:
            o.seed_begin, o.seed_end = int(seed_range[0]), int(seed_range[1])
        if stream is not None:
            o.cuda_stream = int(getattr(stream, "cuda_stream", stream))
        return o

    def match_prefix(self, k: int, p_edges, upto_step: int, *, mode: str = "mono",
                     output: str = "count", motifs="all", seed_range=None, stream=None) -> Frontier:
        """dm_match_prefix: run join steps [0, upto_step) and return level upto_step."""
        pe = _edges_arr(p_edges)
        o = self._opts(mode, output, motifs, seed_range, stream, False, 0, 0)
        h = ctypes.c_void_p()
        _check(lib().dm_match_prefix(self._h, int(k), pe.ctypes.data if pe.size else None,
                                     pe.shape[0], ctypes.byref(o), int(upto_step), ctypes.byref(h)))
        return Frontier(h)

    def match_resume(self, k: int, p_edges, from_step: int, rows, *, mode: str = "mono",
                     output: str = "count", motifs="all", stream=None, profile: bool = False) -> Result:
        """dm_match_resume: finish the plan from a level given as a CUDA int32 tensor
        [rows][stride] (plan column order)."""
        pe = _edges_arr(p_edges)
        o = self._opts(mode, output, motifs, None, stream, profile, 0, 0)
        if rows is not None:
            plan = Plan.for_graph(self, k, pe, mode=mode, output=output, motifs=motifs)
            if not 1 <= int(from_step) < plan.num_steps:
                raise DMError(-1, "from_step must be in [1, num_steps)")
            _check_rows(rows, self, plan.stride(from_step))
        n = int(rows.shape[0]) if rows is not None else 0
        ptr = rows.data_ptr() if n else None
        r = ctypes.c_void_p()
        _check(lib().dm_match_resume(self._h, int(k), pe.ctypes.data if pe.size else None,
                                     pe.shape[0], ctypes.byref(o), int(from_step), ptr, n,
                                     ctypes.byref(r)))
        return self._result(r, k, output)

    def _result(self, r, k, output) -> Result:
        L = lib()
        try:
            cnt = int(L.dm_result_count(r))
            rows = None
            p = L.dm_result_rows(r)
            if p and output in ("table", "both"):
                buf = (ctypes.c_int32 * (cnt * k)).from_address(p)
                rows = np.frombuffer(buf, dtype=np.int32).reshape(cnt, k).copy()
            elif output in ("table", "both"):
                rows = np.zeros((0, k), dtype=np.int32)
            st = _Stats()
            _check(L.dm_result_stats(r, ctypes.byref(st)))
            return Result(cnt, rows, _stats_dict(st))
        finally:
            L.dm_result_free(r)

    def score_layouts(self, k: int, p_edges, node_fid, fid_edges, fid_vals, top_k: int, *,
                      mode: str = "mono", motifs="all", stream=None):
        """dm_score_layouts: the top_k layouts (embeddings) by fidelity score (§6.5).
        Returns (rows [m][k] int32, scores [m] float64, total number of layouts)."""
        pe = _edges_arr(p_edges)
        nf = np.ascontiguousarray(np.asarray(node_fid, dtype=np.float64))
        fe = _edges_arr(fid_edges)
        fv = np.ascontiguousarray(np.asarray(fid_vals, dtype=np.float64).reshape(-1))
        if nf.shape != (self.n,) or fv.shape[0] != fe.shape[0]:
            raise ValueError("node_fid must have n entries and fid_vals one per fidelity edge")
        o = self._opts(mode, "table", motifs, None, stream, False, 0, 0)
        m = max(int(top_k), 1)
        rows = np.zeros((m, k), dtype=np.int32)
        scores = np.zeros(m, dtype=np.float64)
        n_out, cnt = ctypes.c_int64(0), ctypes.c_uint64(0)
        _check(lib().dm_score_layouts(self._h, int(k), pe.ctypes.data if pe.size else None, pe.shape[0],
                                      nf.ctypes.data, fe.ctypes.data if fe.size else None,
                                      fv.ctypes.data if fv.size else None, fe.shape[0], ctypes.byref(o),
                                      int(top_k), rows.ctypes.data, scores.ctypes.data, ctypes.byref(n_out),
                                      ctypes.byref(cnt)))
        return rows[: n_out.value], scores[: n_out.value], int(cnt.value)

    def match(self, k: int, p_edges, *, mode: str = "mono", output: str = "count",
              motifs="all", seed_range=None, stream=None, profile: bool = False,
              mem_budget: int = 0, row_budget: int = 0) -> Result:
        """dm_match: embeddings of the pattern (k, p_edges).  output in {"count", "table",
        "both"}; seed_range=(b, e) restricts f(first plan vertex) to [b, e); stream is a
        torch.cuda.Stream / raw cudaStream_t int (None = legacy default stream)."""
        pe = _edges_arr(p_edges)
        o = self._opts(mode, output, motifs, seed_range, stream, profile, mem_budget, row_budget)
        r = ctypes.c_void_p()
        _check(lib().dm_match(self._h, int(k), pe.ctypes.data if pe.size else None, pe.shape[0],
                              ctypes.byref(o), ctypes.byref(r)))
        return self._result(r, k, output)
