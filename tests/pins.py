"""Independent pins for the oracle (test infrastructure).

Nothing here calls the oracle or the CUDA path: these are closed forms, independent
counting algorithms and brute force, each derived from the mathematics of the definition in
PAPER.md §3.1 l.167 (labelled embeddings = injective edge-preserving maps) -- SURVEY.md
§8(c) "What pins each part".
"""
from __future__ import annotations

import itertools

import numpy as np
import scipy.sparse as sp


def simple_adj(n, edges):
    """Symmetric 0/1 CSR adjacency without self-loops or duplicates."""
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    e = e[e[:, 0] != e[:, 1]]
    r = np.concatenate([e[:, 0], e[:, 1]])
    c = np.concatenate([e[:, 1], e[:, 0]])
    A = sp.csr_matrix((np.ones(r.size, dtype=np.int64), (r, c)), shape=(n, n))
    A.data[:] = 1
    A.sum_duplicates()
    A.data[:] = 1
    return A


def degrees(A):
    return np.asarray(A.sum(axis=1)).ravel().astype(np.int64)


def num_edges(A):
    return int(A.nnz // 2)


# ------------------------------------------------------------------ closed forms (any graph)
def tri_labelled(A):
    """P-tri: labelled triangles = tr(A^3) (closed 3-walks are exactly labelled triangles)."""
    return int((A @ A).multiply(A).sum())


def c4_labelled(A):
    """P-C4: labelled 4-cycles (mono) = tr(A^4) - 2 sum d^2 + 2|E|; tr(A^4) = ||A^2||_F^2."""
    A2 = A @ A
    tr4 = int(A2.multiply(A2).sum())
    d = degrees(A)
    return tr4 - 2 * int((d * d).sum()) + 2 * num_edges(A)


def p3_labelled(A):
    """P-P3: labelled 3-paths = sum_v d_v (d_v - 1)."""
    d = degrees(A)
    return int((d * (d - 1)).sum())


def p4_labelled(A):
    """P-P4: labelled 4-paths (mono) = 2 sum_{uv in E} (d_u-1)(d_v-1) - tr(A^3)."""
    d = degrees(A)
    C = sp.triu(A, k=1).tocoo()
    s = int(((d[C.row] - 1) * (d[C.col] - 1)).sum())
    return 2 * s - tri_labelled(A)


def diamonds_labelled(A):
    """P-dia: labelled diamonds (K4 minus edge 0-3) = 2 sum_{e in E} t_e (t_e - 1)."""
    T = (A @ A).multiply(A)            # T[u,v] = common neighbours of adjacent u, v
    C = sp.triu(T, k=1).tocoo()
    t = C.data.astype(np.int64)
    return int(2 * (t * (t - 1)).sum())


def k4_count_oriented(n, edges):
    """P-K4: number of distinct 4-cliques by a degree-oriented counter (a different
    algorithm from backtracking): orient u->v iff (deg u, u) < (deg v, v); every K4 has a
    unique source-ordered representation u->v->w->x."""
    A = simple_adj(n, edges)
    d = degrees(A)
    rank = lambda v: (int(d[v]), int(v))
    out = [set() for _ in range(n)]
    C = sp.triu(A, k=1).tocoo()
    for a, b in zip(C.row.tolist(), C.col.tolist()):
        if rank(a) < rank(b):
            out[a].add(b)
        else:
            out[b].add(a)
    total = 0
    for u in range(n):
        for v in out[u]:
            common = out[u] & out[v]
            for w in common:
                total += len(common & out[w])
    return total


def tri_count_oriented(n, edges):
    A = simple_adj(n, edges)
    d = degrees(A)
    out = [set() for _ in range(n)]
    C = sp.triu(A, k=1).tocoo()
    for a, b in zip(C.row.tolist(), C.col.tolist()):
        if (d[a], a) < (d[b], b):
            out[a].add(b)
        else:
            out[b].add(a)
    return sum(len(out[u] & out[v]) for u in range(n) for v in out[u])


def paths_nonbacktracking(n, edges, k):
    """P-NB: labelled P_k = 1^T B^(k-2) 1 with B the non-backtracking (Hashimoto) arc matrix;
    exact when k <= girth (a non-backtracking walk with k-1 arcs revisits a vertex only by
    closing a cycle of length <= k-1)."""
    A = simple_adj(n, edges).tocoo()
    src, dst = A.row.astype(np.int64), A.col.astype(np.int64)
    if k == 1:
        return n
    order = np.lexsort((dst, src))
    src, dst = src[order], dst[order]
    na = src.size
    off = np.zeros(n + 1, dtype=np.int64)
    np.add.at(off, src + 1, 1)
    off = np.cumsum(off)
    x = np.ones(na, dtype=object)   # exact big integers
    for _ in range(k - 2):
        # y[a] = sum over arcs b = (dst[a] -> w), w != src[a] of x[b]
        y = np.zeros(na, dtype=object)
        for a in range(na):
            v = dst[a]
            s = 0
            for b in range(off[v], off[v + 1]):
                if dst[b] != src[a]:
                    s += x[b]
            y[a] = s
        x = y
    return int(sum(x))


def tree_locally_injective(n, edges, k, t_edges):
    """P-tree: labelled embeddings of a tree pattern T = locally injective homomorphisms
    (each vertex's tree-neighbours map to distinct data neighbours), valid when
    diam(T) < girth(G).  Rooted DP over arcs (parent image -> own image)."""
    A = simple_adj(n, edges)
    nb = [A.indices[A.indptr[v]:A.indptr[v + 1]].tolist() for v in range(n)]
    tadj = [[] for _ in range(k)]
    for a, b in np.asarray(t_edges).reshape(-1, 2).tolist():
        tadj[a].append(b)
        tadj[b].append(a)
    root = 0
    parent = [-1] * k
    order = [root]
    for v in order:
        for u in tadj[v]:
            if u != parent[v] and u != root and parent[u] == -1:
                parent[u] = v
                order.append(u)
    children = [[u for u in tadj[v] if parent[u] == v] for v in range(k)]
    memo = {}

    def W(v, x, y):
        key = (v, x, y)
        if key in memo:
            return memo[key]
        ch = children[v]
        avail = [z for z in nb[x] if z != y]
        tot = 0
        for tup in itertools.permutations(avail, len(ch)):
            p = 1
            for c, z in zip(ch, tup):
                p *= W(c, z, x)
                if p == 0:
                    break
            tot += p
        memo[key] = tot
        return tot

    return sum(W(root, x, -1) for x in range(n))


# --------------------------------------------------------------------------- brute force
def brute_force(n, edges, k, p_edges, induced=False):
    """P-brute: all n!/(n-k)! injective maps, checked against the definition.
    Returns the sorted list of rows (tuples)."""
    A = simple_adj(n, edges).toarray().astype(bool)
    P = np.zeros((k, k), dtype=bool)
    for a, b in np.asarray(p_edges).reshape(-1, 2).tolist():
        P[a, b] = P[b, a] = True
    pe = [(a, b) for a in range(k) for b in range(a + 1, k) if P[a, b]]
    pn = [(a, b) for a in range(k) for b in range(a + 1, k) if not P[a, b]]
    out = []
    for f in itertools.permutations(range(n), k):
        if all(A[f[a], f[b]] for a, b in pe) and (not induced or not any(A[f[a], f[b]] for a, b in pn)):
            out.append(f)
    return out


def rows_to_tuples(rows):
    return [tuple(int(x) for x in r) for r in np.asarray(rows).tolist()]


# ------------------------------------------------------------------ native full-scale pins
def _pins_native():
    """ctypes handle of tests/pins_native.c (built with gcc on first use; test infra only)."""
    import ctypes
    import os
    import subprocess
    here = os.path.dirname(os.path.abspath(__file__))
    src = os.path.join(here, "pins_native.c")
    lib = os.path.join(here, "libpins_native.so")
    if not os.path.exists(lib) or os.path.getmtime(lib) < os.path.getmtime(src):
        tmp = lib + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-pthread", src, "-o", tmp])
        os.replace(tmp, lib)
    L = ctypes.CDLL(lib)
    for f in ("pins_triangles_labelled", "pins_diamonds_labelled", "pins_k4_distinct"):
        fn = getattr(L, f)
        fn.restype = ctypes.c_uint64
        fn.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int]
    return L


def native_counts(n, edges, which, threads=None):
    """Exact labelled triangles / labelled diamonds / distinct K4 by sorted-list merges."""
    import os
    e = np.ascontiguousarray(np.asarray(edges, dtype=np.int32).reshape(-1, 2))
    L = _pins_native()
    fn = {"tri": L.pins_triangles_labelled, "diamond": L.pins_diamonds_labelled,
          "k4": L.pins_k4_distinct}[which]
    return int(fn(n, e.ctypes.data, e.shape[0], threads or os.cpu_count() or 1))
