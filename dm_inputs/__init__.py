"""Seeded synthetic input generators shared by the CUDA path's tests/bench and the oracle's tests.

This module is the ONLY code the oracle side (``oracle/``) and the product side
(``paper_2508_21287_b200``) have in common, and it holds none of the method's
arithmetic: it only produces raw edge lists (``int32[m][2]`` numpy arrays, possibly with
duplicates / reversed pairs / self-loops, exactly as a user would hand them over) and
pattern graphs.  Each side builds its own adjacency structure from these lists.

Recipes:

* ``falcon27``            IBM Falcon r4 27-qubit coupling map (public; not in the paper).
* ``ibm_heavy_hex(w)``    IBM family: V = 10w^2+12w+1, E = 12w^2+12w (w=3 -> Eagle 127).
* ``hex_lattice_subdivided(m, n)`` networkx-style hexagonal lattice with every edge
                           subdivided: V = 5mn+4m+4n-1 ((11,33) -> 1990, (25,34) -> 4485, the
                           paper's heavy-hex sizes, §6.2 l.439).
* ``square_grid(r, c)``   2-D grid, id = c*i + j (§6.2 l.439 "2D square grid").
* ``grid_diag(k)``        k x k grid plus one diagonal (i,j)-(i+1,j+1) per cell.
* ``er_gnm(n, m, seed)``  Erdos-Renyi G(n, m), m distinct pairs uniformly without replacement.
* ``rmat(scale, ef, seed)`` Graph500 R-MAT (a,b,c,d)=(0.57,0.19,0.19,0.05), ef*2^scale samples,
                           seeded random vertex permutation; raw (self-loops/duplicates kept).
* patterns: ``path``, ``ring``, ``clique``, ``diamond``, ``star``, ``random_tree``,
  ``random_connected_subgraph`` (seeded random-walk accumulation + induced closure),
  ``device_subtree`` (spanning tree of a random connected device subgraph).
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "falcon27", "ibm_heavy_hex", "hex_lattice_subdivided", "square_grid", "grid", "grid_diag",
    "er_gnm", "rmat", "path", "ring", "clique", "diamond", "star", "random_tree",
    "random_connected_subgraph", "device_subtree", "relabel", "CONFIGS",
]


def _arr(edges) -> np.ndarray:
    a = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    return np.ascontiguousarray(a.astype(np.int32))


# --------------------------------------------------------------------------- data graphs
_FALCON27 = [(0, 1), (1, 2), (1, 4), (2, 3), (3, 5), (4, 7), (5, 8), (6, 7), (7, 10), (8, 9),
             (8, 11), (10, 12), (11, 14), (12, 13), (12, 15), (13, 14), (14, 16), (15, 18),
             (16, 19), (17, 18), (18, 21), (19, 20), (19, 22), (21, 23), (22, 25), (23, 24),
             (24, 25), (25, 26)]


def falcon27():
    """IBM Falcon r4 27-qubit heavy-hex coupling map."""
    return 27, _arr(_FALCON27)


def ibm_heavy_hex(w: int):
    """IBM heavy-hex family of width w.

    R = 2w+1 rows, L = 4w+3 columns; row 0 uses columns [0, L-1), row R-1 uses [1, L), the
    others [0, L).  Between rows r and r+1 sit w+1 bridge vertices at columns c = 0 (mod 4)
    (r even) or c = 2 (mod 4) (r odd).  Row-major numbering, each row's bridges after it.
    """
    if w < 1:
        raise ValueError("w >= 1")
    R, L = 2 * w + 1, 4 * w + 3
    ids = {}
    nxt = 0
    edges = []
    bridge_cols = []
    for r in range(R):
        lo, hi = (0, L - 1) if r == 0 else ((1, L) if r == R - 1 else (0, L))
        prev = None
        for c in range(lo, hi):
            ids[(r, c)] = nxt
            if prev is not None:
                edges.append((prev, nxt))
            prev = nxt
            nxt += 1
        if r + 1 < R:
            cols = [c for c in range(L) if c % 4 == (0 if r % 2 == 0 else 2)]
            bridge_cols.append(cols)
            for c in cols:
                ids[("b", r, c)] = nxt
                nxt += 1
    for r in range(R - 1):
        for c in bridge_cols[r]:
            b = ids[("b", r, c)]
            edges.append((ids[(r, c)], b))
            edges.append((b, ids[(r + 1, c)]))
    return nxt, _arr(edges)


def hex_lattice_subdivided(m: int, n: int):
    """Hexagonal lattice of m x n hexagons (networkx ``hexagonal_lattice_graph`` layout) with
    every edge subdivided by a new degree-2 vertex."""
    rows = range(2 * m + 2)
    cols = range(n + 1)
    und = []
    for i in cols:
        for j in rows[: 2 * m + 1]:
            und.append(((i, j), (i, j + 1)))
    for i in cols[:n]:
        for j in rows:
            if i % 2 == j % 2:
                und.append(((i, j), (i + 1, j)))
    dead = {(0, 2 * m + 1), (n, (2 * m + 1) * (n % 2))}
    und = [e for e in und if e[0] not in dead and e[1] not in dead]
    nodes = sorted({x for e in und for x in e})
    idx = {v: t for t, v in enumerate(nodes)}
    nv = len(nodes)
    edges = []
    for (a, b) in und:
        mid = nv
        nv += 1
        edges.append((idx[a], mid))
        edges.append((mid, idx[b]))
    return nv, _arr(edges)


def square_grid(r: int, c: int):
    """r x c grid; id = c*i + j; edges (i,j)-(i,j+1), (i,j)-(i+1,j)."""
    e = []
    for i in range(r):
        for j in range(c):
            v = c * i + j
            if j + 1 < c:
                e.append((v, v + 1))
            if i + 1 < r:
                e.append((v, v + c))
    return r * c, _arr(e)


def grid(k: int):
    return square_grid(k, k)


def grid_diag(k: int):
    """k x k grid plus one diagonal (i,j)-(i+1,j+1) per cell."""
    n, e = square_grid(k, k)
    d = [(k * i + j, k * (i + 1) + j + 1) for i in range(k - 1) for j in range(k - 1)]
    return n, _arr(np.concatenate([e, _arr(d)]) if d else e)


def er_gnm(n: int, m: int, seed: int):
    """G(n, m): m distinct unordered pairs drawn uniformly without replacement."""
    total = n * (n - 1) // 2
    if m > total:
        raise ValueError("m too large")
    rng = np.random.default_rng(seed)
    chosen = np.empty(0, dtype=np.int64)
    while chosen.size < m:
        need = m - chosen.size
        draw = rng.integers(0, total, size=int(need * 1.1) + 16, dtype=np.int64)
        # keep first occurrences in draw order (deterministic), drop already chosen
        cat = np.concatenate([chosen, draw])
        _, first = np.unique(cat, return_index=True)
        first.sort()
        chosen = cat[first][:m]
    # unrank pair index t -> (i, j), i < j, row-major over i
    t = chosen
    # i = largest i with i*(2n-i-1)/2 <= t
    i = np.floor(((2 * n - 1) - np.sqrt((2 * n - 1) ** 2 - 8.0 * t)) / 2).astype(np.int64)
    base = i * (2 * n - i - 1) // 2
    over = base > t
    while over.any():
        i[over] -= 1
        base = i * (2 * n - i - 1) // 2
        over = base > t
    nxt = (i + 1) * (2 * n - i - 2) // 2
    under = nxt <= t
    while under.any():
        i[under] += 1
        base = i * (2 * n - i - 1) // 2
        nxt = (i + 1) * (2 * n - i - 2) // 2
        under = nxt <= t
    j = t - base + i + 1
    return n, _arr(np.stack([i, j], axis=1))


def rmat(scale: int, edge_factor: int = 16, seed: int = 1, a=0.57, b=0.19, c=0.19,
         permute: bool = True):
    """Graph500-style R-MAT: per bit r~U[0,1); row bit = r >= a+b;
    col bit = (a <= r < a+b) or (r >= a+b+c).  Raw samples (self-loops and duplicates kept);
    optional seeded vertex permutation."""
    n = 1 << scale
    M = edge_factor * n
    rng = np.random.default_rng(seed)
    u = np.zeros(M, dtype=np.int64)
    v = np.zeros(M, dtype=np.int64)
    ab, abc = a + b, a + b + c
    for bit in range(scale):
        r = rng.random(M)
        ub = r >= ab
        vb = ((r >= a) & (r < ab)) | (r >= abc)
        u |= ub.astype(np.int64) << bit
        v |= vb.astype(np.int64) << bit
    if permute:
        perm = rng.permutation(n)
        u = perm[u]
        v = perm[v]
    return n, _arr(np.stack([u, v], axis=1))


def relabel(n: int, edges: np.ndarray, seed: int):
    """Apply a seeded random vertex permutation sigma; returns (edges', sigma)."""
    sigma = np.random.default_rng(seed).permutation(n).astype(np.int32)
    return _arr(sigma[edges]), sigma


# ----------------------------------------------------------------------------- patterns
def path(k: int):
    return k, _arr([(i, i + 1) for i in range(k - 1)])


def ring(k: int):
    return k, _arr([(i, (i + 1) % k) for i in range(k)])


def clique(k: int):
    return k, _arr([(i, j) for i in range(k) for j in range(i + 1, k)])


def diamond():
    """K4 minus an edge: 0-1, 0-2, 1-2, 1-3, 2-3."""
    return 4, _arr([(0, 1), (0, 2), (1, 2), (1, 3), (2, 3)])


def star(k: int):
    return k, _arr([(0, i) for i in range(1, k)])


def random_tree(k: int, seed: int, max_degree: int | None = None):
    """Random labelled tree: vertex i>0 attaches to a uniformly random earlier vertex whose
    degree is below max_degree."""
    rng = np.random.default_rng(seed)
    deg = [0] * k
    e = []
    for i in range(1, k):
        while True:
            p = int(rng.integers(0, i))
            if max_degree is None or deg[p] < max_degree:
                break
        deg[p] += 1
        deg[i] += 1
        e.append((p, i))
    return k, _arr(e)


def _adjacency_sets(n, edges):
    adj = [set() for _ in range(n)]
    for a, b in np.asarray(edges).tolist():
        if a != b:
            adj[a].add(b)
            adj[b].add(a)
    return adj


def random_connected_subgraph(n: int, edges, size: int, seed: int, induced: bool = True,
                              start: int | None = None):
    """Seeded random-walk vertex accumulation + induced-edge closure.

    Returns (size, pattern_edges, witness) where witness[i] is the data vertex that pattern
    vertex i was sampled from (so witness is itself one embedding of the pattern)."""
    adj = _adjacency_sets(n, edges)
    rng = np.random.default_rng(seed)
    if size > n:
        raise ValueError("size exceeds graph")
    if start is None:
        cand = [v for v in range(n) if adj[v]] if size > 1 else list(range(n))
        start = int(cand[int(rng.integers(0, len(cand)))])
    chosen = [start]
    inset = {start}
    cur = start
    steps = 0
    while len(chosen) < size:
        nb = sorted(adj[cur])
        if not nb:
            raise ValueError("cannot reach size from start (disconnected)")
        cur = nb[int(rng.integers(0, len(nb)))]
        if cur not in inset:
            inset.add(cur)
            chosen.append(cur)
        steps += 1
        if steps > 1000 * size * max(1, size):
            raise ValueError("random walk failed to reach size")
    pos = {v: i for i, v in enumerate(chosen)}
    pe = []
    if induced:
        for v in chosen:
            for u in adj[v]:
                if u in pos and pos[v] < pos[u]:
                    pe.append((pos[v], pos[u]))
    else:
        raise NotImplementedError
    pe.sort()
    return size, _arr(pe) if pe else np.zeros((0, 2), np.int32), np.asarray(chosen, np.int32)


def device_subtree(n: int, edges, size: int, seed: int):
    """Random spanning tree (BFS from the first sampled vertex) of a random connected
    subgraph of a device graph: a 'circuit interaction graph' that is a tree."""
    k, pe, wit = random_connected_subgraph(n, edges, size, seed)
    adj = _adjacency_sets(k, pe)
    seen = {0}
    order = [0]
    te = []
    for v in order:
        for u in sorted(adj[v]):
            if u not in seen:
                seen.add(u)
                order.append(u)
                te.append((v, u))
    return k, _arr(te)


# ---------------------------------------------------------------------- BASELINE configs
CONFIGS = {
    1: "4-vertex path pattern into IBM 27-qubit heavy-hex coupling graph (table)",
    2: "triangle and 4-cycle into 64x64 grid-with-diagonals and ER G(1e4, avg deg 16) (table)",
    3: "10-20-qubit paths, rings, trees into 127/433/1121-qubit heavy-hex (table)",
    4: "diamond and 4-clique into R-MAT scale 20, edge factor 16 (count)",
    5: "30-vertex path into a ~10k-qubit heavy-hex lattice (IBM w=31, 9983 V) (count)",
}
