"""TEST INFRASTRUCTURE ONLY -- plain CPU reference of layout scoring (quantum layout selection,
PAPER.md §6.5; SPEC layout-scoring module).

Only tests/, __graft_entry__.smoke() and bench.py may import this module; the product path
(paper_2508_21287_b200) never imports it.

The score of a layout (an embedding f, one row of the canonical table, column j = f(j)) is the
product of the node fidelities of its k distinct data vertices times the product of the edge
fidelities of its pattern edges' images ("score = prod node_f over its n distinct vertices x
prod edge_f over its m pattern-edge images"), multiplied in float64 in this order: pattern
vertices 0..k-1, then the pattern edges in the order given.  Ranking: descending score, ties by
ascending lexicographic row order.
"""
from __future__ import annotations

import numpy as np


def edge_fidelity_lookup(n: int, fid_edges, fid_vals):
    """(sorted keys u*n+v for both orientations, values) of an undirected edge-fidelity map."""
    fe = np.asarray(fid_edges, np.int64).reshape(-1, 2)
    fv = np.asarray(fid_vals, np.float64).reshape(-1)
    keys = np.concatenate([fe[:, 0] * n + fe[:, 1], fe[:, 1] * n + fe[:, 0]])
    vals = np.concatenate([fv, fv])
    order = np.argsort(keys, kind="stable")
    return keys[order], vals[order]


def layout_scores(rows, n: int, p_edges, node_fid, fid_edges, fid_vals) -> np.ndarray:
    """Score of every row of an embedding table rows[count][k] (definition above)."""
    rows = np.asarray(rows, np.int64)
    cnt, k = rows.shape
    node = np.asarray(node_fid, np.float64)
    keys, vals = edge_fidelity_lookup(n, fid_edges, fid_vals)
    s = np.ones(cnt, np.float64)
    for v in range(k):
        s = s * node[rows[:, v]]
    for a, b in np.asarray(p_edges, np.int64).reshape(-1, 2):
        q = rows[:, a] * n + rows[:, b]
        pos = np.searchsorted(keys, q)
        assert np.all(keys[np.minimum(pos, len(keys) - 1)] == q), "an image edge has no fidelity"
        s = s * vals[pos]
    return s


def top_layouts(rows, scores, top_k: int):
    """The top_k rows by descending score, ties by ascending lexicographic row order."""
    rows = np.asarray(rows)
    cnt, k = rows.shape if rows.ndim == 2 else (0, 0)
    if cnt == 0:
        return rows.reshape(0, max(k, 0)), np.zeros(0)
    order = np.lexsort(tuple(rows[:, j] for j in range(k - 1, -1, -1)) + (-np.asarray(scores),))
    order = order[:top_k]
    return rows[order], np.asarray(scores)[order]
