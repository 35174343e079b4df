"""TEST INFRASTRUCTURE ONLY -- plain CPU definition of the triangle-apex table (SURVEY §8(a) a1b:
Res(M3-O) of PAPER.md §3.4 P:262 keyed by directed edge; Alg. 2 P:264-279 builds the motif tables
once per data graph).

Only tests/, __graft_entry__.smoke() and bench.py may import this module; the product path
(paper_2508_21287_b200) never imports it.

Definition written out: the data graph's edge table Res(M2) holds both orientations of every
edge, self-loops excluded, duplicates collapsed, in ascending (a, b) order -- arc e is the
e-th pair of that order.  For arc e = (a, b) the apex list is the ascending list of every c with
(a, c) and (b, c) in Res(M2), i.e. the third column of the rows of Res(M3-O) whose first two
columns are (a, b).  Each c is reported as the index of the arc (a, c) in the same order (the
layout the GPU table uses: an "arc index payload").  Plain loops over Python sets;
no blocking, no sorting beyond the definition's order.
"""
from __future__ import annotations

import numpy as np


def arc_list(n: int, edges):
    """Res(M2): every directed pair (a, b), a != b, of the undirected edge list, both
    orientations, deduplicated, ascending."""
    arcs = set()
    for a, b in np.asarray(edges, dtype=np.int64).reshape(-1, 2).tolist():
        if a != b:
            arcs.add((a, b))
            arcs.add((b, a))
    return sorted(arcs)


def apex_table(n: int, edges):
    """(toff int64[num_arcs + 1], apex int32[entries]): apex(a, b) of arc e is
    apex[toff[e]:toff[e+1]], each entry the arc index of (a, c), c ascending."""
    arcs = arc_list(n, edges)
    index = {arc: i for i, arc in enumerate(arcs)}
    nbr = [set() for _ in range(n)]
    for a, b in arcs:
        nbr[a].add(b)
    toff = [0]
    apex = []
    for a, b in arcs:
        for c in sorted(nbr[a] & nbr[b]):
            apex.append(index[(a, c)])
        toff.append(len(apex))
    return np.asarray(toff, dtype=np.int64), np.asarray(apex, dtype=np.int32)
