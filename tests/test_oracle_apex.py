"""Pin the triangle-apex oracle (oracle/apex.py, Res(M3-O) keyed by arc)
to things other than itself: a hand-worked example, the closed forms |apex(a,b)| = (A^2)_ab and
sum |apex| = tr(A^3), and two independent counters it must reproduce when used as a join table
(labelled diamonds = sum_arcs t(t-1), pins.diamonds_labelled; labelled 4-cliques =
24 x the degree-oriented K4 counter)."""
import numpy as np
import pytest

import dm_inputs as g
from oracle.apex import apex_table, arc_list
from pins import diamonds_labelled, k4_count_oriented, simple_adj, tri_labelled


def test_apex_worked_triangle():
    """Triangle 0-1-2.  Arcs in order: (0,1) (0,2) (1,0) (1,2) (2,0) (2,1) = 0..5.
    apex(0,1) = {2} -> arc (0,2) = 1; apex(0,2) = {1} -> (0,1) = 0; apex(1,0) = {2} -> (1,2) = 3;
    apex(1,2) = {0} -> (1,0) = 2; apex(2,0) = {1} -> (2,1) = 5; apex(2,1) = {0} -> (2,0) = 4."""
    toff, apex = apex_table(3, [(0, 1), (1, 2), (2, 0), (0, 1), (2, 2)])  # duplicate + self-loop
    assert toff.tolist() == [0, 1, 2, 3, 4, 5, 6]
    assert apex.tolist() == [1, 0, 3, 2, 5, 4]


def test_apex_worked_diamond_graph():
    """Diamond 0-1, 0-2, 1-2, 1-3, 2-3 (two triangles sharing 1-2): apex(1,2) = {0, 3},
    apex(0,3) does not exist (no arc), apex(0,1) = {2}."""
    n, e = 4, [(0, 1), (0, 2), (1, 2), (1, 3), (2, 3)]
    arcs = arc_list(n, e)
    toff, apex = apex_table(n, e)
    adj = [b for _, b in arcs]
    i12 = arcs.index((1, 2))
    assert [adj[x] for x in apex[toff[i12]:toff[i12 + 1]]] == [0, 3]
    i01 = arcs.index((0, 1))
    assert [adj[x] for x in apex[toff[i01]:toff[i01 + 1]]] == [2]
    assert toff[-1] == 12  # 2 triangles x 6


@pytest.mark.parametrize("name", ["er", "rmat10", "grid_diag", "heavy_hex"])
def test_apex_closed_forms(name):
    n, e = {"er": lambda: g.er_gnm(400, 3000, 3), "rmat10": lambda: g.rmat(10, 16, seed=1),
            "grid_diag": lambda: g.grid_diag(12), "heavy_hex": lambda: g.ibm_heavy_hex(3)}[name]()
    A = simple_adj(n, e)
    arcs = arc_list(n, e)
    toff, apex = apex_table(n, e)
    assert len(toff) == len(arcs) + 1 == A.nnz + 1
    t = np.diff(toff)
    A2 = (A @ A).tocsr()
    want = np.asarray([A2[a, b] for a, b in arcs], dtype=np.int64)
    assert np.array_equal(t, want)                       # |N(a) ∩ N(b)| = (A^2)_ab
    assert int(toff[-1]) == tri_labelled(A)              # sum = tr(A^3)
    # entries: arcs of the same source, strictly ascending, apex vertex adjacent to b
    src = np.asarray([a for a, _ in arcs]); dst = np.asarray([b for _, b in arcs])
    for i in range(0, len(arcs), max(1, len(arcs) // 200)):
        seg = apex[toff[i]:toff[i + 1]]
        assert (src[seg] == src[i]).all() and (np.diff(seg) > 0).all()
        assert all(A[dst[i], c] for c in dst[seg])
    # as a join table: labelled diamonds and 4-cliques (independent counters in pins.py)
    assert int((t * (t - 1)).sum()) == diamonds_labelled(A)
    k4 = 0
    for i in range(len(arcs)):
        S = set(apex[toff[i]:toff[i + 1]].tolist())
        for x0 in S:
            k4 += len(S & set(apex[toff[x0]:toff[x0 + 1]].tolist()))
    assert k4 == 24 * k4_count_oriented(n, e)
