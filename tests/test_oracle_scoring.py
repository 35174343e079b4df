"""Pins of the CPU layout-scoring reference (oracle/scoring.py; §6.5, SPEC
layout-scoring S:472-508) against things other than itself: closed forms (uniform fidelities),
the SPEC worked example, a brute-force enumeration of all injective maps scored by a
dictionary-based restatement, and monotonicity."""
import itertools

import numpy as np

import dm_inputs as g
import oracle
from oracle.scoring import layout_scores, top_layouts


def _rand_fid(n, e, seed):
    rng = np.random.default_rng(seed)
    return rng.uniform(0.9, 1.0, n), e.copy(), rng.uniform(0.8, 1.0, len(e))


def test_uniform_fidelity_closed_form():
    """uniform fidelity f on nodes and edges -> every score is f^(k + m)."""
    n, e = g.falcon27()
    for (k, pe) in (g.path(4), g.path(7), g.ring(12)):
        rows = oracle.match(n, e, k, pe).rows
        s = layout_scores(rows, n, pe, np.full(n, 0.97), e, np.full(len(e), 0.97))
        assert np.allclose(s, 0.97 ** (k + len(pe)), rtol=1e-14, atol=0)
        s1 = layout_scores(rows, n, pe, np.ones(n), e, np.ones(len(e)))
        assert np.all(s1 == 1.0)


def test_spec_m2_example():
    """M2 row (u, v) with node fidelities 0.99 / 0.98 and edge 0.95 -> 0.99*0.98*0.95."""
    node = np.array([0.99, 0.98])
    s = layout_scores(np.array([[0, 1]]), 2, [(0, 1)], node, [(0, 1)], [0.95])
    assert s[0] == 0.99 * 0.98 * 0.95


def test_brute_force_top_layouts():
    """Top layouts = argmax of an exhaustive scoring of every injective map."""
    n, e = g.falcon27()
    node, fe, fv = _rand_fid(n, e, 4)
    ef = {}
    for (a, b), f in zip(fe.tolist(), fv.tolist()):
        ef[(a, b)] = ef[(b, a)] = f
    k, pe = g.path(4)
    brute = []
    for f in itertools.permutations(range(n), k):
        if all((f[a], f[b]) in ef for a, b in pe.tolist()):
            sc = 1.0
            for v in range(k):
                sc *= node[f[v]]
            for a, b in pe.tolist():
                sc *= ef[(f[a], f[b])]
            brute.append((-sc, f))
    brute.sort()
    rows = oracle.match(n, e, k, pe).rows
    s = layout_scores(rows, n, pe, node, fe, fv)
    top, ts = top_layouts(rows, s, 5)
    assert len(brute) == len(rows) == 80
    assert [tuple(r) for r in top.tolist()] == [f for _, f in brute[:5]]
    assert np.array_equal(ts, np.array([-x for x, _ in brute[:5]]))


def test_monotonicity():
    """lowering one edge fidelity lowers exactly the scores of the layouts using it."""
    n, e = g.ibm_heavy_hex(3)
    node, fe, fv = _rand_fid(n, e, 9)
    k, pe = g.path(6)
    rows = oracle.match(n, e, k, pe).rows
    s0 = layout_scores(rows, n, pe, node, fe, fv)
    fv2 = fv.copy()
    fv2[10] *= 0.5
    s1 = layout_scores(rows, n, pe, node, fe, fv2)
    u, v = fe[10]
    uses = np.zeros(len(rows), bool)
    for a, b in pe.tolist():
        uses |= ((rows[:, a] == u) & (rows[:, b] == v)) | ((rows[:, a] == v) & (rows[:, b] == u))
    assert np.all(s1[uses] < s0[uses]) and np.all(s1[~uses] == s0[~uses]) and uses.any()
