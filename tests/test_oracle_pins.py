"""Pin the CPU oracle to things other than itself (SURVEY.md §8(c) "What pins each part").

Each test compares oracle output with brute force over all injective maps, a closed form, an
independent counting algorithm, a worked example printed in SPEC.md, or a metamorphic
invariant.  A plausible bug in the oracle (dropped probe, wrong anchor, missing induced
check, wrong sort) fails at least one of them.
"""
import numpy as np
import pytest

import dm_inputs as g
import oracle
from golden_util import graph_from_name, spec_examples
from pins import (brute_force, c4_labelled, diamonds_labelled, k4_count_oriented, p3_labelled,
                  p4_labelled, paths_nonbacktracking, rows_to_tuples, simple_adj,
                  tree_locally_injective, tri_count_oriented, tri_labelled)


def _random_connected_pattern(rng, k, p):
    while True:
        e = [(a, b) for a in range(k) for b in range(a + 1, k) if rng.random() < p]
        # connect: add a random spanning path if needed
        adj = {i: set() for i in range(k)}
        for a, b in e:
            adj[a].add(b); adj[b].add(a)
        seen, st = {0}, [0]
        while st:
            v = st.pop()
            for u in adj[v]:
                if u not in seen:
                    seen.add(u); st.append(u)
        if len(seen) == k:
            return k, np.asarray(e, dtype=np.int32).reshape(-1, 2)


# ------------------------------------------------------------------------- brute force
@pytest.mark.parametrize("induced", [False, True])
def test_oracle_equals_brute_force(induced):
    """P-brute: exact set equality, both modes."""
    rng = np.random.default_rng(20250821)
    cases = 0
    for trial in range(60):
        n = int(rng.integers(5, 10))
        p = float(rng.uniform(0.2, 0.7))
        e = [(a, b) for a in range(n) for b in range(a + 1, n) if rng.random() < p]
        e = np.asarray(e, dtype=np.int32).reshape(-1, 2)
        k = int(rng.integers(1, 6 if n >= 8 else 5))
        kp, pe = _random_connected_pattern(rng, k, float(rng.uniform(0.3, 0.9)))
        want = brute_force(n, e, kp, pe, induced=induced)
        got = oracle.match(n, e, kp, pe, induced=induced, threads=int(rng.integers(1, 4)))
        assert got.count == len(want)
        assert rows_to_tuples(got.rows) == want          # brute force enumerates in lex order
        cases += 1
    assert cases == 60


def test_oracle_brute_force_n12():
    rng = np.random.default_rng(7)
    n = 12
    e = np.asarray([(a, b) for a in range(n) for b in range(a + 1, n) if rng.random() < 0.35],
                   dtype=np.int32)
    for (k, pe) in [g.path(4), g.ring(4), g.star(4), g.diamond(), g.clique(3), g.ring(5)]:
        for induced in (False, True):
            want = brute_force(n, e, k, pe, induced=induced)
            got = oracle.match(n, e, k, pe, induced=induced)
            assert rows_to_tuples(got.rows) == want


# ----------------------------------------------------------------------- SPEC examples
@pytest.mark.parametrize("case", spec_examples(), ids=lambda c: c[0])
def test_oracle_spec_examples(case):
    name, data, pat, mode, exp, cite = case
    n, e = graph_from_name(data)
    k, pe = graph_from_name(pat)
    r = oracle.match(n, e, k, pe, induced=(mode == "induced"))
    assert r.count == exp, cite
    assert r.rows.shape == (exp, k)


def test_oracle_k1_and_k_gt_n():
    """Degenerate cases: k=1 -> all n vertices; k>n -> 0."""
    n, e = g.ring(5)
    r = oracle.match(n, e, 1, np.zeros((0, 2), np.int32))
    assert r.count == 5 and r.rows[:, 0].tolist() == [0, 1, 2, 3, 4]
    r = oracle.match(3, [(0, 1), (1, 2)], 4, g.path(4)[1])
    assert r.count == 0


def test_oracle_errors():
    with pytest.raises(oracle.OracleError) as ei:
        oracle.match(3, [(0, 3)], 2, [(0, 1)])
    assert ei.value.code == -2
    with pytest.raises(oracle.OracleError) as ei:
        oracle.match(3, [(0, 0), (0, 1)], 2, [(0, 1)])
    assert ei.value.code == -3
    r = oracle.match(3, [(0, 0), (0, 1)], 2, [(0, 1)], drop_self_loops=True)
    assert r.count == 2
    with pytest.raises(oracle.OracleError) as ei:
        oracle.match(4, [(0, 1)], 4, [(0, 1), (2, 3)])
    assert ei.value.code == -4
    # duplicates and reversed pairs collapse
    assert oracle.match(2, [(0, 1), (1, 0), (0, 1)], 2, [(0, 1)]).count == 2


# ------------------------------------------------------------------------ closed forms
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_oracle_closed_forms_er(seed):
    """P-tri, P-C4, P-P3, P-P4, P-dia on ER graphs."""
    n, e = g.er_gnm(300, 1500, seed)
    A = simple_adj(n, e)
    assert oracle.match(n, e, *g.clique(3), table=False).count == tri_labelled(A)
    assert oracle.match(n, e, *g.ring(4), table=False).count == c4_labelled(A)
    assert oracle.match(n, e, *g.path(3), table=False).count == p3_labelled(A)
    assert oracle.match(n, e, *g.path(4), table=False).count == p4_labelled(A)
    assert oracle.match(n, e, *g.diamond(), table=False).count == diamonds_labelled(A)


def test_oracle_closed_forms_er_config2():
    """Config 2 (ii) ER G(1e4, 8e4): triangles and C4 against tr(A^3) and the C4 form."""
    n, e = g.er_gnm(10_000, 80_000, 1)
    A = simple_adj(n, e)
    assert oracle.match(n, e, *g.clique(3), table=False).count == tri_labelled(A)
    assert oracle.match(n, e, *g.ring(4), table=False).count == c4_labelled(A)


@pytest.mark.parametrize("k", [3, 4, 5, 7])
def test_oracle_grid_closed_forms(k):
    """P-grid: C4 = 8(k-1)^2 (only unit squares), triangles 0, P3 = 12k^2-24k+8,
    induced P4 = mono P4 - 8(k-1)^2 (every non-induced P4 is a square minus one edge)."""
    n, e = g.grid(k)
    assert oracle.match(n, e, *g.ring(4), table=False).count == 8 * (k - 1) ** 2
    assert oracle.match(n, e, *g.ring(4), induced=True, table=False).count == 8 * (k - 1) ** 2
    assert oracle.match(n, e, *g.clique(3), table=False).count == 0
    assert oracle.match(n, e, *g.path(3), table=False).count == 12 * k * k - 24 * k + 8
    mono = oracle.match(n, e, *g.path(4), table=False).count
    assert mono == p4_labelled(simple_adj(n, e))
    if k >= 3:
        assert mono == 36 * k * k - 100 * k + 56
    assert oracle.match(n, e, *g.path(4), induced=True, table=False).count == mono - 8 * (k - 1) ** 2


@pytest.mark.parametrize("k", [3, 8, 64])
def test_oracle_grid_diag_closed_forms(k):
    """P-gdiag (config 2 (i)): triangles 12(k-1)^2; C4 mono 8(k-1)(3k-5); C4 induced 0."""
    n, e = g.grid_diag(k)
    assert oracle.match(n, e, *g.clique(3), table=False).count == 12 * (k - 1) ** 2
    assert oracle.match(n, e, *g.ring(4), table=False).count == 8 * (k - 1) * (3 * k - 5)
    assert oracle.match(n, e, *g.ring(4), table=False).count == c4_labelled(simple_adj(n, e))
    assert oracle.match(n, e, *g.ring(4), induced=True, table=False).count == 0


def test_oracle_falcon_paths_nonbacktracking():
    """P-NB on Falcon-27 (girth 12): labelled P_k for k = 2..12; config 1 (P4) = 80."""
    n, e = g.falcon27()
    for k in range(2, 13):
        assert oracle.match(n, e, *g.path(k), table=False).count == paths_nonbacktracking(n, e, k)
    assert oracle.match(n, e, *g.path(4)).count == 80


@pytest.mark.parametrize("w", [3, 6, 10])
def test_oracle_heavy_hex_paths_and_cycles(w):
    """P-NB (paths, k <= girth 12) and P-hh (C12 = 48 w^2; odd / C10 cycles 0) on config 3."""
    n, e = g.ibm_heavy_hex(w)
    for k in (2, 5, 10, 12):
        assert oracle.match(n, e, *g.path(k), table=False).count == paths_nonbacktracking(n, e, k)
    assert oracle.match(n, e, *g.ring(12), table=False).count == 48 * w * w
    assert oracle.match(n, e, *g.ring(10), table=False).count == 0
    assert oracle.match(n, e, *g.ring(11), table=False).count == 0
    assert oracle.match(n, e, *g.clique(3), table=False).count == 0


def test_oracle_heavy_hex_w31_nonbacktracking():
    """Config 5 data graph: P10/P12 = 1^T B^(k-2) 1 (361,296 / 714,984 per SURVEY P-NB)."""
    n, e = g.ibm_heavy_hex(31)
    for k in (10, 12):
        nb = paths_nonbacktracking(n, e, k)
        assert oracle.match(n, e, *g.path(k), table=False).count == nb
    assert nb == 714_984


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_oracle_heavy_hex_device_subtrees(seed):
    """P-tree: tree patterns with diameter < girth(12) -> locally injective homomorphisms."""
    n, e = g.ibm_heavy_hex(6)
    for size in (6, 10):
        k, te = g.device_subtree(n, e, size, seed)
        want = tree_locally_injective(n, e, k, te)
        assert oracle.match(n, e, k, te, table=False).count == want
    k, te = g.random_tree(8, seed, max_degree=3)
    assert oracle.match(n, e, k, te, table=False).count == tree_locally_injective(n, e, k, te)


@pytest.mark.parametrize("scale", [7, 9])
def test_oracle_rmat_diamond_k4(scale):
    """P-dia and P-K4 on small R-MAT (config 4 family, self-loops dropped)."""
    n, e = g.rmat(scale, 16, seed=1)
    A = simple_adj(n, e)
    assert oracle.match(n, e, *g.clique(3), table=False, drop_self_loops=True).count == \
        6 * tri_count_oriented(n, e) == tri_labelled(A)
    assert oracle.match(n, e, *g.diamond(), table=False, drop_self_loops=True).count == diamonds_labelled(A)
    assert oracle.match(n, e, *g.clique(4), table=False, drop_self_loops=True).count == \
        24 * k4_count_oriented(n, e)


def test_native_pins_agree_with_closed_forms_and_oracle():
    """The native full-scale counters (tests/pins_native.c) against tr(A^3), the diamond closed
    form, and the oracle's K4 count, on R-MAT scale 11/12."""
    from pins import native_counts
    for scale in (11, 12):
        n, e = g.rmat(scale, 16, seed=2)
        A = simple_adj(n, e)
        assert native_counts(n, e, "tri") == tri_labelled(A)
        assert native_counts(n, e, "diamond") == diamonds_labelled(A)
    n, e = g.rmat(11, 16, seed=2)
    assert 24 * native_counts(n, e, "k4") == oracle.match(n, e, *g.clique(4), drop_self_loops=True,
                                                          table=False).count
    n, e = g.clique(7)
    assert native_counts(n, e, "k4") == 35 and native_counts(n, e, "tri") == 210


# ------------------------------------------------------------------------- metamorphic
def test_oracle_relabel_equivariance():
    """P-meta: relabelling the data graph by sigma maps the result set by sigma."""
    n, e = g.er_gnm(40, 160, 5)
    e2, sigma = g.relabel(n, e, 11)
    for (k, pe) in [g.path(4), g.ring(4), g.diamond(), g.star(4)]:
        r1 = oracle.match(n, e, k, pe)
        r2 = oracle.match(n, e2, k, pe)
        mapped = sigma[r1.rows]
        mapped = mapped[np.lexsort(mapped.T[::-1])]
        assert np.array_equal(mapped, r2.rows)


def test_oracle_root_ranges_partition():
    """Root-range restriction partitions the result (used for bounded samples and the
    multi-rank host logic)."""
    n, e = g.ibm_heavy_hex(3)
    full = oracle.match(n, e, *g.path(6))
    parts = [oracle.match(n, e, *g.path(6), roots=(a, b)) for a, b in [(0, 40), (40, 41), (41, n)]]
    assert sum(p.count for p in parts) == full.count
    cat = np.concatenate([p.rows for p in parts])
    cat = cat[np.lexsort(cat.T[::-1])]
    assert np.array_equal(cat, full.rows)


def test_oracle_generator_sizes():
    """Generator pins."""
    assert g.square_grid(40, 40)[0] == 1600 and len(g.square_grid(40, 40)[1]) == 3120
    assert g.square_grid(2, 2)[0] == 4 and len(g.square_grid(2, 2)[1]) == 4
    assert len(g.square_grid(1, 5)[1]) == 4
    assert g.hex_lattice_subdivided(1, 1)[0] == 12
    assert g.hex_lattice_subdivided(11, 33)[0] == 1990
    assert g.hex_lattice_subdivided(25, 34)[0] == 4485
    for w in (3, 6, 10, 31):
        n, e = g.ibm_heavy_hex(w)
        assert n == 10 * w * w + 12 * w + 1 and len(e) == 12 * w * w + 12 * w
        assert simple_adj(n, e).sum(axis=1).max() == 3
    n, e = g.falcon27()
    d = np.bincount(np.asarray(simple_adj(n, e).sum(axis=1)).ravel())
    assert n == 27 and len(e) == 28 and d.tolist() == [0, 6, 13, 8]
