"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element,
on the same seeded inputs.  Integer work -> bit-exact tables and counts.

Sizes: small cases span several 256-row tiles with ragged tails; the BASELINE configs run at
full size (config 5 = bench.py's workload, compared on the full count)."""
import numpy as np
import pytest

import dm_inputs as g
import oracle
from golden_util import graph_from_name, spec_examples
from pins import c4_labelled, diamonds_labelled, simple_adj, tri_labelled

pytestmark = pytest.mark.gpu

MOTIF_SETS = ["M2", "M3", "M3O", "all"]


def _pattern(rng, k, p):
    import itertools
    while True:
        e = [(a, b) for a, b in itertools.combinations(range(k), 2) if rng.random() < p]
        adj = {i: set() for i in range(k)}
        for a, b in e:
            adj[a].add(b); adj[b].add(a)
        seen, st = {0}, [0]
        while st:
            v = st.pop()
            for u in adj[v] - seen:
                seen.add(u); st.append(u)
        if len(seen) == k:
            return k, np.asarray(e, np.int32).reshape(-1, 2)


def _same(dm, n, e, k, pe, mode="mono", motifs="all", drop=False, **kw):
    G = dm.Graph(n, e, drop_self_loops=drop)
    r = G.match(k, pe, mode=mode, output="both", motifs=motifs, **kw)
    o = oracle.match(n, e, k, pe, induced=(mode == "induced"), drop_self_loops=drop)
    assert r.count == o.count
    assert r.rows.shape == o.rows.shape
    assert np.array_equal(r.rows, o.rows)
    return r


# ------------------------------------------------------------------------- CSR builder
def test_csr_builder_matches_definition(dm):
    """Res(M2) = E_d minus self-loops, both orientations, sorted, deduplicated."""
    for n, e in [g.rmat(12, 8, seed=3), g.er_gnm(5000, 40000, 2), g.ibm_heavy_hex(10)]:
        e2 = np.concatenate([e, e[: len(e) // 3, ::-1]])   # duplicates + reversed pairs
        G = dm.Graph(n, e2, drop_self_loops=True)
        off, adj = G.csr()
        A = simple_adj(n, e2)
        assert np.array_equal(off, A.indptr.astype(np.int64))
        assert np.array_equal(adj, A.indices.astype(np.int32))
        assert G.num_arcs == A.nnz
        assert G.max_degree == int(np.diff(A.indptr).max())


def test_graph_errors(dm):
    with pytest.raises(dm.DMError) as ei:
        dm.Graph(3, [(0, 3)])
    assert ei.value.code == -2
    with pytest.raises(dm.DMError) as ei:
        dm.Graph(3, [(1, 1)])
    assert ei.value.code == -3
    G = dm.Graph(3, [(1, 1), (0, 1)], drop_self_loops=True)
    assert G.num_arcs == 2
    G = dm.Graph(5, np.zeros((0, 2), np.int32))
    assert G.num_arcs == 0
    assert G.match(2, [(0, 1)]).count == 0
    assert G.match(1, np.zeros((0, 2), np.int32)).count == 5
    with pytest.raises(dm.DMError) as ei:
        G.match(4, [(0, 1), (2, 3)])
    assert ei.value.code == -4


# ------------------------------------------------------------------- small exhaustive
@pytest.mark.parametrize("motifs", MOTIF_SETS)
@pytest.mark.parametrize("mode", ["mono", "induced"])
def test_parity_random_er(dm, motifs, mode):
    """SPEC acceptance 1: seeded ER data graphs n in [10,40], p in [0.15,0.4],
    connected patterns of 3-8 vertices; exact table equality with the oracle."""
    rng = np.random.default_rng(1000 + MOTIF_SETS.index(motifs) + (10 if mode == "induced" else 0))
    for trial in range(40):
        n = int(rng.integers(10, 41))
        p = float(rng.uniform(0.15, 0.4))
        n, e = g.er_gnm(n, max(1, int(p * n * (n - 1) / 2)), int(rng.integers(0, 1 << 30)))
        k, pe = _pattern(rng, int(rng.integers(3, 9)), float(rng.uniform(0.25, 0.7)))
        _same(dm, n, e, k, pe, mode=mode, motifs=motifs)


@pytest.mark.parametrize("mode", ["mono", "induced"])
def test_parity_count_mode_random(dm, mode):
    """Count mode (count-only last step: row-serial, candidate-partitioned or shared-key pair
    kernel depending on degree and plan) against the oracle's count; denser ER graphs make the
    planner choose shared-key pair last steps."""
    rng = np.random.default_rng(77 + (mode == "induced"))
    for trial in range(40):
        n = int(rng.integers(20, 120))
        m = int(n * rng.uniform(2.0, 8.0))
        n, e = g.er_gnm(n, min(m, n * (n - 1) // 2), int(rng.integers(0, 1 << 30)))
        k, pe = _pattern(rng, int(rng.integers(3, 7)), float(rng.uniform(0.3, 0.9)))
        G = dm.Graph(n, e)
        r = G.match(k, pe, mode=mode)
        o = oracle.match(n, e, k, pe, induced=(mode == "induced"), table=False)
        assert r.count == o.count, (trial, k, pe.tolist())
    for pat in (g.diamond(), g.clique(4), g.path(3), g.star(3)):
        n, e = g.rmat(11, 16, seed=5)
        G = dm.Graph(n, e, drop_self_loops=True)
        for mode2 in ("mono", "induced"):
            assert G.match(*pat, mode=mode2).count == oracle.match(
                n, e, *pat, drop_self_loops=True, induced=(mode2 == "induced"), table=False).count


@pytest.mark.parametrize("case", spec_examples(), ids=lambda c: c[0])
def test_parity_spec_examples(dm, case):
    name, data, pat, mode, exp, cite = case
    n, e = graph_from_name(data)
    k, pe = graph_from_name(pat)
    r = _same(dm, n, e, k, pe, mode=mode)
    assert r.count == exp, cite


def test_degenerate_cases(dm):
    n, e = g.ring(7)
    r = _same(dm, n, e, 1, np.zeros((0, 2), np.int32))
    assert r.count == 7
    r = _same(dm, 3, [(0, 1), (1, 2)], 4, g.path(4)[1])       # k > n -> 0
    assert r.count == 0
    _same(dm, 12, g.er_gnm(12, 20, 3)[1], *g.clique(5))       # typically empty
    # isolated vertices in the data graph (Q6)
    _same(dm, 50, [(0, 1), (1, 2), (2, 0), (10, 11)], *g.path(3))


# --------------------------------------------------------------------- BASELINE configs
def test_config1_falcon_p4(dm):
    n, e = g.falcon27()
    r = _same(dm, n, e, *g.path(4))
    assert r.count == 80


@pytest.mark.parametrize("pat", ["tri", "c4"])
def test_config2_grid_diag_64(dm, pat):
    n, e = g.grid_diag(64)
    k, pe = g.clique(3) if pat == "tri" else g.ring(4)
    r = _same(dm, n, e, k, pe)
    assert r.count == (47_628 if pat == "tri" else 94_248)
    assert _same(dm, n, e, k, pe, mode="induced").count == (47_628 if pat == "tri" else 0)


@pytest.mark.parametrize("seed", [1, 2])
def test_config2_er(dm, seed):
    n, e = g.er_gnm(10_000, 80_000, seed)
    A = simple_adj(n, e)
    r = _same(dm, n, e, *g.clique(3))
    assert r.count == tri_labelled(A)
    for motifs in ("M2", "all"):
        r = _same(dm, n, e, *g.ring(4), motifs=motifs)
        assert r.count == c4_labelled(A)


@pytest.mark.parametrize("w", [3, 6, 10])
def test_config3_heavy_hex(dm, w):
    n, e = g.ibm_heavy_hex(w)
    pats = [g.path(10), g.path(12), g.path(16), g.path(20), g.ring(10), g.ring(12), g.ring(20)]
    for s in (1, 2, 3):
        pats.append(g.device_subtree(n, e, 10 if w == 3 else 15, s))
        k, pe, _ = g.random_connected_subgraph(n, e, 12 if w == 3 else 20, s)
        pats.append((k, pe))
    for (k, pe) in pats:
        _same(dm, n, e, k, pe)
    if w == 10:
        G = dm.Graph(n, e)
        assert G.match(*g.path(20)).count == 808_020
        assert G.match(*g.ring(12)).count == 4_800 and G.match(*g.ring(20)).count == 21_640


def test_config4_rmat_tables(dm):
    """R-MAT scale 10 (config 4 down-scaled): full tables, every motif set."""
    n, e = g.rmat(10, 16, seed=1)
    for pat in (g.diamond(), g.clique(4), g.clique(3)):
        for motifs in ("all", "M2"):
            _same(dm, n, e, *pat, drop=True, motifs=motifs)


def test_config4_rmat12(dm):
    """Scale 12: triangle table + diamond / K4 counts (2.3e8 / 9.7e7 rows exceed the table
    row budget) against the oracle."""
    n, e = g.rmat(12, 16, seed=1)
    _same(dm, n, e, *g.clique(3), drop=True)
    G = dm.Graph(n, e, drop_self_loops=True)
    for pat in (g.diamond(), g.clique(4)):
        assert G.match(*pat).count == oracle.match(n, e, *pat, drop_self_loops=True, table=False).count


def test_config4_rmat16_counts(dm):
    """Scale 16 counts: P-tri / P-dia closed forms (2.1e10 labelled diamonds)."""
    n, e = g.rmat(16, 16, seed=1)
    A = simple_adj(n, e)
    G = dm.Graph(n, e, drop_self_loops=True)
    assert G.match(*g.clique(3)).count == tri_labelled(A)
    assert G.match(*g.diamond()).count == diamonds_labelled(A)


def test_config4_full_scale_diamond_k4(dm):
    """Config 4 at full size in bench.py's launch configuration (R-MAT scale 20, ef 16, count
    mode): labelled diamonds and 4-cliques against the native exact counters (P-dia via
    per-edge sorted merges; P-K4 via a degree-oriented counter) -- the oracle would need ~1e5
    core-seconds here."""
    from pins import native_counts
    n, e = g.rmat(20, 16, seed=1)
    G = dm.Graph(n, e, drop_self_loops=True)
    assert G.match(*g.diamond()).count == native_counts(n, e, "diamond")
    assert G.match(*g.clique(4)).count == 24 * native_counts(n, e, "k4")


def test_config4_rmat13_k4_count(dm):
    n, e = g.rmat(13, 16, seed=2)
    G = dm.Graph(n, e, drop_self_loops=True)
    k4 = G.match(*g.clique(4)).count
    assert k4 == oracle.match(n, e, *g.clique(4), drop_self_loops=True, table=False).count


def test_config5_p30_count_full(dm):
    """bench.py's workload at full size: P30 into IBM heavy-hex w=31 (9,983 V), count mode,
    against the oracle's full count (213,555,092); also with a tiny mem_budget (chunked)."""
    n, e = g.ibm_heavy_hex(31)
    G = dm.Graph(n, e)
    want = oracle.match(n, e, *g.path(30), table=False).count
    assert want == 213_555_092
    r = G.match(*g.path(30), profile=True)
    assert r.count == want
    r2 = G.match(*g.path(30), mem_budget=64 << 20)
    assert r2.count == want and r2.stats["num_chunks"] > r.stats["num_chunks"]


@pytest.mark.parametrize("w", [3, 10])
def test_heavy_hex_count_mode_deep_steps(dm, w):
    """Count mode on max-degree-3 graphs: the planner ends with a 3-4 vertex depth-first step
    (ELL row-serial kernel); counts must equal the oracle's, for paths, rings, trees and random
    subgraphs, in both modes."""
    n, e = g.ibm_heavy_hex(w)
    G = dm.Graph(n, e)
    pats = [g.path(7), g.path(12), g.ring(12), g.path(20) if w == 10 else g.path(9)]
    for s in (1, 2):
        pats.append(g.device_subtree(n, e, 12, s))
        k, pe, _ = g.random_connected_subgraph(n, e, 14, s)
        pats.append((k, pe))
    for (k, pe) in pats:
        for mode in ("mono", "induced"):
            r = G.match(k, pe, mode=mode)
            o = oracle.match(n, e, k, pe, induced=(mode == "induced"), table=False)
            assert r.count == o.count, (k, pe.tolist(), mode)


@pytest.mark.parametrize("graph", ["grid120", "hh31"])
def test_deep_tail_counts(dm, graph):
    """Count mode with a deep tail (3-4 new vertices enumerated per row, never materialized) on
    large max-degree-3/4 lattices (several tiles per level, 16-bit frontier levels): paths,
    rings (closing edge into the materialized columns), trees, stars and random subgraphs
    (several keys per vertex, known-duplicate shortcut only on the first key), both modes;
    counts must equal the oracle's."""
    if graph == "grid120":
        n, e = g.grid(120)
        pats = [g.path(9), g.ring(10), g.ring(8), g.star(4)]
        sizes = (9, 10)
    else:
        n, e = g.ibm_heavy_hex(31)
        pats = [g.path(12), g.path(14), g.ring(12), g.star(3)]
        sizes = (12, 14)
    G = dm.Graph(n, e)
    for s in (1, 2):
        pats.append(g.random_tree(sizes[0], s, max_degree=3) if graph == "grid120"
                    else g.device_subtree(n, e, sizes[0], s))
        k, pe, _ = g.random_connected_subgraph(n, e, sizes[1], s)
        pats.append((k, pe))
    deep = 0
    for (k, pe) in pats:
        for mode in ("mono", "induced"):
            r = G.match(k, pe, mode=mode, profile=True)
            st = r.stats
            deep += (st["width_out"][-1] - st["width_in"][-1]) >= 3
            o = oracle.match(n, e, k, pe, induced=(mode == "induced"), table=False)
            assert r.count == o.count, (graph, k, pe.tolist(), mode)
    assert deep >= 4


def test_pipelined_repeat_queries(dm):
    """A repeated count query is enqueued without per-step host synchronisation (capacities
    from the previous identical run, sizes read on the device) when every materializing step
    runs in the row-serial kernel (max degree <= 4 here; the others stay on the synchronising
    path): counts and per-step row statistics must equal the first run and the oracle, for
    several graphs, patterns, modes and seed ranges."""
    cases = [(g.ibm_heavy_hex(10), g.path(16), "mono", None), (g.ibm_heavy_hex(10), g.ring(12), "induced", None),
             (g.grid(60), g.path(8), "mono", (100, 2000)), (g.grid_diag(40), g.ring(5), "mono", None),
             (g.er_gnm(2000, 6000, 3), g.path(6), "induced", None)]
    for (n, e), (k, pe), mode, seeds in cases:
        G = dm.Graph(n, e)
        kw = {"seed_range": seeds} if seeds else {}
        first = G.match(k, pe, mode=mode, profile=True, **kw)
        assert not first.stats["pipelined"]
        if seeds:  # a seed shard: the first (synchronising) run is the reference
            want = first.count
        else:
            want = oracle.match(n, e, k, pe, induced=(mode == "induced"), table=False).count
            assert first.count == want
        for _ in range(2):
            r = G.match(k, pe, mode=mode, profile=True, **kw)
            assert r.count == want
            assert r.stats["rows_out"][:-1] == first.stats["rows_out"][:-1]
            assert r.stats["candidates"] == first.stats["candidates"]
        if G.max_degree <= 4 and first.stats["num_steps"] > 1:  # every step row-serial
            assert r.stats["pipelined"], (k, mode)


def test_config5_random_subgraphs(dm):
    n, e = g.ibm_heavy_hex(31)
    G = dm.Graph(n, e)
    for s in (1, 2, 3):
        k, pe, _ = g.random_connected_subgraph(n, e, 30, s)
        r = G.match(k, pe, output="both")
        o = oracle.match(n, e, k, pe)
        assert np.array_equal(r.rows, o.rows)


# ---------------------------------------------------------------------- metamorphic
def test_seed_ranges_partition(dm):
    """Disjoint seed ranges partition the result (the multi-GPU sharding contract)."""
    n, e = g.ibm_heavy_hex(6)
    G = dm.Graph(n, e)
    k, pe = g.path(9)
    full = G.match(k, pe, output="table").rows
    cuts = [0, 17, 18, 200, n]
    parts = [G.match(k, pe, output="table", seed_range=(a, b)).rows for a, b in zip(cuts, cuts[1:])]
    cat = np.concatenate(parts)
    cat = cat[np.lexsort(cat.T[::-1])]
    assert np.array_equal(cat, full)


def test_prefix_resume_split(dm):
    """dm_match_prefix + dm_match_resume: a level cut into two row sets and finished separately
    gives the oracle's result (the multi-GPU frontier exchange contract)."""
    import torch
    cases = [(g.ibm_heavy_hex(6), g.path(11), False), (g.rmat(10, 16, seed=3), g.diamond(), True),
             (g.grid_diag(20), g.ring(5), False), (g.er_gnm(300, 2000, 4), g.clique(4), False)]
    for (n, e), (k, pe), drop in cases:
        G = dm.Graph(n, e, drop_self_loops=drop)
        full = G.match(k, pe, output="both")
        o = oracle.match(n, e, k, pe, drop_self_loops=drop)
        assert full.count == o.count and np.array_equal(full.rows, o.rows)
        nsteps = dm.Plan(k, pe, stats=G.stats(count_only=False)).num_steps
        assert nsteps == full.stats["num_steps"]
        assert dm.Plan(k, pe, stats=G.stats()).num_steps == G.match(k, pe).stats["num_steps"]
        for step in range(1, max(2, nsteps)):
            try:
                fr = G.match_prefix(k, pe, step, output="both")
            except dm.DMError:
                continue
            rows = fr.rows_tensor()
            assert rows.shape == (fr.rows, fr.stride) and fr.work_tensor().shape == (fr.rows,)
            cut = fr.rows // 3
            a = G.match_resume(k, pe, step, rows[:cut].contiguous(), output="both")
            b = G.match_resume(k, pe, step, rows[cut:].contiguous(), output="both")
            assert a.count + b.count == o.count
            cat = np.concatenate([a.rows, b.rows])
            cat = cat[np.lexsort(cat.T[::-1])]
            assert np.array_equal(cat, o.rows)
            c = G.match_resume(k, pe, step, rows, output="both")
            assert c.count == o.count
            with pytest.raises(ValueError):   # wrong layout is rejected before the library call
                G.match_resume(k, pe, step, rows[:, :-1].contiguous(), output="both")
    with pytest.raises(dm.DMError):
        G.match_prefix(k, pe, 0)


def test_chunking_and_budgets(dm):
    n, e = g.ibm_heavy_hex(10)
    G = dm.Graph(n, e)
    k, pe = g.path(14)
    a = G.match(k, pe, output="table")
    b = G.match(k, pe, output="table", mem_budget=1 << 16)
    assert np.array_equal(a.rows, b.rows) and b.stats["num_chunks"] > a.stats["num_chunks"]
    assert G.match(k, pe).count == a.count
    with pytest.raises(dm.DMError) as ei:
        G.match(k, pe, output="table", row_budget=1000)
    assert ei.value.code == -6


def test_plan_invariance_and_relabel(dm):
    n, e = g.grid(12)
    e2, sigma = g.relabel(n, e, 5)
    G, G2 = dm.Graph(n, e), dm.Graph(n, e2)
    for (k, pe) in (g.ring(6), g.path(6), g.star(4)):
        tabs = [G.match(k, pe, output="table", motifs=m).rows for m in MOTIF_SETS]
        for t in tabs[1:]:
            assert np.array_equal(t, tabs[0])
        t2 = G2.match(k, pe, output="table").rows
        m = sigma[tabs[0]]
        m = m[np.lexsort(m.T[::-1])]
        assert np.array_equal(m, t2)


def test_stream_argument(dm):
    import torch
    n, e = g.ibm_heavy_hex(6)
    G = dm.Graph(n, e)
    s = torch.cuda.Stream()
    r = G.match(*g.path(12), stream=s)
    assert r.count == G.match(*g.path(12)).count
