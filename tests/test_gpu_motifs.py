"""GPU: the motif database (Alg. 2) and table steps (larger motifs, §3.4-3.5,
P:282-287; topology-aware motif sets) against the CPU oracle.

* Res(M) tables: each built table equals the oracle's table of the motif template taken as a
  pattern (every labelled embedding, canonical order), and its arc index points at the first row
  of every (position 0, position 1) arc;
* motif-set invariance: tables / counts identical to the oracle for every motif set, both
  modes, on lattices (ELL path) and non-lattice graphs (CSR path);
* the config-5 count with table tails at full size."""
import numpy as np
import pytest

import dm_inputs as g
import oracle

pytestmark = pytest.mark.gpu

TABLE_MOTIFS = {"M4": (4, False), "M5": (5, False), "M6": (6, False), "M7": (7, False), "M8": (8, False),
                "M4-O": (4, True), "M6-O": (6, True), "M12-O": (12, True)}
SETS = ["heavy-hex", "grid", "M2,M5", "M2,M3,M6", "M2,M7", "M2,M3,M8", "M2,M12-O",
        "M2,M3,M3-O,M4,M4-O,M6-O", "M2,M3,M4,M5,M6,M7,M8,M4-O,M6-O,M12-O"]


def _template(L, cycle):
    e = [(i, i + 1) for i in range(L - 1)]
    if cycle:
        e.append((L - 1, 0))
    return L, np.asarray(e, np.int32)


@pytest.mark.parametrize("graph", ["hh6", "grid20", "er300"])
def test_motif_tables_are_res_m(dm, graph):
    """Res(M) = every labelled embedding of the template (the oracle's table of the template as a
    pattern); toff[arc] = first row whose first two positions are >= that arc."""
    n, e = {"hh6": g.ibm_heavy_hex(6), "grid20": g.grid(20), "er300": g.er_gnm(300, 900, 2)}[graph]
    G = dm.Graph(n, e)
    names = [m for m in TABLE_MOTIFS if not (graph == "er300" and m in ("M8", "M12-O"))]
    info = G.build_motifs(",".join(["M2"] + names))
    off, adj = G.csr()
    src = np.repeat(np.arange(n), np.diff(off))
    for name in names:
        L, cyc = TABLE_MOTIFS[name]
        rows, toff = G.motif_table(name)
        want = oracle.match(n, e, *_template(L, cyc)).rows
        assert info[name][0] == len(want)
        assert np.array_equal(rows, want), name
        key = rows[:, 0].astype(np.int64) * n + rows[:, 1] if len(rows) else np.zeros(0, np.int64)
        arck = src.astype(np.int64) * n + adj
        assert np.array_equal(toff[:-1], np.searchsorted(key, arck, side="left")), name
        assert toff[-1] == len(rows)


@pytest.mark.parametrize("mode", ["mono", "induced"])
@pytest.mark.parametrize("motifs", SETS)
def test_motif_set_invariance_lattices(dm, motifs, mode):
    """S:431 motif-set invariance on heavy-hex (configs 1, 3) and grid lattices: tables equal the
    oracle for paths, rings, device subtrees and random connected subgraphs."""
    cases = [(g.falcon27(), [g.path(4), g.path(9), g.ring(12)]),
             (g.ibm_heavy_hex(6), [g.path(10), g.ring(12), g.device_subtree(*g.ibm_heavy_hex(6), 10, 1)]),
             (g.grid(14), [g.ring(4), g.ring(6), g.path(7), g.random_tree(8, 2, max_degree=4)])]
    for (n, e), pats in cases:
        G = dm.Graph(n, e)
        for s in (1, 2):
            k, pe, _ = g.random_connected_subgraph(n, e, 12, s)
            pats = pats + [(k, pe)]
        for k, pe in pats:
            r = G.match(k, pe, mode=mode, output="both", motifs=motifs)
            o = oracle.match(n, e, k, pe, induced=(mode == "induced"))
            assert r.count == o.count and np.array_equal(r.rows, o.rows), (motifs, mode, k, pe.tolist())
            c = G.match(k, pe, mode=mode, motifs=motifs)
            assert c.count == o.count, (motifs, mode, k, "count")


@pytest.mark.parametrize("motifs", ["heavy-hex", "grid", "M2,M3,M3-O,M4,M4-O,M6-O"])
def test_motif_set_invariance_csr_graphs(dm, motifs):
    """Table steps on graphs without the ELL layout (max degree > 4): seeded ER graphs (SPEC
    acceptance) and grid-with-diagonals, tables and counts, both modes."""
    rng = np.random.default_rng(31)
    for trial in range(12):
        n = int(rng.integers(12, 40))
        n, e = g.er_gnm(n, int(n * rng.uniform(1.5, 3.0)), int(rng.integers(0, 1 << 30)))
        G = dm.Graph(n, e)
        for k, pe in (g.path(5), g.ring(4), g.ring(6), g.star(3)):
            for mode in ("mono", "induced"):
                r = G.match(k, pe, mode=mode, output="both", motifs=motifs)
                o = oracle.match(n, e, k, pe, induced=(mode == "induced"))
                assert np.array_equal(r.rows, o.rows), (trial, motifs, mode, k)
    n, e = g.grid_diag(30)
    G = dm.Graph(n, e)
    for k, pe in (g.ring(4), g.ring(6), g.path(6)):
        r = G.match(k, pe, output="both", motifs=motifs)
        assert np.array_equal(r.rows, oracle.match(n, e, k, pe).rows)


@pytest.mark.parametrize("motifs", ["heavy-hex", "M2,M5", "M2,M3,M6", "M2,M7", "M2,M3,M8"])
def test_config5_p30_motif_sets(dm, motifs):
    """bench.py's workload with table steps: P30 into IBM heavy-hex w=31, count mode, at full size
    (213,555,092 = the oracle's count), repeated (pipelined path) and with a small memory
    budget (chunked)."""
    n, e = g.ibm_heavy_hex(31)
    G = dm.Graph(n, e)
    want = 213_555_092
    for _ in range(3):
        assert G.match(*g.path(30), motifs=motifs).count == want
    assert G.match(*g.path(30), motifs=motifs, mem_budget=64 << 20).count == want


def test_config5_random_subgraphs_motif_sets(dm):
    n, e = g.ibm_heavy_hex(31)
    G = dm.Graph(n, e)
    for s in (1, 2, 3):
        k, pe, _ = g.random_connected_subgraph(n, e, 30, s)
        o = oracle.match(n, e, k, pe)
        for motifs in ("heavy-hex", "M2,M3,M6", "M2,M12-O"):
            r = G.match(k, pe, output="both", motifs=motifs)
            assert np.array_equal(r.rows, o.rows), (s, motifs)


def test_motif_db_save_load(dm, tmp_path):
    """Motif-database persistence: save -> load into a fresh graph built
    from the same edge set in another order gives bit-identical tables (no rebuild) and the same
    results; another graph -> fingerprint error; truncated / corrupted file -> DM_ERR_IO."""
    n, e = g.ibm_heavy_hex(10)
    G = dm.Graph(n, e)
    info = G.build_motifs("M2,M5,M7,M6-O,M12-O")
    path = str(tmp_path / "hh10.dmdb")
    G.save_motifs(path)
    G2 = dm.Graph(n, e[::-1, ::-1].copy())
    G2.load_motifs(path)
    # the triangle-apex table (a1b) persists too
    nr, er = g.rmat(11, 16, seed=2)
    R1 = dm.Graph(nr, er, drop_self_loops=True)
    R1.build_motifs("apex")
    rpath = str(tmp_path / "rmat11.dmdb")
    R1.save_motifs(rpath)
    R2 = dm.Graph(nr, er, drop_self_loops=True)
    R2.load_motifs(rpath)
    assert dm.lib().dm_graph_apex_build_ms(R2._h) == 0.0  # loaded, not built
    ta, tb = R1.apex_table(), R2.apex_table()
    assert np.array_equal(ta[0], tb[0]) and np.array_equal(ta[1], tb[1])
    assert R2.match(*g.clique(4), motifs="apex").count == oracle.match(nr, er, *g.clique(4), drop_self_loops=True,
                                                                       table=False).count
    for m in ("M5", "M7", "M6-O", "M12-O"):
        a, b = G.motif_table(m), G2.motif_table(m)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and info[m][0] == len(b[0])
        assert dm.lib().dm_graph_motif_build_ms(G2._h, dm.MOTIF_BITS[m]) == 0.0   # loaded, not built
    want = oracle.match(n, e, *g.path(20), table=False).count
    assert G2.match(*g.path(20), motifs="M2,M7").count == want
    G3 = dm.Graph(*g.ibm_heavy_hex(6))
    with pytest.raises(dm.DMError) as ei:
        G3.load_motifs(path)
    assert ei.value.code == -1 and "fingerprint" in str(ei.value)
    data = open(path, "rb").read()
    bad = str(tmp_path / "trunc.dmdb")
    open(bad, "wb").write(data[: len(data) // 2])
    G4 = dm.Graph(n, e)
    with pytest.raises(dm.DMError) as ei:
        G4.load_motifs(bad)
    assert ei.value.code == -9
    flip = bytearray(data)
    flip[len(flip) // 2] ^= 0xFF
    open(bad, "wb").write(bytes(flip))
    with pytest.raises(dm.DMError) as ei:
        G4.load_motifs(bad)
    assert ei.value.code == -9
    with pytest.raises(dm.DMError) as ei:
        G4.load_motifs(str(tmp_path / "missing.dmdb"))
    assert ei.value.code == -9


def test_table_step_two_chunk_tail_16bit(dm):
    """A materializing M12-O table step on a 16-bit level whose new columns span two output chunks
    (theta graph of two 12-cycles sharing a 3-vertex path, plus a pendant): the flush packs the
    staged tail into two 16-byte chunks.  Counts against the oracle, both modes, and tables."""
    n, e = g.ibm_heavy_hex(6)
    ed = [(i, (i + 1) % 12) for i in range(12)]
    chain = [2] + list(range(12, 21)) + [0]
    ed += [(chain[i], chain[i + 1]) for i in range(len(chain) - 1)]
    ed.append((6, 21))
    k, pe = 22, np.array(ed, np.int32)
    G = dm.Graph(n, e)
    steps = G.plan(k, pe, motifs="M2,M12-O").describe()["steps"]
    assert any(st.get("table") == "M12-O" for st in steps[:-1])  # an intermediate table step
    for mode in ("mono", "induced"):
        want = oracle.match(n, e, k, pe, table=False, induced=mode == "induced").count
        for motifs in ("M2,M12-O", "all"):
            assert G.match(k, pe, mode=mode, motifs=motifs).count == want, (mode, motifs)
    o = oracle.match(n, e, k, pe)
    r = G.match(k, pe, output="both", motifs="M2,M12-O")
    assert r.count == o.count and np.array_equal(r.rows, o.rows)
