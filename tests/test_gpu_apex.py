"""GPU: the triangle-apex table (Res(M3-O) keyed by arc, Alg. 2)
built on the device equals the oracle's definition (oracle/apex.py) entry for entry, and the
shared-key pair steps that read it (diamond, 4-clique; motif set "apex") equal the oracle's counts,
both modes, at sizes that span many warps and a ragged tail, and at config 4's full size against
the native exact counters."""
import numpy as np
import pytest

import dm_inputs as g
import oracle
from oracle.apex import apex_table
from pins import diamonds_labelled, simple_adj, tri_labelled

pytestmark = pytest.mark.gpu

GRAPHS = {
    "falcon27": lambda: (g.falcon27(), False),           # triangle-free: empty table
    "grid_diag16": lambda: (g.grid_diag(16), False),
    "er1000": lambda: (g.er_gnm(1000, 8000, 2), False),
    "rmat10": lambda: (g.rmat(10, 16, seed=1), True),
    "rmat12": lambda: (g.rmat(12, 16, seed=3), True),
}


@pytest.mark.parametrize("name", list(GRAPHS))
def test_apex_table_equals_definition(dm, name):
    (n, e), drop = GRAPHS[name]()
    G = dm.Graph(n, e, drop_self_loops=drop)
    info = G.build_motifs("apex")
    toff, apex = G.apex_table()
    ee = np.asarray(e).reshape(-1, 2)
    wt, wa = apex_table(n, ee[ee[:, 0] != ee[:, 1]])
    assert info["apex"][0] == len(wa) == tri_labelled(simple_adj(n, e))
    assert np.array_equal(toff, wt) and np.array_equal(apex, wa)


def test_apex_empty_graph(dm):
    G = dm.Graph(5, np.zeros((0, 2), np.int32))
    G.build_motifs("apex")
    toff, apex = G.apex_table()
    assert toff.tolist() == [0] and apex.size == 0
    assert G.match(*g.clique(4), motifs="apex").count == 0


@pytest.mark.parametrize("mode", ["mono", "induced"])
@pytest.mark.parametrize("name", ["grid_diag16", "er1000", "rmat10", "rmat12"])
def test_apex_pair_steps_vs_oracle(dm, name, mode):
    (n, e), drop = GRAPHS[name]()
    G = dm.Graph(n, e, drop_self_loops=drop)
    for pat in (g.diamond(), g.clique(4)):
        want = oracle.match(n, e, *pat, drop_self_loops=drop, table=False, induced=mode == "induced").count
        r = G.match(*pat, motifs="apex", mode=mode, profile=True)
        assert r.count == want, (name, mode, pat)
        assert G.match(*pat, mode=mode).count == want  # implicit-motif path agrees


def test_apex_rmat16_closed_forms(dm):
    n, e = g.rmat(16, 16, seed=1)
    A = simple_adj(n, e)
    G = dm.Graph(n, e, drop_self_loops=True)
    G.build_motifs("apex")
    toff, _ = G.apex_table()
    assert int(toff[-1]) == tri_labelled(A)
    assert G.match(*g.diamond(), motifs="apex").count == diamonds_labelled(A)
    assert G.match(*g.clique(4), motifs="apex").count == G.match(*g.clique(4)).count


def test_apex_full_scale_config4(dm):
    """Config 4 at full size (R-MAT scale 20, ef 16) through the apex pair steps, in bench.py's
    launch configuration: labelled diamonds and 4-cliques against the native exact counters."""
    from pins import native_counts
    n, e = g.rmat(20, 16, seed=1)
    G = dm.Graph(n, e, drop_self_loops=True)
    G.build_motifs("apex")
    assert G.match(*g.diamond(), motifs="apex").count == native_counts(n, e, "diamond")
    assert G.match(*g.clique(4), motifs="apex").count == 24 * native_counts(n, e, "k4")
