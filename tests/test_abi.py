"""C-ABI boundary checks that need no GPU: the library loads, exports every symbol
include/deltamotif.h declares, reports errors through status codes, and the host planner
(dm_plan_*) produces a valid decomposition (§3.3)."""
import ctypes
import itertools
import os
import re

import numpy as np
import pytest

import dm_inputs as g

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def dm():
    import paper_2508_21287_b200 as dm_mod
    dm_mod.lib()
    return dm_mod


def header_symbols():
    src = open(os.path.join(ROOT, "include", "deltamotif.h")).read()
    return sorted(set(re.findall(r"DM_API[^;(]*?\b(dm_\w+)\s*\(", src)))


def test_exports_every_header_symbol(dm):
    syms = header_symbols()
    assert len(syms) >= 20
    assert sorted(dm.EXPORTS) == syms
    raw = ctypes.CDLL(dm.LIB_PATH)
    for s in syms:
        assert getattr(raw, s) is not None


def test_abi_version_and_opts_defaults(dm):
    L = dm.lib()
    assert L.dm_abi_version() == dm.ABI_VERSION
    o = dm._Opts()
    L.dm_match_opts_init(ctypes.byref(o))
    assert o.mode == dm.DM_MONO and o.output == dm.DM_OUT_COUNT and o.seed_end == -1
    assert o.motifs == dm.DM_MOTIF_M2 | dm.DM_MOTIF_M3 | dm.DM_MOTIF_M3O


def test_no_cpu_fallback(dm):
    """Without a CUDA device the computational entry points fail loudly (DM_ERR_CUDA)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(dm.DMError) as ei:
        dm.Graph(3, [(0, 1), (1, 2)])
    assert ei.value.code == -7


# ------------------------------------------------------------------------------ planner
def _check_plan(dm, k, pe, motifs, mode="mono"):
    P = dm.Plan(k, pe, motifs=motifs, mode=mode)
    d = P.describe()
    padj = np.zeros((k, k), bool)
    for a, b in np.asarray(pe).reshape(-1, 2).tolist():
        padj[a, b] = padj[b, a] = True
    tmpl = {"M2": [(0, 1)], "M3": [(0, 1), (1, 2)], "M3-O": [(0, 1), (1, 2), (0, 2)]}
    covered = set()
    union = set()
    for i, s in enumerate(P.slices()):
        vs = s["vertices"]
        assert len(set(vs)) == len(vs)
        for a, b in tmpl[s["motif"]]:          # replay: template edges -> pattern edges
            assert padj[vs[a], vs[b]]
            covered.add((min(vs[a], vs[b]), max(vs[a], vs[b])))
        assert sorted(s["constraints"]) == sorted(set(vs) & union)   # shared vertices
        if i > 0:
            assert s["constraints"], "every join after the first has constraints (S:330)"
        union |= set(vs)
    edges = {(a, b) for a in range(k) for b in range(a + 1, k) if padj[a, b]}
    assert covered == edges, "full edge coverage (S:329)"
    # join program: every vertex placed once, every pattern edge enforced exactly once at its
    # later endpoint, every non-edge enforced in induced mode
    cols = d["col_pvert"]
    assert sorted(cols) == list(range(k)) and cols[0] == P.first_vertex
    enforced, nonenf = [], []
    for st in d["steps"]:
        assert 1 <= len(st["new"]) <= 2
        w = st["in_w"]
        for j, nv in enumerate(st["new"]):
            col = w + j
            assert cols[col] == nv["pvert"]
            assert nv["nbr_cols"], "each new vertex is joined on at least one key"
            for c in nv["nbr_cols"]:
                assert c < col
                enforced.append(tuple(sorted((cols[c], nv["pvert"]))))
            for c in nv["non_cols"]:
                nonenf.append(tuple(sorted((cols[c], nv["pvert"]))))
    assert sorted(enforced) == sorted(edges)
    if mode == "induced":
        non = {(a, b) for a in range(k) for b in range(a + 1, k) if not padj[a, b]}
        assert sorted(nonenf) == sorted(non)
    else:
        assert not nonenf
    return P, d


def test_plan_paths_use_wedge_chain(dm):
    P, d = _check_plan(dm, *g.path(30), "all")
    sl = P.slices()
    assert [s["motif"] for s in sl] == ["M3"] * 14 + ["M2"]
    assert sl[0]["vertices"] == [0, 1, 2] and sl[1]["vertices"] == [2, 3, 4]
    assert sl[1]["constraints"] == [2]
    assert P.num_steps == 15


def test_plan_m2_only_slice_count(dm):
    """M2-only: #slices = |E_p| (§6.3)."""
    rng = np.random.default_rng(3)
    for trial in range(40):
        n, e = g.ibm_heavy_hex(3)
        k, pe, _ = g.random_connected_subgraph(n, e, int(rng.integers(2, 25)), int(rng.integers(0, 1 << 30)))
        P, _ = _check_plan(dm, k, pe, "M2")
        assert len(P.slices()) == len(pe)


def test_plan_cycle_and_cliques(dm):
    P, d = _check_plan(dm, *g.ring(4), "all")
    assert [s["motif"] for s in P.slices()] == ["M3", "M3"]
    assert P.slices()[1]["constraints"] == [0, 2]        # 2-key join: N(f(0)) ∩ N(f(2))
    P, _ = _check_plan(dm, *g.clique(3), "all")
    assert [s["motif"] for s in P.slices()] == ["M3-O"]
    P, _ = _check_plan(dm, *g.diamond(), "all")
    assert [s["motif"] for s in P.slices()] == ["M3-O", "M3-O"]
    assert P.slices()[1]["constraints"] == [1, 2]
    P, _ = _check_plan(dm, *g.clique(4), "all")
    assert P.slices()[0]["motif"] == "M3-O"


@pytest.mark.parametrize("motifs", ["M2", "M3", "M3O", "all"])
@pytest.mark.parametrize("mode", ["mono", "induced"])
def test_plan_random_patterns_valid(dm, motifs, mode):
    rng = np.random.default_rng(11)
    for trial in range(30):
        k = int(rng.integers(1, 12))
        while True:
            e = [(a, b) for a, b in itertools.combinations(range(k), 2) if rng.random() < 0.45]
            adj = {i: set() for i in range(k)}
            for a, b in e:
                adj[a].add(b); adj[b].add(a)
            seen, st = {0}, [0]
            while st:
                v = st.pop()
                for u in adj[v] - seen:
                    seen.add(u); st.append(u)
            if len(seen) == k:
                break
        _check_plan(dm, k, np.asarray(e, np.int32).reshape(-1, 2), motifs, mode)


def test_plan_errors(dm):
    with pytest.raises(dm.DMError) as ei:
        dm.Plan(4, [(0, 1), (2, 3)])
    assert ei.value.code == -4
    with pytest.raises(dm.DMError) as ei:
        dm.Plan(3, [(0, 0), (0, 1), (1, 2)])
    assert ei.value.code == -3
    with pytest.raises(dm.DMError) as ei:
        dm.Plan(3, [(0, 5)])
    assert ei.value.code == -2
    with pytest.raises(dm.DMError) as ei:
        dm.Plan(129, [(i, i + 1) for i in range(128)])
    assert ei.value.code == -8
    P = dm.Plan(100, [(i, i + 1) for i in range(99)])   # the paper's Table 2 sizes go to 100
    assert P.width(P.num_steps) == 100 and P.num_steps <= dm.DM_MAX_STEPS
    P = dm.Plan(1, np.zeros((0, 2), np.int32))
    assert P.num_steps == 0 and P.first_vertex == 0


def test_plan_cost_model_prefers_shared_key_pairs(dm):
    """With skewed, clustered graph statistics (R-MAT-like) the planner regroups the diamond /
    4-clique placement so the count-only last step adds both apexes from one edge (shared-key
    pair); with lattice statistics a path's last step adds two vertices."""
    rm = dict(n=1 << 20, arcs=31404412, sum_d2=31404412 * 3000.0, closure=0.03, count_only=True)
    d = dm.Plan(*g.diamond(), stats=rm).describe()
    assert [len(s["new"]) for s in d["steps"]] == [1, 2]
    last = d["steps"][-1]["new"]
    assert sorted(last[0]["nbr_cols"]) == sorted(last[1]["nbr_cols"]) == [0, 1]
    d = dm.Plan(*g.clique(4), stats=rm).describe()
    last = d["steps"][-1]["new"]
    assert len(last) == 2 and sorted(last[1]["nbr_cols"]) == sorted(last[0]["nbr_cols"] + [2])
    hh = dict(n=9983, arcs=23808, sum_d2=23808 * 2.5, closure=0.0, count_only=True)
    d = dm.Plan(*g.path(30), stats=hh).describe()
    assert len(d["steps"][-1]["new"]) == 2 and len(d["steps"]) == 15
    with pytest.raises(dm.DMError):
        dm.Plan(*g.path(3), stats=dict(n=0, arcs=1, sum_d2=1))
