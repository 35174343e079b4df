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


def test_checked_variant_exports_every_header_symbol():
    """The bounds-checked build (DM_LIBRARY_VARIANT=checked) is the same ABI with device asserts."""
    import subprocess
    import sys
    code = ("import ctypes, paper_2508_21287_b200 as dm; assert dm.LIB_PATH.endswith('libdeltamotif_checked.so'); "
            "L = dm.lib(); assert L.dm_abi_version() == dm.ABI_VERSION; "
            "raw = ctypes.CDLL(dm.LIB_PATH); [getattr(raw, s) for s in dm.EXPORTS]; print('ok')")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=300,
                       env=dict(os.environ, DM_LIBRARY_VARIANT="checked"))
    assert r.returncode == 0 and r.stdout.strip() == "ok", r.stderr[-2000:]


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
    tmpl = _templates()
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
    slices = P.slices()
    for st in d["steps"]:
        if "table" in st:   # table step: one slice's fresh vertices from Res(M) (Alg. 1 l.6)
            w = st["in_w"]
            T = slices[st["slice"]]
            assert T["motif"] == st["table"]
            pos = {0: cols[st["key0"]]}
            if st["key1"] >= 0:
                pos[1] = cols[st["key1"]]
            for p, c in st["eq"]:
                assert c < w
                pos[p] = cols[c]
            for j, p in enumerate(st["newpos"]):
                pos[p] = cols[w + j]
            L = len(T["vertices"])
            assert sorted(pos) == list(range(L)) and sorted(pos.values()) == sorted(T["vertices"])
            assert st["key0"] < w and all(c < w for c in [st["key1"]] if c >= 0)
            newv = {cols[w + j] for j in range(st["n_new"])}
            for a, b in tmpl[st["table"]]:   # the template maps onto pattern edges
                assert padj[pos[a], pos[b]]
                if pos[a] in newv or pos[b] in newv:
                    enforced.append(tuple(sorted((pos[a], pos[b]))))
            for j, c, neg in st["probes"]:
                assert c < w + j
                (nonenf if neg else enforced).append(tuple(sorted((cols[c], cols[w + j]))))
            if mode == "induced":   # non-edges inside the slice are probed too
                pass
            continue
        assert 1 <= len(st["new"]) <= 4
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


def _templates():
    t = {"M2": [(0, 1)], "M3": [(0, 1), (1, 2)], "M3-O": [(0, 1), (1, 2), (0, 2)]}
    for L in (4, 5, 6, 7, 8):
        t[f"M{L}"] = [(i, i + 1) for i in range(L - 1)]
    for L in (4, 6, 12):
        t[f"M{L}-O"] = [(i, i + 1) for i in range(L - 1)] + [(L - 1, 0)]
    return t


TABLE_SETS = ["heavy-hex", "grid", "M2,M5", "M2,M3,M6", "M2,M7", "M2,M3,M8", "M2,M12-O",
              "M2,M3,M3-O,M4,M5,M6,M7,M8,M4-O,M6-O,M12-O"]


@pytest.mark.parametrize("motifs", TABLE_SETS)
@pytest.mark.parametrize("mode", ["mono", "induced"])
def test_plan_table_motifs_valid(dm, motifs, mode):
    """Decompositions with the larger motifs and their table steps: every
    template maps onto pattern edges, full edge coverage, every pattern edge enforced
    exactly once (by a Res(M) template edge of the step that places it, or a probe), every
    non-edge probed in induced mode."""
    rng = np.random.default_rng(11)
    cases = [g.path(30), g.ring(12), g.ring(6), g.path(7)]
    for lat in (g.ibm_heavy_hex(6), g.grid(12), g.hex_lattice_subdivided(3, 4)):
        for sz in (8, 14, 25):
            k, pe, _ = g.random_connected_subgraph(*lat, sz, int(rng.integers(0, 1 << 30)))
            cases.append((k, pe))
    for k, pe in cases:
        _check_plan(dm, k, pe, motifs, mode=mode)


def test_plan_table2_sizes_fast(dm):
    """100-vertex random subgraphs of the paper's lattices plan in well under a
    second with every motif set (the decomposition is <1% of the runtime)."""
    import time
    for lat, sets in ((g.hex_lattice_subdivided(25, 34), ("all", "heavy-hex")), (g.grid(60), ("all", "grid"))):
        for seed in (1, 2):
            k, pe, _ = g.random_connected_subgraph(*lat, 100, seed)
            for m in sets:
                t = time.perf_counter()
                P = dm.Plan(k, pe, motifs=m)
                assert time.perf_counter() - t < 1.0
                assert P.width(P.num_steps) == 100


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
