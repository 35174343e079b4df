"""GPU: dm_score_layouts (layout scoring + top-k, §6.5) against the
CPU reference oracle/scoring.py on the oracle's table: identical top-k rows, scores equal
(same float64 product order on both sides; tolerance 1e-12 relative), ties in lexicographic
order, motif-set invariance of the ranking, argument errors."""
import numpy as np
import pytest

import dm_inputs as g
import oracle
from oracle.scoring import layout_scores, top_layouts

pytestmark = pytest.mark.gpu


def _fid(n, e, seed, quantize=False):
    rng = np.random.default_rng(seed)
    node, ef = rng.uniform(0.9, 1.0, n), rng.uniform(0.8, 1.0, len(e))
    if quantize:  # few distinct values -> many equal scores: exercises the tie order
        node, ef = np.round(node, 1), np.round(ef, 1)
    return node, ef


@pytest.mark.parametrize("case", ["falcon-p4", "falcon-p8", "hh3-ring12", "hh3-sub10", "hh10-p12", "grid12-c4"])
@pytest.mark.parametrize("quant", [False, True])
def test_score_layouts_vs_reference(dm, case, quant):
    (n, e), (k, pe) = {
        "falcon-p4": (g.falcon27(), g.path(4)), "falcon-p8": (g.falcon27(), g.path(8)),
        "hh3-ring12": (g.ibm_heavy_hex(3), g.ring(12)),
        "hh3-sub10": (g.ibm_heavy_hex(3), g.random_connected_subgraph(*g.ibm_heavy_hex(3), 10, 3)[:2]),
        "hh10-p12": (g.ibm_heavy_hex(10), g.path(12)), "grid12-c4": (g.grid(12), g.ring(4))}[case]
    node, ef = _fid(n, e, 17, quant)
    G = dm.Graph(n, e)
    rows = oracle.match(n, e, k, pe).rows
    s = layout_scores(rows, n, pe, node, e, ef)
    for top_k in (1, 7, 100000):
        want_r, want_s = top_layouts(rows, s, top_k)
        for motifs in ("all", "M2,M5,M6-O"):
            got_r, got_s, total = G.score_layouts(k, pe, node, e, ef, top_k, motifs=motifs)
            assert total == len(rows)
            assert np.array_equal(got_r, want_r), (case, top_k, motifs)
            assert np.allclose(got_s, want_s, rtol=1e-12, atol=0)


def test_score_layouts_errors(dm):
    n, e = g.falcon27()
    G = dm.Graph(n, e)
    node, ef = _fid(n, e, 1)
    with pytest.raises(dm.DMError):
        G.score_layouts(*g.path(4), node, e, ef, 0)                  # top_k <= 0
    bad = node.copy()
    bad[3] = 1.3
    with pytest.raises(dm.DMError):
        G.score_layouts(*g.path(4), bad, e, ef, 5)                   # fidelity > 1
    with pytest.raises(dm.DMError):
        G.score_layouts(*g.path(4), node, e[1:], ef[1:], 5)          # a coupling without fidelity
    with pytest.raises(dm.DMError):
        G.score_layouts(*g.path(4), node, np.vstack([e, [[0, 26]]]), np.append(ef, 0.9), 5)  # non-edge
    r, s, total = G.score_layouts(*g.clique(3), node, e, ef, 5)      # no layouts: empty, not an error
    assert total == 0 and len(r) == 0
