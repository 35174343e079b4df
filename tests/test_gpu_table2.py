"""GPU: the paper's Table 2 workload shape (§6.2) against the oracle.

Data graphs: heavy-hex as subdivided hexagonal lattices (11,33) -> 1,990 V and (25,34) -> 4,485 V
(DESIGN reading Q16), square grids 40x40 and 60x60.  Patterns: seeded random connected subgraphs
of 20 / 40 / 60 vertices (tables, element by element) and 80 / 100 vertices (counts), with the
implicit motif set and the paper's topology-aware sets ({M2, M4} heavy-hex, {M2, M4-O, M6-O} grid,
P:439).  Seeds are ours (the paper's 200 seeds are not published: parity unpinned for
seed-for-seed numbers); they are screened by scripts/pick_table2_seeds.py (oracle only) to keep
the CPU oracle within seconds -- random-walk subgraphs of lattices are often trees with 1e7-1e8
labelled embeddings -- and stored with their oracle counts in tests/golden/table2_seeds.json."""
import json
import os

import numpy as np
import pytest

import dm_inputs as g
import oracle

pytestmark = pytest.mark.gpu

SEEDS = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "table2_seeds.json")))["seeds"]

LATTICES = {
    "hex11x33": (lambda: g.hex_lattice_subdivided(11, 33), "heavy-hex"),
    "hex25x34": (lambda: g.hex_lattice_subdivided(25, 34), "heavy-hex"),
    "grid40": (lambda: g.grid(40), "grid"),
    "grid60": (lambda: g.grid(60), "grid"),
}


@pytest.mark.parametrize("size", [20, 40, 60])
@pytest.mark.parametrize("lattice", list(LATTICES))
def test_table2_tables(dm, lattice, size):
    gfn, tset = LATTICES[lattice]
    n, e = gfn()
    G = dm.Graph(n, e)
    for seed, want in SEEDS[f"{lattice}/{size}"]:
        k, pe, wit = g.random_connected_subgraph(n, e, size, seed)
        o = oracle.match(n, e, k, pe)
        assert o.count == want >= 1  # the sampled subgraph itself is an embedding
        for motifs in ("all", tset):
            r = G.match(k, pe, output="both", motifs=motifs)
            assert r.count == o.count and np.array_equal(r.rows, o.rows), (lattice, size, seed, motifs)
        # the witness embedding is one of the rows
        assert (r.rows == wit).all(axis=1).any()
    if size == 40:  # induced mode on one of them (the patterns are induced subgraphs of the lattice)
        k, pe, _ = g.random_connected_subgraph(n, e, size, SEEDS[f"{lattice}/{size}"][0][0])
        o = oracle.match(n, e, k, pe, induced=True)
        r = G.match(k, pe, mode="induced", output="both", motifs=tset)
        assert r.count == o.count and np.array_equal(r.rows, o.rows)


# grid60/100: no seed among those tried had an oracle count finishing within the picker's time
# limit (the oracle's depth-first order explodes on those patterns), so that cell has no case
LARGE = [(lat, size) for lat in LATTICES for size in (80, 100) if f"{lat}/{size}" in SEEDS]


@pytest.mark.parametrize("lattice,size", LARGE)
def test_table2_counts_large_patterns(dm, lattice, size):
    """80- and 100-vertex patterns (beyond the round-1 cap of 64): counts against the oracle's
    counts stored by scripts/pick_table2_seeds.py (the oracle needs up to ~70 s per lattice here)."""
    gfn, tset = LATTICES[lattice]
    n, e = gfn()
    G = dm.Graph(n, e)
    for seed, want in SEEDS[f"{lattice}/{size}"]:
        k, pe, _ = g.random_connected_subgraph(n, e, size, seed)
        assert k == size
        for motifs in ("all", tset):
            assert G.match(k, pe, motifs=motifs).count == want, (lattice, size, seed, motifs)
