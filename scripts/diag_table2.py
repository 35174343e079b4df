"""Per-seed device time and level sizes of the Table 2 count cases (diagnostic)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dm_inputs as g  # noqa: E402
import paper_2508_21287_b200 as dm  # noqa: E402

S = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "table2_seeds.json")))["seeds"]
LAT = {"hex11x33": (lambda: g.hex_lattice_subdivided(11, 33), "heavy-hex"),
       "hex25x34": (lambda: g.hex_lattice_subdivided(25, 34), "heavy-hex"),
       "grid40": (lambda: g.grid(40), "grid"), "grid60": (lambda: g.grid(60), "grid")}
for lat in sys.argv[1].split(","):
    gfn, tset = LAT[lat]
    n, e = gfn()
    G = dm.Graph(n, e)
    for size in [int(x) for x in sys.argv[2].split(",")]:
        for seed, want in S.get(f"{lat}/{size}", []):
            k, pe, _ = g.random_connected_subgraph(n, e, size, seed)
            for motifs in ("all", tset):
                t = time.time()
                r = G.match(k, pe, motifs=motifs, profile=True, output="count" if size > 60 else "both")
                st = r.stats
                print(f"{lat}/{size} seed {seed} {motifs}: {time.time() - t:.2f}s count {r.count} want {want} "
                      f"steps {st['num_steps']} max level {max(st['rows_out']):.3g} chunks {st['num_chunks']}", flush=True)
