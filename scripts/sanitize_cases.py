"""Small workloads for compute-sanitizer (scripts/sanitize.sh): configs 1-3, R-MAT-10 diamond /
K4, HH10 P16 count (repeated -> the pipelined sync-free path), table steps (M7 / heavy-hex motif
sets), the triangle-apex table and its 4-clique pair step, a chunked run, the exchange kernels.  Counts are checked against the oracle so a silent corruption fails loudly too."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import dm_inputs as g  # noqa: E402
import oracle  # noqa: E402
import paper_2508_21287_b200 as dm  # noqa: E402

cases = [(g.falcon27(), g.path(4), False, "table"), (g.grid_diag(24), g.ring(4), False, "table"),
         (g.er_gnm(2000, 16000, 1), g.clique(3), False, "table"), (g.ibm_heavy_hex(3), g.path(12), False, "table"),
         (g.rmat(10, 16, seed=1), g.diamond(), True, "count"), (g.rmat(10, 16, seed=1), g.clique(4), True, "count"),
         (g.ibm_heavy_hex(10), g.path(16), False, "count"), (g.ibm_heavy_hex(6), g.ring(12), False, "both")]
for (n, e), (k, pe), drop, out in cases:
    G = dm.Graph(n, e, drop_self_loops=drop)
    o = oracle.match(n, e, k, pe, drop_self_loops=drop, table=(out != "count"))
    for rep in range(3 if out == "count" else 1):
        r = G.match(k, pe, output=out)
        assert r.count == o.count, (n, k, r.count, o.count)
        if out != "count":
            assert np.array_equal(r.rows, o.rows)
    G.close()
# table steps (motif database, k_table single / count on 16-bit tiles) and the triangle-apex
# table with its 4-clique pair step
n, e = g.ibm_heavy_hex(10)
G = dm.Graph(n, e)
want = oracle.match(n, e, *g.path(20), table=False).count
for rep in range(3):
    assert G.match(*g.path(20), motifs="M2,M7").count == want
k, pe, _ = g.random_connected_subgraph(n, e, 16, 1)
o = oracle.match(n, e, k, pe)
assert np.array_equal(G.match(k, pe, output="table", motifs="heavy-hex").rows, o.rows)
nr, er = g.rmat(10, 16, seed=1)
R = dm.Graph(nr, er, drop_self_loops=True)
assert R.match(*g.clique(4), motifs="apex").count == oracle.match(nr, er, *g.clique(4), drop_self_loops=True,
                                                                  table=False).count
n, e = g.ibm_heavy_hex(6)
G = dm.Graph(n, e)
r = G.match(*g.path(10), output="table", mem_budget=1 << 15)
assert r.count == oracle.match(n, e, *g.path(10), table=False).count
rows = torch.randint(0, 1000, (3000, 8), dtype=torch.int32, device="cuda")
work = torch.randint(0, 100, (3000,), dtype=torch.int64, device="cuda")
dm.partition_by_work(rows, work, 10, int(work.sum()) + 20, 3)
dm.partition_by_key(rows, 0, [300, 600], 3)
dm.table_sort(rows, 1000)
torch.cuda.synchronize()
print("sanitize cases ok")
