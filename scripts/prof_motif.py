"""Run one workload with a motif set a few times (for ncu captures of the table-step kernels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2508_21287_b200 as dm  # noqa: E402

wl, motifs, reps = sys.argv[1], sys.argv[2], int(sys.argv[3])
desc, gfn, pfn, drop = bench.WORKLOADS[wl]
n, e = gfn()
k, pe = pfn()
G = dm.Graph(n, e, drop_self_loops=drop)
for _ in range(reps):
    r = G.match(k, pe, motifs=motifs)
torch.cuda.synchronize()
print(r.count)
