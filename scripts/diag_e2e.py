"""Where the end-to-end time of config 5 goes (graph build, motif database, first query)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import dm_inputs as g  # noqa: E402
import paper_2508_21287_b200 as dm  # noqa: E402

n, e = g.ibm_heavy_hex(31)
k, pe = g.path(30)
pin = torch.from_numpy(np.ascontiguousarray(e)).pin_memory().numpy()
s = torch.cuda.current_stream()
for it in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    G = dm.Graph(n, pin)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    G.build_motifs("M2,M7", stream=s)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    r = G.match(k, pe, motifs="M2,M7", stream=s)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    r2 = G.match(k, pe, motifs="M2,M7", stream=s)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    G.close()
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    print(f"graph {1e3*(t1-t0):.2f} ms  motif db {1e3*(t2-t1):.2f} ms  first match {1e3*(t3-t2):.2f} ms  "
          f"repeat {1e3*(t4-t3):.2f} ms  close {1e3*(t5-t4):.2f} ms  count {r.count}", flush=True)
# the bench's e2e loop shape: create + lazy motif build inside the first match + close
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    G = dm.Graph(n, pin)
    r = G.match(k, pe, motifs="M2,M7", stream=s)
    G.close()
    torch.cuda.synchronize()
    print(f"e2e step {1e3*(time.perf_counter()-t0):.2f} ms", flush=True)
