"""Per-motif-set timing of one workload (device ms per dm_match, per-step kernel ms, table build)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2508_21287_b200 as dm  # noqa: E402

wl, motifs = sys.argv[1], sys.argv[2]
desc, gfn, pfn, drop = bench.WORKLOADS[wl]
n, e = gfn()
k, pe = pfn()
G = dm.Graph(n, e, drop_self_loops=drop)
t0 = time.perf_counter()
info = G.build_motifs(motifs) if motifs not in ("all",) else {}
build_s = time.perf_counter() - t0
plan = G.plan(k, pe, motifs=motifs)
s = torch.cuda.current_stream()
for _ in range(3):
    r = G.match(k, pe, motifs=motifs, stream=s)
ts = []
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    r = G.match(k, pe, motifs=motifs, stream=s, profile=True)
    b.record(s)
    b.synchronize()
    ts.append(a.elapsed_time(b))
st = r.stats
steps = [(x.get("table") or len(x.get("new", []))) for x in plan.describe()["steps"]]
print(f"{wl} motifs={motifs} count={r.count} ms={min(ts):.3f} med={sorted(ts)[5]:.3f} build_s={build_s:.2f} "
      f"tables={info} steps={steps} pipelined={st['pipelined']}")
print("   per-step ms:", [round(a + b, 3) for a, b in zip(st["ms_count"], st["ms_write"])])
print("   rows_out:", st["rows_out"])
print("   cand:", st["candidates"])
