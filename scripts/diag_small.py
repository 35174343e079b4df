import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2508_21287_b200 as dm
for wl in ("c3-p20", "c2-er-c4"):
    desc, gfn, pfn, drop = bench.WORKLOADS[wl]
    n, e = gfn(); k, pe = pfn()
    G = dm.Graph(n, e, drop_self_loops=drop)
    s = torch.cuda.current_stream()
    for _ in range(5): G.match(k, pe, stream=s)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(50): r = G.match(k, pe, stream=s)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t) / 50 * 1e3
    r = G.match(k, pe, stream=s, profile=True)
    st = r.stats
    print(wl, f"wall/match {wall:.3f} ms, device kernels {sum(st['ms_count'])+sum(st['ms_write']):.3f} ms, total {st['ms_total']:.3f}, steps {st['num_steps']}")
    t = time.perf_counter()
    for _ in range(200): P = dm.Plan(k, pe, stats=G.stats())
    print("  plan build", (time.perf_counter() - t) / 200 * 1e3, "ms")
