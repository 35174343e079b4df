import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2508_21287_b200 as dm
desc, gfn, pfn, drop = bench.WORKLOADS["c5"]
n, e = gfn(); k, pe = pfn()
G = dm.Graph(n, e)
s = torch.cuda.current_stream()
flush = torch.empty(int(300e6) // 4, dtype=torch.int32, device="cuda")
for prof in (False, True):
    for fl in (False, True):
        for _ in range(3): G.match(k, pe, stream=s, profile=prof)
        ts = []
        for _ in range(10):
            if fl: flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s); t0 = time.perf_counter()
            r = G.match(k, pe, stream=s, profile=prof, seed_range=(0, n))
            b.record(s); torch.cuda.synchronize(); t1 = time.perf_counter()
            ts.append((a.elapsed_time(b), (t1 - t0) * 1e3))
        print(f"profile={prof} flush={fl}: device ms {sum(x for x,_ in ts)/len(ts):.2f} wall ms {sum(y for _,y in ts)/len(ts):.2f}  stats_total {r.stats['ms_total']:.2f}")
