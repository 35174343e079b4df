import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench, paper_2508_21287_b200 as dm
desc, gfn, pfn, drop = bench.WORKLOADS["c3-p20"]
n, e = gfn(); k, pe = pfn()
G = dm.Graph(n, e)
s = torch.cuda.current_stream()
for _ in range(5): G.match(k, pe, stream=s)
torch.cuda.synchronize()
print("---- traced", file=sys.stderr, flush=True)
G.match(k, pe, stream=s)
