"""Run one workload a few times and print per-step stats (rows, candidates, ms per pass)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2508_21287_b200 as dm

wl = sys.argv[1] if len(sys.argv) > 1 else "c5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
motifs = sys.argv[3] if len(sys.argv) > 3 else bench.MOTIFS.get(wl, "all")
desc, gfn, pfn, drop = bench.WORKLOADS[wl]
n, e = gfn(); k, pe = pfn()
G = dm.Graph(n, e, drop_self_loops=drop)
if motifs != "all":
    G.build_motifs(motifs)
s = torch.cuda.current_stream()
for i in range(reps):
    t = time.perf_counter()
    r = G.match(k, pe, stream=s, profile=True, motifs=motifs)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t) * 1e3
st = r.stats
print(f"{desc} motifs={motifs}: count={r.count} wall={wall:.2f}ms device_total={st['ms_total']:.2f}ms other={st['ms_other']:.2f}ms launches={st['num_launches']} chunks={st['num_chunks']}")
for i in range(st["num_steps"]):
    print(f"step {i:2d} w {st['width_in'][i]:2d}->{st['width_out'][i]:2d} rows {st['rows_in'][i]:>11d} -> {st['rows_out'][i]:>11d} "
          f"cand {st['candidates'][i]:>11d} probes {st['probes'][i]:>10d} count {st['ms_count'][i]:7.3f}ms write {st['ms_write'][i]:7.3f}ms "
          f"model {st['bytes_model'][i]/1e9:7.3f}GB")
