"""Summarise an ncu --metrics launch list (csv) per kernel kind: time share and DRAM bytes
per launch; writes profiles/traffic.json[workload][kind] for bench.py's roofline.traffic."""
import csv, json, os, re, sys, collections
path, workload = sys.argv[1], sys.argv[2]
rows = [r for r in csv.reader(open(path)) if r]
h = next(r for r in rows if "Kernel Name" in r)
data = [dict(zip(h, r)) for r in rows[rows.index(h) + 1:] if len(r) == len(h)]
per = collections.defaultdict(lambda: collections.defaultdict(float))
for d in data:
    k = d["Kernel Name"]
    per[(d["ID"], k)][d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
kinds = collections.defaultdict(lambda: [0, 0.0, 0.0])
tot_t = 0.0
for (i, k), m in per.items():
    t = m.get("gpu__time_duration.sum", 0.0)
    tot_t += t
    mk = re.search(r"k_(?:rows|step|table)<(\d)", k)
    if "k_pairs" in k or "k_deep" in k:
        kind = "join_count"
    elif mk:
        kind = {"0": "join_count", "1": "join_rerun", "2": "join_single"}[mk.group(1)]
    else:
        kind = "other:" + k.split("(")[0][-40:]
    kinds[kind][0] += 1
    kinds[kind][1] += t
    kinds[kind][2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
out = {}
for kind, (n, t, b) in sorted(kinds.items(), key=lambda kv: -kv[1][1]):
    print(f"{kind:28s} launches {n:4d} time {t/1e6:9.3f} ms share {t/tot_t*100:5.1f}%  dram/launch {b/max(n,1)/1e9:8.3f} GB")
    out[kind] = {"launches": n, "share": t / tot_t, "bytes_per_launch": b / max(n, 1),
                 "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum ({os.path.basename(path)})"}
tp = "profiles/traffic.json"
allv = json.load(open(tp)) if os.path.exists(tp) else {}
allv[workload] = out
json.dump(allv, open(tp, "w"), indent=1)
