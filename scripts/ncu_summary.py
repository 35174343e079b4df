"""Print the key ncu --set full metrics of every kernel in a report, plus the hottest source lines."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.DictReader(io.StringIO(out)))
want = {"Duration", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Executed Ipc Active", "Issue Slots Busy", "Warp Cycles Per Issued Instruction",
        "Avg. Active Threads Per Warp", "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Eligible Warps Per Scheduler", "L1/TEX Hit Rate", "L2 Hit Rate", "Grid Size", "Mem Busy", "Max Bandwidth"}
seen = {}
for r in rows:
    kid = r["ID"]
    if r["Metric Name"] in want:
        seen.setdefault(kid, [r["Kernel Name"][:60]]).append(f'{r["Metric Name"]}={r["Metric Value"]}{r["Metric Unit"]}')
for kid, v in seen.items():
    print(kid, v[0])
    print("   " + "; ".join(v[1:]))
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
if len(rr) > 2:
    hdr = rr[0]
    for row in rr[2:]:
        d = dict(zip(hdr, row))
        stalls = {k: d[k] for k in hdr if k.startswith("smsp__average_warp_latency_issue_stalled") or
                  (k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"))}
        top = sorted(((float(v.replace(",", "")) if v.replace(",", "").replace(".", "").isdigit() else 0.0, k)
                      for k, v in stalls.items()), reverse=True)[:8]
        print("   stalls:", ", ".join(f"{k.split('stalled_')[-1]}={v:g}" for v, k in top))
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum", "gpu__time_duration.sum"):
            if k in d:
                print(f"   {k} = {d[k]}")
