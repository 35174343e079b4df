"""Copy the judged evidence of one GPU call from gpurun_out/ into profiles/ (tracked):
bench lines, the ncu launch list summary (per kernel kind) and key metrics of the full capture.
usage: python scripts/collect_profiles.py <tag>   (e.g. r01)"""
import csv, glob, json, os, subprocess, sys
tag = sys.argv[1]
os.makedirs("profiles", exist_ok=True)
for f in glob.glob("gpurun_out/bench_*.json"):
    lines = [l for l in open(f).read().splitlines() if l.startswith("{")]
    if lines:
        name = os.path.basename(f)[len("bench_"):]
        open(f"profiles/{tag}_bench_{name}", "w").write(lines[-1] + "\n")
out = [f"# {tag} ncu summaries\n"]
for f in sorted(glob.glob("gpurun_out/launches_*.csv")):
    wl = os.path.basename(f)[len("launches_"):-4]
    open(f"profiles/{tag}_launches_{wl}.csv", "w").write(open(f).read())  # the raw launch list
    r = subprocess.run([sys.executable, "scripts/ncu_traffic.py", f, wl], capture_output=True, text=True)
    out += [f"## launch list {wl} (ncu --metrics gpu__time_duration.sum,dram__bytes_*; one dm_match)", "```", r.stdout.strip(), "```", ""]
want = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "No Eligible", "Achieved Occupancy", "Theoretical Occupancy", "Avg. Active Threads Per Warp",
        "Executed Instructions", "Registers Per Thread", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Dynamic Shared Memory Per Block", "Grid Size"]
for f in sorted(glob.glob("gpurun_out/*.ncu-rep")):
    r = subprocess.run(["ncu", "-i", f, "--page", "details", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(r.stdout.splitlines()))
    if not rows:
        continue
    h = rows[0]
    out += [f"## ncu --set full: {os.path.basename(f)}", "```"]
    for row in rows[1:]:
        d = dict(zip(h, row))
        if d.get("Metric Name") in want:
            out.append(f"{d['ID']:>2} {d['Kernel Name'][:48]:48s} {d['Metric Name']:32s} {d['Metric Value']} {d['Metric Unit']}")
    r = subprocess.run(["ncu", "-i", f, "--page", "raw", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(r.stdout.splitlines()))
    if len(rows) > 2:
        h, units = rows[0], dict(zip(rows[0], rows[1]))  # second row: the unit of every column
        for row in rows[2:]:
            d = dict(zip(h, row))
            try:
                rd = float(d["dram__bytes_read.sum"].replace(",", ""))
                wr = float(d["dram__bytes_write.sum"].replace(",", ""))
            except Exception:
                continue
            ur, uw = units.get("dram__bytes_read.sum", "?"), units.get("dram__bytes_write.sum", "?")
            out.append(f"{d['ID']:>2} {d['Kernel Name'][:48]:48s} dram read {rd:.4g} {ur}, write {wr:.4g} {uw}")
    out += ["```", ""]
for f in sorted(glob.glob("gpurun_out/steps_*.txt")):
    out += [f"## per-step statistics ({os.path.basename(f)})", "```", open(f).read().strip(), "```", ""]
open(f"profiles/{tag}_ncu_summary.md", "w").write("\n".join(out) + "\n")
print("\n".join(out)[:3000])
