"""Hottest CUDA source lines of an ncu report (instructions executed, stall samples)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.split("\n")
cur, rows, i = None, [], 0
while i < len(out):
    l = out[i]
    if l.startswith('"File Path"'):
        cur = l.split(",")[1].strip('"').split("/")[-1]
    elif l.startswith('"Line No"'):
        hdr = next(csv.reader([l]))
        i += 1
        while i < len(out) and out[i] and not out[i].startswith('"File Path"') and not out[i].startswith('"Function Name"'):
            r = next(csv.reader([out[i]]))
            if len(r) == len(hdr):
                rows.append((cur, dict(zip(hdr, r))))
            i += 1
        continue
    i += 1


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


tot = sum(num(d.get("Instructions Executed", 0)) for _, d in rows)
print(f"total warp instructions {tot:.3e}")
rows.sort(key=lambda x: -num(x[1].get("Instructions Executed", 0)))
for f, d in rows[:top]:
    print(f"{f}:{d['Line No']:>5} {num(d.get('Instructions Executed', 0)) / max(tot, 1):6.1%} "
          f"samples {int(num(d.get('Warp Stall Sampling (All Samples)', 0))):>7}  {d['Source'].strip()[:100]}")
