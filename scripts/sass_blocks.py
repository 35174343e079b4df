"""Group the SASS of one kernel in an ncu report (--page source --print-source sass csv export)
into straight-line blocks by execution count; print the heaviest blocks with their opcode mix."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 22
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h) and r[0] != "Address"]


def n(x):
    try:
        return int(x)
    except ValueError:
        return 0


blocks = []
for i, d in enumerate(data):
    ex = n(d["Instructions Executed"])
    toks = d["Source"].strip().split()
    op = (toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else ""))
    if blocks and blocks[-1][1] == ex:
        blocks[-1][2] += 1
        blocks[-1][4].append(op)
    else:
        blocks.append([i, ex, 1, d["Avg. Threads Executed"], [op]])
tot = sum(b[1] * b[2] for b in blocks)
print("total warp instructions", tot)
for b in sorted(blocks, key=lambda b: -b[1] * b[2])[:top_n]:
    ops = {}
    for o in b[4]:
        ops[o] = ops.get(o, 0) + 1
    top = sorted(ops.items(), key=lambda x: -x[1])[:7]
    print(f"@{b[0]:5d} exec {b[1]:>10d} x{b[2]:3d} = {100 * b[1] * b[2] / tot:5.1f}%  thr {b[3]:>5s}  {top}")
