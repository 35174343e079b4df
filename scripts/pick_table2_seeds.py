"""Pick the Table 2 test seeds (tests/test_gpu_table2.py): random connected subgraphs of the
paper's lattices whose embedding count keeps the CPU oracle within seconds.  Many
random-walk subgraphs of lattices are trees with 1e7-1e8 labelled embeddings (the oracle needs
minutes for those), so seeds are screened with a root-sampled oracle estimate and then counted
exactly; an exact count that does not finish within TIMEOUT seconds drops the seed.  Calls only
oracle/ and dm_inputs; writes tests/golden/table2_seeds.json.  Usage: pick_table2_seeds.py
[lattice ...] [--sizes 20,40,...] [--timeout S] (default: all lattices and sizes, 90 s; results of
other lattices / sizes already in the file are kept)."""
import json
import multiprocessing as mp
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dm_inputs as g  # noqa: E402
import oracle  # noqa: E402

LATTICES = {"hex11x33": lambda: g.hex_lattice_subdivided(11, 33), "hex25x34": lambda: g.hex_lattice_subdivided(25, 34),
            "grid40": lambda: g.grid(40), "grid60": lambda: g.grid(60)}
LIMIT = {20: 2_000_000, 40: 2_000_000, 60: 2_000_000, 80: 20_000_000, 100: 20_000_000}
TIMEOUT = 90
PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden", "table2_seeds.json")


def _count(args, q):
    n, e, k, pe = args
    q.put(oracle.match(n, e, k, pe, table=False).count)


def exact_count(n, e, k, pe):
    q = mp.Queue()
    pr = mp.Process(target=_count, args=((n, e, k, pe), q))
    pr.start()
    pr.join(TIMEOUT)
    if pr.is_alive():
        pr.kill()
        pr.join()
        return None
    return q.get()


args = sys.argv[1:]
sizes = list(LIMIT)
if "--sizes" in args:
    i = args.index("--sizes")
    sizes = [int(x) for x in args[i + 1].split(",")]
    del args[i:i + 2]
if "--timeout" in args:
    i = args.index("--timeout")
    TIMEOUT = int(args[i + 1])
    del args[i:i + 2]
out = json.load(open(PATH))["seeds"] if os.path.exists(PATH) else {}
todo = args or list(LATTICES)
for name, fn in LATTICES.items():
    if name not in todo:
        continue
    n, e = fn()
    for size, lim in LIMIT.items():
        if size not in sizes:
            continue
        picked = []
        seed = 0
        while len(picked) < (5 if size <= 60 else 3) and seed < 120:
            seed += 1
            k, pe, _ = g.random_connected_subgraph(n, e, size, seed)
            R = max(1, n // 200)
            est = oracle.match(n, e, k, pe, table=False, roots=(0, R)).count * (n / R)
            if est > 3 * lim:
                continue
            c = exact_count(n, e, k, pe)
            if c is not None and c <= lim:
                picked.append([seed, int(c)])
        out[f"{name}/{size}"] = picked
        print(name, size, picked, flush=True)
        json.dump({"source": "scripts/pick_table2_seeds.py (oracle counts; P:437-443 workload shape)", "seeds": out},
                  open(PATH, "w"), indent=1)
