"""Multi-rank collective sequencing on CPU (gloo, world_size 2 and 3): the frontier rebalance
(C1 all_gather of work totals + C2 all_to_all of rows), the count all_reduce (C3) and the range
partition + exchange + sort of the canonical table (C4) of paper_2508_21287_b200.dist.

dist.py takes its device operations (the library's partition / sort kernels) as parameters; here
they are replaced by plain CPU definitions written in this file, so the test checks the
collective plumbing and the SURVEY §8(e) invariants (rows conserved, every rank ~1/world of the
work, sharded results identical to the unsharded oracle).  The same functions run with the
library kernels on the GPU in tests/test_gpu_dist.py."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import dm_inputs as g


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


# ---- CPU definitions of the library's device operations (test-side reference) -------------
def cpu_partition_by_work(rows, work, base, total, parts, stream=None):
    import torch
    n = int(rows.shape[0])
    if n == 0:
        return rows.clone(), [0] * parts
    excl = torch.cumsum(work, 0) - work
    dest = [min(parts - 1, ((base + int(e)) * parts) // total) if total else 0 for e in excl.tolist()]
    order = sorted(range(n), key=lambda i: dest[i])          # stable
    counts = [dest.count(r) for r in range(parts)]
    return rows[order].contiguous(), counts


def cpu_partition_by_key(rows, col, splitters, parts, stream=None):
    n = int(rows.shape[0])
    if n == 0:
        return rows.clone(), [0] * parts
    dest = [int(np.searchsorted(np.asarray(splitters, np.int64), int(v), side="right"))
            for v in rows[:, col].tolist()]
    order = sorted(range(n), key=lambda i: dest[i])
    return rows[order].contiguous(), [dest.count(r) for r in range(parts)]


def cpu_sort(rows, n_vertices, stream=None):
    import torch
    a = rows.numpy()
    if a.shape[0] == 0:
        return rows
    return torch.from_numpy(np.ascontiguousarray(a[np.lexsort(a.T[::-1])]))


def _spawn(target, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q, *args)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def _init(rank, world, port):
    import torch.distributed as tdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    return tdist


def _table_worker(rank, world, port, out):
    import torch

    import oracle
    from paper_2508_21287_b200.dist import gather_table, reduce_count, shard_table
    tdist = _init(rank, world, port)
    try:
        ok = True
        for (n, e), (k, pe) in [(g.ibm_heavy_hex(3), g.path(7)), (g.grid_diag(12), g.ring(4)),
                                (g.er_gnm(40, 160, 3), g.clique(3))]:
            full = oracle.match(n, e, k, pe, threads=1)
            # oracle roots are its first pattern vertex; any cut of [0, n) partitions the result
            cuts = [0] + [n * r // world for r in range(1, world)] + [n]
            part = oracle.match(n, e, k, pe, roots=(cuts[rank], cuts[rank + 1]), threads=1)
            total = reduce_count(part.count)                                     # C3
            # a rank's table in canonical order, then C4 with the splitters cuts[1..world-1]
            mine = shard_table(torch.from_numpy(part.rows), cuts, n, rank=rank, world=world,
                               partition=cpu_partition_by_key, sort=cpu_sort)
            col0 = mine[:, 0].numpy()
            ok &= bool(np.all((col0 >= cuts[rank]) & (col0 < cuts[rank + 1])))
            got = gather_table(mine)
            ok &= total == full.count and bool(np.array_equal(got, full.rows))
        out.put((rank, ok))
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_table_gloo(world):
    """Seed shards (roots) -> C3 count + C4 range partition / exchange / sort: the rank-order
    concatenation equals the unsharded canonical table."""
    res = _spawn(_table_worker, world)
    assert all(ok for _, ok in res), res


def _rebalance_worker(rank, world, port, out):
    import torch

    from paper_2508_21287_b200.dist import rebalance_rows
    tdist = _init(rank, world, port)
    try:
        gen = torch.Generator().manual_seed(100 + rank)
        n = [37, 5, 0][rank % 3] if world == 3 else [40, 3][rank]
        rows = torch.randint(0, 1000, (n, 4), generator=gen, dtype=torch.int32)
        rows[:, 0] = rank * 1000 + torch.arange(n, dtype=torch.int32)   # unique row ids
        work = torch.randint(1, 50, (n,), generator=gen, dtype=torch.int64)
        got = rebalance_rows(rows, work, int(work.sum()), rank=rank, world=world,
                             partition=cpu_partition_by_work)
        everything = [None] * world
        tdist.all_gather_object(everything, (rows.tolist(), work.tolist(), got.tolist()))
        idmap, before, after = {}, [], []
        for rr, ww, gg in everything:
            for row, wk in zip(rr, ww):
                idmap[row[0]] = wk
            before += [tuple(r) for r in rr]
            after += [tuple(r) for r in gg]
        before.sort()
        after.sort()
        total = sum(idmap.values())
        mywork = sum(idmap[r[0]] for r in got.tolist())
        maxw = max(idmap.values()) if idmap else 0
        out.put((rank, before == after, abs(mywork - total / world) <= maxw + 1))
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_rebalance_rows_gloo(world):
    """C1 + C2: rows are conserved and every rank ends with ~1/world of the total work."""
    res = _spawn(_rebalance_worker, world)
    assert all(ok1 and ok2 for _, ok1, ok2 in res), res


def test_cpu_reference_partitions():
    """The test-side partition definitions themselves (stable grouping, counts)."""
    import torch
    rows = torch.tensor([[5, 0], [1, 1], [9, 2], [3, 3]], dtype=torch.int32)
    p, c = cpu_partition_by_key(rows, 0, [4], 2)
    assert c == [2, 2] and p[:, 1].tolist() == [1, 3, 0, 2]
    w = torch.tensor([1, 1, 1, 1], dtype=torch.int64)
    p, c = cpu_partition_by_work(rows, w, 0, 4, 2)
    assert c == [2, 2] and p[:, 1].tolist() == [0, 1, 2, 3]
