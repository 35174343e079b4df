"""Multi-rank host logic on CPU (gloo, world_size 2): equal-work seed cuts, the count
all_reduce (C3) and the table gather + canonical merge (C4).  The per-rank matcher is the
oracle restricted to the rank's root range, so the test checks that the sharding partitions
the result exactly (SURVEY §8(e) invariant: 1/2/4/8-rank results are identical)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import dm_inputs as g
from paper_2508_21287_b200.dist import equal_work_cuts, match_sharded, merge_tables


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_equal_work_cuts():
    wp = np.cumsum([0] + [3] * 10)
    assert equal_work_cuts(wp, 1) == [0, 10]
    c = equal_work_cuts(wp, 2)
    assert c[0] == 0 and c[-1] == 10 and c == sorted(c)
    assert equal_work_cuts(np.array([0, 0, 0]), 4) == [0, 0, 0, 0, 2]
    wp = np.cumsum([0, 100, 1, 1, 1, 1])
    c = equal_work_cuts(wp, 3)
    assert c[0] == 0 and c[-1] == 5 and all(a <= b for a, b in zip(c, c[1:]))


def _worker(rank, world, port, out):
    import torch.distributed as tdist

    import oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, e = g.ibm_heavy_hex(3)
        k, pe = g.path(7)
        # oracle roots are its first pattern vertex (order[0]); work prefix = arcs per vertex
        deg = np.bincount(np.concatenate([e[:, 0], e[:, 1]]), minlength=n)
        wp = np.concatenate([[0], np.cumsum(deg)])

        def local(b, ee):
            r = oracle.match(n, e, k, pe, roots=(b, ee), threads=1)
            return r.count, r.rows

        cnt, rows = match_sharded(local, wp, k, rank=rank, world=world, table=True)
        full = oracle.match(n, e, k, pe, threads=1)
        out.put((rank, cnt == full.count, bool(np.array_equal(rows, full.rows))))
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_match_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(c and t for _, c, t in res), res


def test_merge_tables():
    a = np.array([[3, 1], [0, 2]], np.int32)
    b = np.array([[1, 5]], np.int32)
    m = merge_tables([a, b, np.zeros((0, 2), np.int32)], 2)
    assert m.tolist() == [[0, 2], [1, 5], [3, 1]]


def _rebalance_worker(rank, world, port, out):
    import torch
    import torch.distributed as tdist
    from paper_2508_21287_b200.dist import rebalance_rows
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(100 + rank)
        n = [37, 5, 0][rank % 3] if world == 3 else [40, 3][rank]
        rows = torch.randint(0, 1000, (n, 4), generator=g, dtype=torch.int32)
        rows[:, 0] = rank * 1000 + torch.arange(n, dtype=torch.int32)   # unique row ids
        work = torch.randint(1, 50, (n,), generator=g, dtype=torch.int64)
        got = rebalance_rows(rows, work, rank=rank, world=world)
        # gather everything (pickled) to check conservation and balance
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
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rebalance_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok1 and ok2 for _, ok1, ok2 in res), res
