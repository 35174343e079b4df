"""GPU: the multi-rank path through the CUDA library against the CPU
oracle.  2 and 3 ranks are spawned on cuda:0 (one box has one GPU; NCCL refuses two ranks on
one device, so the collectives run over gloo on CPU copies -- the data path, i.e. every
partition, sort, prefix and join, is the library's).  Also: the step-level C ABI
(dm_plan_seed / dm_plan_step / dm_plan_finish_table) and the exchange kernels against plain
definitions."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import dm_inputs as g
import oracle

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CASES = {
    "hh10-p16-table": (lambda: g.ibm_heavy_hex(10), lambda: g.path(16), False, "table"),
    "hh10-c12-table": (lambda: g.ibm_heavy_hex(10), lambda: g.ring(12), False, "table"),
    "gd64-c4-table": (lambda: g.grid_diag(64), lambda: g.ring(4), False, "table"),
    "rmat12-diamond": (lambda: g.rmat(12, 16, seed=1), g.diamond, True, "count"),
    "rmat12-k4": (lambda: g.rmat(12, 16, seed=1), lambda: g.clique(4), True, "count"),
}


def _worker(rank, world, port, out, names):
    import torch
    import torch.distributed as tdist

    import paper_2508_21287_b200 as dm
    from paper_2508_21287_b200.dist import match_rebalanced, match_sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    cpu = torch.device("cpu")
    res = []
    try:
        for name in names:
            gfn, pfn, drop, output = CASES[name]
            n, e = gfn()
            k, pe = pfn()
            G = dm.Graph(n, e, drop_self_loops=drop, device=0)
            o = oracle.match(n, e, k, pe, drop_self_loops=drop, table=(output == "table"))
            cnt, tab = match_sharded(G, k, pe, rank=rank, world=world, output="both" if output == "table" else "count",
                                     coll_device=cpu)
            ok = cnt == o.count
            if output == "table":
                ok &= tab is not None and np.array_equal(tab, o.rows)
            nsteps = G.plan(k, pe).num_steps
            for step in range(1, nsteps):
                rc, mine = match_rebalanced(G, k, pe, rank=rank, world=world, step=step, coll_device=cpu)
                ok &= rc == o.count
            res.append((name, bool(ok), int(cnt), int(o.count)))
            G.close()
        out.put((rank, res))
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_multi_rank_vs_oracle(world):
    """match_sharded (C3 count, C4 range-partitioned table) and match_rebalanced at every level
    (C1 + C2 exchange by the library's work partition, then dm_match_resume) on 2-3 ranks equal
    the oracle element by element."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    names = list(CASES)
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, names)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=900) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, res in got:
        for name, ok, cnt, want in res:
            assert ok, (rank, name, cnt, want)


# ------------------------------------------------------------------ step-level C ABI
@pytest.mark.parametrize("case", ["hh6-p11", "rmat10-diamond", "gd20-c5", "er-k4", "hh10-p20-count"])
def test_plan_steps_chain_vs_oracle(dm, case):
    """dm_plan_seed -> dm_plan_step ... -> dm_plan_finish_table (or the count-only last step)
    reproduces the oracle's table / count; the plan equals the one dm_match runs."""
    import torch
    (n, e), (k, pe), drop, table = {
        "hh6-p11": (g.ibm_heavy_hex(6), g.path(11), False, True),
        "rmat10-diamond": (g.rmat(10, 16, seed=3), g.diamond(), True, True),
        "gd20-c5": (g.grid_diag(20), g.ring(5), False, True),
        "er-k4": (g.er_gnm(300, 2000, 4), g.clique(4), False, True),
        "hh10-p20-count": (g.ibm_heavy_hex(10), g.path(20), False, False),
    }[case]
    G = dm.Graph(n, e, drop_self_loops=drop)
    o = oracle.match(n, e, k, pe, drop_self_loops=drop, table=table)
    plan = G.plan(k, pe, output="table" if table else "count")
    ns = plan.num_steps
    assert ns == G.match(k, pe, output="table" if table else "count").stats["num_steps"]
    fr = plan.seed(G)
    assert fr.width == plan.width(1) and fr.stride == plan.stride(1)
    for step in range(1, ns):
        rows = fr.rows_tensor()
        if step == ns - 1 and not table:
            assert plan.step(G, step, rows, materialize=False) == o.count
            return
        nxt = plan.step(G, step, rows)
        assert nxt.width == plan.width(step + 1)
        fr = nxt
    if not table:  # single-step plan
        assert fr.rows == o.count
        return
    assert fr.rows == o.count and fr.work_tensor() is None
    canon = plan.finish_table(G, fr.rows_tensor()[:, :].contiguous())
    assert np.array_equal(canon.cpu().numpy(), o.rows)
    r = plan.run(G, output="table")
    assert np.array_equal(r.rows, o.rows)
    # cuts: an equal-work partition of [0, n)
    cuts = plan.seed_cuts(G, 4)
    assert cuts[0] == 0 and cuts[-1] == n and cuts == sorted(cuts)
    wp = plan.seed_work(G)
    assert wp.shape == (n + 1,) and wp[0] == 0 and np.all(np.diff(wp.astype(np.int64)) >= 1)


def test_partition_and_sort_kernels(dm):
    """dm_rows_partition_by_work / _by_key / dm_table_sort against their plain definitions
    (stable grouping by destination; lexicographic order = np.lexsort)."""
    import torch
    rng = np.random.default_rng(5)
    for n, stride, parts in [(0, 4, 3), (1, 4, 2), (1000, 8, 3), (70_000, 4, 7), (5000, 28, 8)]:
        rows = torch.as_tensor(rng.integers(0, 1 << 20, (n, stride)).astype(np.int32)).cuda()
        work = torch.as_tensor(rng.integers(0, 1 << 40, n).astype(np.int64)).cuda()
        tot_local = int(work.sum().item()) if n else 0
        base = int(rng.integers(0, 1 << 41))
        total = base + tot_local + int(rng.integers(0, 1 << 41))
        packed, counts = dm.partition_by_work(rows, work, base, total, parts)
        w = work.cpu().numpy().astype(object)
        excl = np.concatenate([[0], np.cumsum(w)[:-1]]) if n else np.zeros(0, object)
        dest = np.array([min(parts - 1, ((base + int(x)) * parts) // total) for x in excl], np.int64)
        order = np.argsort(dest, kind="stable")
        assert counts == [int((dest == r).sum()) for r in range(parts)]
        assert np.array_equal(packed.cpu().numpy(), rows.cpu().numpy()[order])
        spl = sorted(rng.integers(0, 1 << 20, parts - 1).tolist())
        packed, counts = dm.partition_by_key(rows, 1 % stride, spl, parts)
        dest = np.searchsorted(np.asarray(spl), rows.cpu().numpy()[:, 1 % stride], side="right")
        order = np.argsort(dest, kind="stable")
        assert counts == [int((dest == r).sum()) for r in range(parts)]
        assert np.array_equal(packed.cpu().numpy(), rows.cpu().numpy()[order])
        t = torch.as_tensor(rng.integers(0, 50, (n, 5)).astype(np.int32)).cuda()
        want = t.cpu().numpy()
        want = want[np.lexsort(want.T[::-1])] if n else want
        dm.table_sort(t, 50)
        assert np.array_equal(t.cpu().numpy(), want)
