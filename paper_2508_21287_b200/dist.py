"""Multi-GPU driver: one process per GPU (torch.distributed over NCCL; gloo for the CPU tests).

Sharding: the data graph (Res(M2)) is replicated on every rank and the
partial-embedding frontier is row-sharded -- every row is an independent candidate (§4.1),
so any row partition of a level is valid and the results of the parts are disjoint.

  * seed sharding: rank r expands the seed vertices [cuts[r], cuts[r+1]) of the plan's first
    vertex, cut by equal estimated work (dm_plan_seed_cuts);
  * frontier rebalance (C1 + C2): a level materialized with dm_match_prefix is re-cut by its
    position in the GLOBAL work order (dm_rows_partition_by_work) and exchanged with one
    all_to_all_single; each rank finishes its rows with dm_match_resume;
  * count (C3): all_reduce(SUM) of the uint64 count;
  * table (C4): every rank's canonical table is range-partitioned by its first column
    (dm_rows_partition_by_key with the seed cuts as splitters), exchanged with all_to_all_single
    and sorted on the device (dm_table_sort): rank r then holds the rows whose first column lies
    in [cuts[r], cuts[r+1]) in canonical order, and the concatenation in rank order is the
    canonical table.

This module only sequences collectives and library calls; the partitions, sorts and work
prefixes are computed inside libdeltamotif.  The device operations are parameters so the
collective sequencing can be tested on CPU with gloo (tests/test_dist_gloo.py) while the GPU tests
run the library ones (tests/test_gpu_dist.py).
"""
from __future__ import annotations

from typing import Callable


def _to(t, dev):
    return t if dev is None or t.device == dev else t.to(dev)


def _all_gather_int(x: int, coll_device):
    import torch
    import torch.distributed as tdist
    world = tdist.get_world_size()
    t = torch.tensor([int(x)], dtype=torch.int64, device=coll_device)
    out = [torch.zeros(1, dtype=torch.int64, device=coll_device) for _ in range(world)]
    tdist.all_gather(out, t)
    return [int(o.item()) for o in out]


def exchange_rows(packed, send_counts, *, coll_device=None):
    """all_to_all of the per-destination row counts, then all_to_all_single of the rows
    (C2 / C4 payload).  packed: [n, stride] rows grouped by destination (send_counts[r] rows for
    rank r).  Returns the received rows on packed's device, grouped by source rank."""
    import torch
    import torch.distributed as tdist
    dev = packed.device
    send = torch.tensor(send_counts, dtype=torch.int64, device=coll_device)
    recv = torch.empty_like(send)
    tdist.all_to_all_single(recv, send)
    recv_l = [int(x) for x in recv.tolist()]
    src = _to(packed, coll_device).contiguous()
    out = torch.empty((sum(recv_l), int(packed.shape[1])), dtype=packed.dtype, device=src.device)
    tdist.all_to_all_single(out, src, output_split_sizes=recv_l, input_split_sizes=list(send_counts))
    return _to(out, dev)


def rebalance_rows(rows, work, work_total: int, *, rank: int, world: int, coll_device=None,
                   partition: Callable | None = None, stream=None):
    """Frontier rebalancing (C1 + C2): all_gather of the per-rank work totals, the library packs
    this rank's rows by their position in the global work order, one all_to_all exchanges them.
    Returns this rank's rows (a contiguous ~1/world share of the total work)."""
    if partition is None:
        from . import partition_by_work as partition
    tots = _all_gather_int(work_total, coll_device)                       # C1
    packed, send = partition(rows, work, sum(tots[:rank]), sum(tots), world, stream=stream)
    return exchange_rows(packed, send, coll_device=coll_device)           # C2


def reduce_count(count: int, *, coll_device=None) -> int:
    """C3: all_reduce(SUM) of the per-rank count."""
    import torch
    import torch.distributed as tdist
    t = torch.tensor([int(count)], dtype=torch.int64, device=coll_device)
    tdist.all_reduce(t, op=tdist.ReduceOp.SUM)
    return int(t.item())


def shard_table(rows, cuts, n_vertices: int, *, rank: int, world: int, coll_device=None,
                partition: Callable | None = None, sort: Callable | None = None, stream=None):
    """C4: range-partition a per-rank canonical table [n, k] (CUDA int32) by its first column at
    the splitters cuts[1..world-1], exchange, sort the received runs.  Returns this rank's rows
    (first column in [cuts[rank], cuts[rank+1])) in canonical order."""
    if partition is None:
        from . import partition_by_key as partition
    if sort is None:
        from . import table_sort as sort
    packed, send = partition(rows, 0, list(cuts[1:world]), world, stream=stream)
    mine = exchange_rows(packed, send, coll_device=coll_device)
    return sort(mine, n_vertices, stream=stream)


def gather_table(rows, *, coll_device=None):
    """Concatenate the per-rank range tables in rank order (every rank receives the whole
    canonical table; for tests / small results)."""
    import torch
    import torch.distributed as tdist
    sizes = _all_gather_int(int(rows.shape[0]), coll_device)
    k = int(rows.shape[1])
    mx = max(sizes) if sizes else 0
    local = torch.zeros((mx, k), dtype=torch.int32, device=coll_device)
    if rows.shape[0]:
        local[: rows.shape[0]] = _to(rows, coll_device)
    bufs = [torch.zeros((mx, k), dtype=torch.int32, device=coll_device) for _ in sizes]
    tdist.all_gather(bufs, local)
    return torch.cat([b[:s] for b, s in zip(bufs, sizes)]).cpu().numpy()


def match_sharded(graph, k: int, p_edges, *, rank: int, world: int, output: str = "count",
                  mode: str = "mono", motifs="all", stream=None, coll_device=None,
                  gather: bool = True):
    """Seed-sharded dm_match on this rank + C3 (count) / C4 (table).  Returns (count, table):
    table = the whole canonical table (gather=True, numpy) or this rank's range (CUDA tensor)."""
    import torch
    from . import Plan
    plan = Plan.for_graph(graph, k, p_edges, mode=mode, output="table" if output != "count" else "count",
                          motifs=motifs)
    cuts = plan.seed_cuts(graph, world)
    r = graph.match(k, p_edges, mode=mode, output=output, motifs=motifs,
                    seed_range=(cuts[rank], cuts[rank + 1]), stream=stream)
    total = reduce_count(r.count, coll_device=coll_device)
    if output == "count":
        return total, None
    dev = torch.device("cuda", graph.device)
    local = torch.as_tensor(r.rows).to(dev) if r.rows is not None and r.rows.size else \
        torch.zeros((0, k), dtype=torch.int32, device=dev)
    mine = shard_table(local, cuts, graph.n, rank=rank, world=world, coll_device=coll_device,
                       stream=stream)
    return total, (gather_table(mine, coll_device=coll_device) if gather else mine)


def match_rebalanced(graph, k: int, p_edges, *, rank: int, world: int, step: int, stream=None,
                     mode: str = "mono", motifs="all", coll_device=None, reduce: bool = True):
    """Count mode with a frontier exchange: level `step` of this rank's seed shard
    (dm_match_prefix), rebalanced by work across ranks (C1 + C2), finished locally
    (dm_match_resume), count all_reduced (C3).  Returns (count, rows this rank finished)."""
    from . import Plan
    plan = Plan.for_graph(graph, k, p_edges, mode=mode, output="count", motifs=motifs)
    cuts = plan.seed_cuts(graph, world)
    fr = graph.match_prefix(k, p_edges, step, mode=mode, motifs=motifs,
                            seed_range=(cuts[rank], cuts[rank + 1]), stream=stream)
    mine = rebalance_rows(fr.rows_tensor(), fr.work_tensor(), fr.work_total, rank=rank, world=world,
                          coll_device=coll_device, stream=stream)
    r = graph.match_resume(k, p_edges, step, mine, mode=mode, motifs=motifs, stream=stream)
    del fr
    if not reduce:
        return int(r.count), int(mine.shape[0])
    return reduce_count(r.count, coll_device=coll_device), int(mine.shape[0])
