"""Multi-GPU driver: one process per GPU (torch.distributed over NCCL; gloo for CPU tests).

Sharding: the data graph (Res(M2)) is replicated on every rank and the
partial-embedding frontier is row-sharded at its root: rank r expands only the seed rows whose
first plan vertex f(v_0) lies in its vertex range.  Disjoint seed ranges partition the result
(every embedding has exactly one image of v_0), so no frontier exchange is needed for
correctness; the ranges are cut by equal estimated work (arc prefix of the CSR, i.e. the seed
step's candidate count), and the only data-path collectives are the final reduction of the
uint64 count (C3: all_reduce SUM) and, in table mode, the gather of per-rank tables (C4)
followed by a k-way merge into canonical order.

Everything here is host-side plumbing; the matching itself is `Graph.match` (the C ABI).
"""
from __future__ import annotations

from typing import Callable

import numpy as np


def equal_work_cuts(work_prefix: np.ndarray, parts: int) -> list[int]:
    """Cut points c_0=0 <= c_1 <= ... <= c_parts=n over vertices so that each range holds about
    1/parts of the total work.  work_prefix[v] = work of vertices < v (length n+1, e.g. the
    CSR offsets: arcs per seed vertex)."""
    wp = np.asarray(work_prefix, dtype=np.int64)
    n = wp.size - 1
    total = int(wp[-1])
    cuts = [0]
    for r in range(1, parts):
        target = (total * r) // parts
        v = int(np.searchsorted(wp, target, side="left"))
        cuts.append(min(max(v, cuts[-1]), n))
    cuts.append(n)
    return cuts


def merge_tables(tables: list[np.ndarray], k: int) -> np.ndarray:
    """Canonical (lexicographic) order of the union of per-rank canonical tables."""
    if not tables:
        return np.zeros((0, k), np.int32)
    cat = np.concatenate([np.asarray(t, np.int32).reshape(-1, k) for t in tables])
    if cat.shape[0] == 0:
        return cat
    return cat[np.lexsort(cat.T[::-1])]


def match_sharded(local_match: Callable[[int, int], tuple[int, np.ndarray | None]],
                  work_prefix: np.ndarray, k: int, *, rank: int, world: int, device=None,
                  table: bool = False):
    """Run `local_match(seed_begin, seed_end) -> (count, rows|None)` on this rank's shard and
    combine: all_reduce(SUM) of the count; in table mode all_gather of the per-rank row counts
    (C1) and a gather of the rows to every rank, merged canonically.  Returns (count, rows)."""
    import torch
    import torch.distributed as tdist

    cuts = equal_work_cuts(work_prefix, world)
    cnt, rows = local_match(cuts[rank], cuts[rank + 1])
    dev = device if device is not None else torch.device("cpu")
    t = torch.tensor([int(cnt)], dtype=torch.int64, device=dev)
    tdist.all_reduce(t, op=tdist.ReduceOp.SUM)
    total = int(t.item())
    if not table:
        return total, None
    sizes = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    tdist.all_gather(sizes, torch.tensor([int(cnt)], dtype=torch.int64, device=dev))
    sizes = [int(s.item()) for s in sizes]
    mx = max(sizes) if sizes else 0
    local = torch.zeros((mx, k), dtype=torch.int32, device=dev)
    if cnt:
        local[:cnt] = torch.as_tensor(np.asarray(rows, np.int32)).to(dev)
    bufs = [torch.zeros((mx, k), dtype=torch.int32, device=dev) for _ in range(world)]
    tdist.all_gather(bufs, local)
    parts = [b[:s].cpu().numpy() for b, s in zip(bufs, sizes)]
    return total, merge_tables(parts, k)


def rebalance_rows(rows, work, *, rank: int, world: int):
    """Frontier rebalancing (collectives C1 + C2): every rank holds `rows`
    ([n_r, stride] int32) with per-row work estimates `work` ([n_r] int64).  Rows are assigned
    to ranks by their position in the global work prefix (rank order, then row order), so each
    rank receives a contiguous 1/world share of the total work; returns this rank's rows.
    all_gather of per-rank work totals (C1), all_to_all of row counts, all_to_all_single of the
    rows themselves (C2).  Works with NCCL (CUDA tensors) and gloo (CPU tensors)."""
    import torch
    import torch.distributed as tdist

    dev = rows.device
    n = int(rows.shape[0])
    stride = int(rows.shape[1]) if rows.dim() == 2 else 1
    w = work.to(torch.int64)
    tot = torch.tensor([int(w.sum().item()) if n else 0], dtype=torch.int64, device=dev)
    tots = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    tdist.all_gather(tots, tot)
    tots = [int(t.item()) for t in tots]
    total = sum(tots)
    base = sum(tots[:rank])
    if n:
        pos = base + torch.cumsum(w, 0) - w                      # exclusive global prefix
        dest = torch.clamp((pos * world) // max(total, 1), 0, world - 1) if total else \
            torch.zeros(n, dtype=torch.int64, device=dev)
        send = torch.bincount(dest, minlength=world).to(torch.int64)
    else:
        send = torch.zeros(world, dtype=torch.int64, device=dev)
    recv = torch.empty_like(send)
    tdist.all_to_all_single(recv, send)
    send_l = [int(x) for x in send.tolist()]
    recv_l = [int(x) for x in recv.tolist()]
    out = torch.empty((sum(recv_l), stride), dtype=rows.dtype, device=dev)
    src = rows.reshape(n, stride).contiguous()
    tdist.all_to_all_single(out, src, output_split_sizes=recv_l, input_split_sizes=send_l)
    return out


def match_rebalanced(graph, k: int, p_edges, work_prefix, *, rank: int, world: int, step: int,
                     stream=None, mode: str = "mono", reduce: bool = True):
    """Count mode with a frontier exchange: run the plan to level `step` on this rank's seed
    shard (dm_match_prefix), rebalance the level by estimated work across ranks (NCCL
    all-to-all), finish locally (dm_match_resume) and all_reduce the count (C3)."""
    import torch
    import torch.distributed as tdist

    cuts = equal_work_cuts(work_prefix, world)
    fr = graph.match_prefix(k, p_edges, step, mode=mode, seed_range=(cuts[rank], cuts[rank + 1]),
                            stream=stream)
    rows = fr.rows_tensor()
    work = fr.work_tensor()
    mine = rebalance_rows(rows, work, rank=rank, world=world)
    r = graph.match_resume(k, p_edges, step, mine, mode=mode, stream=stream)
    if not reduce:
        return int(r.count), int(mine.shape[0])
    t = torch.tensor([int(r.count)], dtype=torch.int64, device=rows.device)
    tdist.all_reduce(t, op=tdist.ReduceOp.SUM)
    return int(t.item()), int(mine.shape[0])


def graph_local_match(graph, k: int, p_edges, *, output: str = "count", stream=None, **kw):
    """local_match adapter over Graph.match for match_sharded."""
    def run(b: int, e: int):
        r = graph.match(k, p_edges, output=output, seed_range=(b, e), stream=stream, **kw)
        return r.count, r.rows
    return run
