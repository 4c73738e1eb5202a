"""Multi-GPU driver: replica grids partitioned over the GPUs of one box (BASELINE north_star (5)).

Partition (DESIGN.md §"Multi-GPU"): group g (all C candidates of one (rate, profile, seed)) runs on
rank g % world -- interleaved so that cheap (saturated) and expensive (low-load) groups spread evenly
-- and is claimed dynamically by the persistent K1 of that rank.  Whole groups stay on one rank, so the
per-group argmin (K3) is local.  The one exchange step of the method is merging the per-cell integer
histograms and counters: ONE all_reduce(SUM) of each integer cell buffer (NCCL over NVLink/NVSwitch),
plus an all_gather of the per-group best tables.  Integer addition is associative, so the reduced
cells and every derived argmin are bit-identical for any world size.
"""
import numpy as np

from . import sdas


def local_group_ids(n_groups, rank, world, group_range=None):
    """Global group ids handled by `rank` (the partition libsdas applies, sdas_grid.rank/world)."""
    gb, ge = group_range if group_range is not None else (0, n_groups)
    first = gb + (rank - gb % world) % world
    return np.arange(first, ge, world, dtype=np.int64)


def _staged(group):
    """gloo (the CPU test backend, or several ranks sharing one GPU) collects host tensors; NCCL device ones."""
    import torch.distributed as dist
    return dist.get_backend(group) == "gloo"


def _all_reduce_sum(x, group):
    import torch.distributed as dist
    if _staged(group) and x.is_cuda:
        h = x.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
        x.copy_(h)
    else:
        dist.all_reduce(x, op=dist.ReduceOp.SUM, group=group)


def reduce_cells(result, group=None):
    """all_reduce(SUM) of the int64 counters and int32 histograms of every cell (in place)."""
    import torch
    L = result.layout
    cnt = result.t["cell_cnt"][: L.n_cells * sdas.NCNT * 8].view(dtype=torch.int64)
    hist = result.t["cell_hist"][: L.n_cells * sdas.NHIST * sdas.NBINS * 4].view(dtype=torch.int32)
    _all_reduce_sum(cnt, group)
    _all_reduce_sum(hist, group)
    cs = result.t.get("cell_series")
    if cs is not None and cs.numel():                  # M15 cell-summed series: integer sums as well
        _all_reduce_sum(cs[: L.cell_series_bytes].view(dtype=torch.int64), group)


def gather_best_groups(result, n_groups, rank, world, group=None, group_range=None):
    """all_gather of the per-group best tables -> global int32 table [n_groups] on every rank (-1 outside
    group_range)."""
    import torch
    import torch.distributed as dist
    gb, ge = group_range if group_range is not None else (0, n_groups)
    per = (ge - gb + world - 1) // world + 1
    L = result.layout
    mine = torch.full((per,), -1, dtype=torch.int32, device=result.t["best_group"].device)
    n = L.n_local_groups
    if n:
        mine[:n] = result.t["best_group"][: n * 4].view(torch.int32)
    dev = mine.device
    if _staged(group) and mine.is_cuda:
        mine = mine.cpu()
    out = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(out, mine, group=group)
    out = [o.to(dev) for o in out]
    table = torch.full((n_groups,), -1, dtype=torch.int32, device=dev)
    for r in range(world):
        ids = torch.as_tensor(local_group_ids(n_groups, r, world, group_range), device=dev)
        table[ids] = out[r][: len(ids)]
    return table


def sweep(pipe, grid, objective="p99_e2e", objective_slo=0, rank=0, world=1, device="cuda", group=None,
          flags=0, result=None, pipeline=None, group_range=None):
    """One full distributed sweep: K1 + K3 on the local partition, the collective, then K4/K5.
    Returns (result, global best-group table or None, pipeline, grid view)."""
    P = pipeline or sdas.Pipeline(pipe)
    gv = sdas.GridView(pipe, grid, flags=flags, rank=rank, world=world, group_range=group_range)
    res = sdas.control_sweep(P, gv, objective=objective, objective_slo=objective_slo, device=device, result=result)
    table = None
    if world > 1:
        reduce_cells(res, group)
        table = gather_best_groups(res, res.layout.n_groups, rank, world, group, group_range)
    sdas.finalize(P, gv, res, objective=objective, objective_slo=objective_slo, device=device)
    return res, table, P, gv
