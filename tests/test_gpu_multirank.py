"""The multi-rank path on a device (north_star (5)): world = 2 and 3 processes, all on
cuda:0 with gloo (one GPU in this environment; NCCL refuses two ranks on one device), each running
parallel.sweep -- K1 + K3 on its group-interleaved partition, the all_reduce(SUM) of the integer cell
buffers, the all_gather of the per-group best tables, K4/K5 on the reduced cells -- and the reduced
cells, the gathered best-group table and best_row must equal the world = 1 run byte for byte (integer
addition is associative).  The world = 1 run is itself checked against the oracle."""
import os
import socket

import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _grid():
    # ragged: 8 rates x 5 seeds = 40 groups (not a multiple of 3), TOKEN overflows at high load
    p, g = W.config1(n_seeds=5, n_requests=300)
    g["candidates"].append(W.adaptive(["function"], lo=300, hi=700))
    return p, g


def _collect(res, table):
    cnt, hist = res.cells()
    return {"cnt": cnt.copy(), "hist": hist.copy(), "best_row": res.best_row().copy(),
            "table": None if table is None else table.cpu().numpy().copy()}


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    from paper_2601_03197_b200 import parallel
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p, g = _grid()
        res, table, _, _ = parallel.sweep(p, g, objective="p99_e2e", rank=rank, world=world, device="cuda:0")
        torch.cuda.synchronize()
        out[rank] = _collect(res, table)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_multirank_sweep_equals_world1(world):
    import torch
    import torch.multiprocessing as mp
    from paper_2601_03197_b200 import parallel
    p, g = _grid()
    res1, _, _, _ = parallel.sweep(p, g, objective="p99_e2e", device="cuda:0")
    torch.cuda.synchronize()
    one = _collect(res1, None)
    # world 1 == oracle
    o = oracle.simulate(p, g, records=False)
    cnt, hist = oracle.cells(p, g, o)
    np.testing.assert_array_equal(one["cnt"], cnt)
    np.testing.assert_array_equal(one["hist"].astype(np.int64), hist)
    np.testing.assert_array_equal(one["best_row"], oracle.argmin_rows(p, g, cnt, hist, "p99_e2e"))
    best_groups = oracle.argmin_groups(p, g, o["summary"], "p99_e2e")
    np.testing.assert_array_equal(res1.best_group(), best_groups)
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    mp.start_processes(_worker, args=(world, _free_port(), out), nprocs=world, join=True, start_method="spawn")
    assert sorted(out.keys()) == list(range(world))
    for r in range(world):
        got = out[r]
        np.testing.assert_array_equal(got["cnt"], one["cnt"])
        np.testing.assert_array_equal(got["hist"], one["hist"])
        np.testing.assert_array_equal(got["best_row"], one["best_row"])
        np.testing.assert_array_equal(got["table"], best_groups)      # ragged partitions padded with -1 internally
