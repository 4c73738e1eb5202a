"""Multi-process (gloo, world_size 2, CPU) coverage of the N>1 path of paper_2601_03197_b200.parallel:
the group-interleaved partition, the all_reduce(SUM) of the integer cell buffers and the all_gather
of per-group best tables.  Cell contributions of each rank come from the CPU oracle
on that rank's replicas; the reduced buffers must equal the oracle's full-grid cells bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import workloads as W
from paper_2601_03197_b200 import parallel, sdas


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class FakeLayout:
    def __init__(self, n_cells, n_local_groups, n_groups):
        self.n_cells, self.n_local_groups, self.n_groups = n_cells, n_local_groups, n_groups


class FakeResult:
    """Host-tensor stand-in for sdas.Result with the same buffer layout (uint8 views)."""

    def __init__(self, cnt, hist, best):
        self.layout = FakeLayout(cnt.shape[0], len(best), None)
        self.t = {"cell_cnt": torch.from_numpy(np.ascontiguousarray(cnt).view(np.uint8).copy()),
                  "cell_hist": torch.from_numpy(np.ascontiguousarray(hist.astype(np.int32)).view(np.uint8).copy()),
                  "best_group": torch.from_numpy(np.ascontiguousarray(best.astype(np.int32)).view(np.uint8).copy())}


def _partial_cells(p, g, res, ids):
    """Cell sums over the given replicas (same counter layout as libsdas / oracle.cells)."""
    C, S, K, I = len(g["candidates"]), g["n_seeds"], len(g["arrivals"][0]), len(g["arrivals"])
    cnt = np.zeros((I * K * C, sdas.NCNT), np.int64)
    hist = np.zeros((I * K * C, sdas.NHIST, sdas.NBINS), np.int64)
    F = {n: i for i, n in enumerate(sdas.CELL_FIELDS)}
    for x, r in enumerate(ids):
        s = res["summary"][x]
        cell = (r // C // S) * C + r % C
        q = cnt[cell]
        q[F["n_replicas"]] += 1
        if s["status"] == 1:
            q[F["n_overflow"]] += 1
            continue
        q[F["n_ok"]] += s["status"] == 0
        q[F["n_truncated"]] += s["status"] == 2
        for f in ("admitted", "dropped", "completed", "sum_e2e", "sum_ff", "int_nsys", "good", "large_items",
                  "arrivals", "deliveries", "recv_steps", "decode_steps", "window_closes", "mode_switches", "tokens",
                  "batch_changes", "select_changes", "n_saturated", "kv_transfers", "completed_int", "rejected",
                  "sum_e2e_int", "good_int"):
            q[F[f]] += int(s[f])
        q[F["makespan_sum"]] += int(s["makespan"])
        hist[cell] += res["hists"][x]
    return cnt, hist


def _worker(rank, world, port, p, g, full_cnt, full_hist, full_best, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        C = len(g["candidates"])
        n_groups = W.grid_size(g) // C
        groups = parallel.local_group_ids(n_groups, rank, world)
        ids = np.array([gg * C + c for gg in groups for c in range(C)], dtype=np.uint64)
        res = oracle.simulate(p, g, ids=ids, threads=2)
        cnt, hist = _partial_cells(p, g, res, ids.astype(np.int64))
        best = np.full(len(groups), -1, np.int32)
        # local per-group argmin via the oracle on the local summaries (groups are whole on one rank)
        for li in range(len(groups)):
            one = W.grid(g["candidates"], [g["arrivals"][0]], n_seeds=1, n_requests=g["n_requests"])
            best[li] = oracle.argmin_groups(p, one, np.ascontiguousarray(res["summary"][li * C:(li + 1) * C]),
                                            "p99_e2e")[0]
        fr = FakeResult(cnt, hist, best)
        parallel.reduce_cells(fr)
        table = parallel.gather_best_groups(fr, n_groups, rank, world)
        rc = fr.t["cell_cnt"].numpy().view(np.int64).reshape(full_cnt.shape)
        rh = fr.t["cell_hist"].numpy().view(np.int32).reshape(full_hist.shape)
        ok = (np.array_equal(rc, full_cnt) and np.array_equal(rh.astype(np.int64), full_hist)
              and np.array_equal(table.numpy(), full_best))
        out[rank] = 1 if ok else 0
    finally:
        dist.destroy_process_group()


def test_partition_covers_every_group_once():
    for n_groups in (1, 7, 40, 1000):
        for world in (1, 2, 3, 8):
            ids = np.concatenate([parallel.local_group_ids(n_groups, r, world) for r in range(world)])
            assert sorted(ids.tolist()) == list(range(n_groups))
            for r in range(world):
                assert all(int(x) % world == r for x in parallel.local_group_ids(n_groups, r, world))


@pytest.mark.parametrize("world", [2])
def test_gloo_world2_cells_and_best_tables_bit_exact(world):
    p, g = W.config1(n_seeds=3, n_requests=250, rates=[0, 3, 7])
    full = oracle.simulate(p, g, threads=4)
    full_cnt, full_hist = oracle.cells(p, g, full)
    full_best = oracle.argmin_groups(p, g, full["summary"], "p99_e2e")
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, _free_port(), p, g, full_cnt, full_hist, full_best, out), nprocs=world,
             join=True)
    assert dict(out) == {r: 1 for r in range(world)}
