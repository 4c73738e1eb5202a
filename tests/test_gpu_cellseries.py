"""GPU parity of the cell-summed window series (SDAS_FLAG_CELL_SERIES; DESIGN.md R-CSER):
K1 accumulates every window close of every replica into its cell with integer atomics; the result must
equal the oracle's cell series bit for bit -- on the bench's controller config, the routed 4-agent DAG,
an overloaded grid whose replicas overflow after closing windows, the two-level-ring kernel, and after the
world-2 all_reduce (gloo, both ranks on cuda:0)."""
import numpy as np
import pytest

import oracle
import workloads as W
from paper_2601_03197_b200 import sdas

pytestmark = pytest.mark.gpu


def _gpu_cell_series(p, g, extra=0):
    import torch
    P = sdas.Pipeline(p)
    gv = sdas.GridView(p, g, flags=sdas.FLAG_CELL_SERIES | extra)
    r = sdas.simulate(P, gv)
    torch.cuda.synchronize()
    return r, r.cell_series(g["series_windows"], P.n_inst)


@pytest.mark.parametrize("which", ["config2", "config3", "overloaded", "spill"])
def test_cell_series_parity(which):
    extra = 0
    if which == "config2":
        p, g = W.config2(n_seeds=4, n_requests=400, series_stride=0, series_windows=300)
    elif which == "config3":
        p, g = W.config3(n_seeds=2, n_requests=250)
        g["series_windows"] = 200
    elif which == "overloaded":
        p, g = W.config1(n_seeds=3, n_requests=1000)
        g["series_windows"] = 400
    else:
        p, g = W.config3(n_seeds=2, n_requests=250)
        g["series_windows"] = 200
        extra = sdas.FLAG_SPILL
    r, cs = _gpu_cell_series(p, g, extra)
    o = oracle.simulate(p, g, records=False, cell_series=True)
    np.testing.assert_array_equal(cs, o["cell_series"])
    assert cs[:, :, :, 2].sum() > 0
    if which == "overloaded":
        assert (o["summary"]["status"] == 1).any()


def _worker(rank, world, port, out):
    import os
    import torch
    import torch.distributed as dist
    from paper_2601_03197_b200 import parallel
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p, g = W.config2(n_seeds=3, n_requests=300, series_stride=0, series_windows=200)
        res, _, P, _ = parallel.sweep(p, g, rank=rank, world=world, device="cuda:0", flags=sdas.FLAG_CELL_SERIES)
        torch.cuda.synchronize()
        out[rank] = res.cell_series(200, P.n_inst).copy()
    finally:
        dist.destroy_process_group()


def test_cell_series_all_reduce_world2():
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = mp.get_context("spawn").Manager().dict()
    mp.start_processes(_worker, args=(2, port, out), nprocs=2, join=True, start_method="spawn")
    p, g = W.config2(n_seeds=3, n_requests=300, series_stride=0, series_windows=200)
    o = oracle.simulate(p, g, records=False, cell_series=True)
    for r in range(2):
        np.testing.assert_array_equal(out[r], o["cell_series"])
