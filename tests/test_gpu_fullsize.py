"""Full-size parity in the launch configuration bench.py times (BASELINE.json configs 1-5).

Config 1 (384 replicas x 10,000 requests) is compared in full: every summary, record, cell and both
argmin tables.  Config 2 (1,048,576 replicas x 1000 requests, in-loop controller) runs entirely on
the GPU exactly as bench.py runs it (flags 0, one sdas_control_sweep + sdas_finalize); the oracle
recomputes a deterministic sample of replicas one by one and every summary field must match.  Configs
3-5 run at full size (3) or as 1M-replica slices of their full grids (4: 16.7M, 5: 64M), sampled the same way."""
import numpy as np
import pytest

import oracle
import workloads as W
from gpu_parity import compare_records, compare_summaries, full_check, run_gpu
from paper_2601_03197_b200 import sdas

pytestmark = pytest.mark.gpu


def test_config1_full():
    p, g = W.config1()
    gg = run_gpu(p, g, records=True, objective="p99_e2e")
    sdas.finalize(gg["P"], gg["gv"], gg["res"], objective="p99_e2e")
    import torch
    torch.cuda.synchronize()
    o = oracle.simulate(p, g)
    compare_summaries(gg["summary"], o["summary"], where="config1")
    compare_records(gg["records"], o["records"], gg["summary"])
    cnt, hist = oracle.cells(p, g, o)
    gcnt, ghist = gg["res"].cells()
    np.testing.assert_array_equal(gcnt, cnt)
    np.testing.assert_array_equal(ghist.astype(np.int64), hist)
    np.testing.assert_array_equal(gg["best_group"], oracle.argmin_groups(p, g, o["summary"], "p99_e2e"))
    np.testing.assert_array_equal(gg["res"].best_row(), oracle.argmin_rows(p, g, cnt, hist, "p99_e2e"))


def test_config2_full_size_sampled():
    p, g = W.config2(series_stride=0)
    P = sdas.Pipeline(p)
    gv = sdas.GridView(p, g)
    res = sdas.control_sweep(P, gv, objective="p99_e2e")
    sdas.finalize(P, gv, res, objective="p99_e2e")
    import torch
    torch.cuda.synchronize()
    summ = res.summary()
    R = W.grid_size(g)
    assert len(summ) == R == 1 << 20
    ids = np.asarray(W.sample_ids(R, 4096), dtype=np.uint64)         # 4096 sampled replicas
    o = oracle.simulate(p, g, ids=ids, records=False, hists=False)
    compare_summaries(summ[ids.astype(np.int64)], o["summary"], where="config2 sample")
    cnt, _ = res.cells()
    F = {n: i for i, n in enumerate(sdas.CELL_FIELDS)}
    assert int(cnt[:, F["n_replicas"]].sum()) == R
    assert int(cnt[:, F["arrivals"]].sum()) == int(summ["arrivals"].astype(np.int64).sum())
    assert int(cnt[:, F["mode_switches"]].sum()) == int(summ["mode_switches"].astype(np.int64).sum())


def test_config2_full_size_records_sampled():
    """The bench's config-2 launch with exact per-request records on (FLAG_RECORDS, 8.4 GB): every record of
    1024 sampled replicas (e2e and first feedback of each of their 1000 requests) equals the oracle's."""
    import torch
    p, g = W.config2(series_stride=0)
    P = sdas.Pipeline(p)
    gv = sdas.GridView(p, g, flags=sdas.FLAG_RECORDS)
    res = sdas.control_sweep(P, gv, objective="p99_e2e")
    torch.cuda.synchronize()
    ids = np.asarray(W.sample_ids(W.grid_size(g), 1024), dtype=np.int64)
    o = oracle.simulate(p, g, ids=ids.astype(np.uint64), records=True, hists=False)
    N = g["n_requests"]
    rec = res.t["records"].view(torch.int64).view(-1, N)[torch.as_tensor(ids, device=res.t["records"].device)]
    rec = rec.cpu().numpy().view(np.uint32).reshape(len(ids), N, 2)
    summ = res.summary()[ids]
    compare_summaries(summ, o["summary"], where="config2 records sample")
    compare_records(rec, o["records"], summ)


def test_max_requests_and_full_batches():
    """N = 65535 requests per replica (SDAS_MAX_REQUESTS) with B = 32 (every lane a sequence), bit-exact."""
    p = W.p2_x()
    p["roles"][0]["max_num_seqs"] = 32
    p["roles"][1]["max_num_seqs"] = 32
    g = W.grid([W.static("token"), W.static("batch")], [W.poisson(1_300_000)], n_seeds=2, n_requests=65535)
    gg, o = full_check(p, g, threads=4)
    assert (gg["summary"]["completed"] == 65535).all()


@pytest.mark.parametrize("cfg", ["config3", "config4", "config5"])
def test_full_size_grid_sampled(cfg):
    """Configs 3-5 at their full BASELINE sizes (replica coordinates of the full grid): config 3 whole
    (1,048,576 replicas); configs 4 (16.7M) and 5 (64M) as a contiguous 1M-replica slice of groups taken
    from the middle of the grid.  One sdas_control_sweep as bench.py launches it (flags 0); the oracle
    recomputes a deterministic sample of the slice's replicas one by one."""
    import torch
    p, g = {"config3": W.config3, "config4": W.config4, "config5": W.config5}[cfg]()
    C = len(g["candidates"])
    G = W.grid_size(g) // C
    n_groups = min(G, (1 << 20) // C)
    g0 = ((G - n_groups) // 2 // n_groups) * n_groups
    objective = "large_under_slo" if cfg == "config4" else "p99_e2e"
    slo = 6_000_000 if cfg == "config4" else 0
    P = sdas.Pipeline(p)
    gv = sdas.GridView(p, g, group_range=(g0, g0 + n_groups))
    res = sdas.control_sweep(P, gv, objective=objective, objective_slo=slo)
    torch.cuda.synchronize()
    summ = res.summary()
    assert len(summ) == n_groups * C == 1 << 20
    local = np.asarray(W.sample_ids(len(summ), 2048), dtype=np.int64)
    ids = (local + g0 * C).astype(np.uint64)
    o = oracle.simulate(p, g, ids=ids, records=False, hists=False)
    compare_summaries(summ[local], o["summary"], where="%s slice sample" % cfg)
    assert int(summ["arrivals"].astype(np.int64).sum()) > 0
