"""Helpers for GPU <-> oracle parity (imported by the -m gpu tests)."""
import numpy as np

import oracle
from paper_2601_03197_b200 import sdas

# product summary field -> oracle summary field
FIELDS = ["status", "admitted", "dropped", "completed", "sum_e2e", "sum_ff", "int_nsys", "p50_e2e", "p99_e2e",
          "p50_ff", "p99_ff", "max_e2e", "n_saturated", "arrivals", "deliveries", "recv_steps", "decode_steps",
          "window_closes", "mode_switches", "good", "large_items", "tokens", "batch_changes", "select_changes",
          "kv_transfers", "p90_e2e", "completed_int", "rejected", "sum_e2e_int", "p50_e2e_int", "p99_e2e_int",
          "good_int", "gate_changes"]
BINS = ["bin_p50_e2e", "bin_p99_e2e", "bin_p50_ff", "bin_p99_ff"]


def run_gpu(pipe, grid, records=True, series=False, trace_replica=None, objective=None, objective_slo=0,
            rank=0, world=1, group_range=None, stepwise=False, generic=False, mid=False, spill=False):
    flags = (sdas.FLAG_RECORDS if records else 0) | (sdas.FLAG_SERIES if series else 0)
    flags |= (sdas.FLAG_STEPWISE if stepwise else 0) | (sdas.FLAG_GENERIC if generic else 0)
    flags |= sdas.FLAG_MID if mid else 0
    flags |= sdas.FLAG_SPILL if spill else 0
    P = sdas.Pipeline(pipe)
    gv = sdas.GridView(pipe, grid, flags=flags, rank=rank, world=world, group_range=group_range,
                       trace_replica=trace_replica, trace_cap=1 << 18)
    res = sdas.simulate(P, gv, objective=objective, objective_slo=objective_slo)
    import torch
    torch.cuda.synchronize()
    out = {"P": P, "gv": gv, "res": res, "summary": res.summary()}
    if records:
        out["records"] = res.records(grid["n_requests"])
    if series:
        out["series"] = res.series(grid["series_slots"], grid["series_windows"], P.n_inst)
    if trace_replica is not None:
        out["trace"] = res.trace()
    out["cells"] = res.cells()
    if objective is not None:
        out["best_group"] = res.best_group()
    return out


def compare_summaries(gs, osum, ids=None, where=""):
    """Field-by-field, bit-exact comparison of product and oracle summaries."""
    assert len(gs) == len(osum)
    bad = []
    for x in range(len(gs)):
        g, o = gs[x], osum[x]
        for f in FIELDS:
            if int(g[f]) != int(o[f]):
                bad.append((x, f, int(g[f]), int(o[f])))
        for f in BINS:
            if int(g[f]) != (int(o[f]) & 0xFFFF):
                bad.append((x, f, int(g[f]), int(o[f])))
        mk = int(o["stop_tick"]) if int(o["status"]) == 1 else int(o["makespan"])
        if int(g["makespan"]) != mk:
            bad.append((x, "makespan", int(g["makespan"]), mk))
        if len(bad) > 20:
            break
    assert not bad, "%s first mismatches: %s" % (where, bad[:20])


def compare_records(grec, orec, gs):
    for x in range(len(gs)):
        n = int(gs[x]["completed"])
        if int(gs[x]["status"]) == 1:
            continue
        np.testing.assert_array_equal(grec[x, :n], orec[x, :n], err_msg="records of local replica %d" % x)


def sorted_trace(tr):
    rows = [(int(r["tick"]), int(r["code"]), int(r["a"]), int(r["b"]), int(r["c"])) for r in tr]
    return sorted(rows)


def first_divergence(a, b):
    for k, (x, y) in enumerate(zip(a, b)):
        if x != y:
            return k, x, y
    if len(a) != len(b):
        return min(len(a), len(b)), None, None
    return None


def full_check(pipe, grid, series=False, objective="p99_e2e", objective_slo=0, threads=None, **kw):
    """GPU vs oracle on a whole (small) grid: summaries, records, series, cells, argmins."""
    g = run_gpu(pipe, grid, records=True, series=series, objective=objective, objective_slo=objective_slo, **kw)
    o = oracle.simulate(pipe, grid, series=series, threads=threads)
    compare_summaries(g["summary"], o["summary"])
    compare_records(g["records"], o["records"], g["summary"])
    if series:
        np.testing.assert_array_equal(g["series"].view(np.uint8), o["series"].view(np.uint8))
    cnt, hist = oracle.cells(pipe, grid, o)
    gcnt, ghist = g["cells"]
    np.testing.assert_array_equal(gcnt, cnt)
    np.testing.assert_array_equal(ghist.astype(np.int64), hist)
    if objective is not None:
        ob = oracle.argmin_groups(pipe, grid, o["summary"], objective, objective_slo)
        np.testing.assert_array_equal(g["best_group"], ob)
    return g, o
