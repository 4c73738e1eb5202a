"""GPU (libsdas through the C-ABI) vs oracle parity for the rest of the boundary:

* K4/K5 per-row argmin (sdas_finalize) and K3 (sdas_group_argmin) under every objective (rule M20, R-KEYS);
* sdas_metrics at CELL / GROUP / ROW scope against the oracle's cells and argmins,
  lower-edge pooled percentiles exact, fp64 means / throughput / goodput to 1e-12 (north_star);
* Table-1 knobs: sdas_set values reach the launch, sdas_reset restores the result;
* the encodings: > 65535 max_num_seqs / model-selection changes per replica, latencies reaching
  2^32 us (exact sums, saturated records), admission gate with one request class;
* the hand-derived control / routing scenarios of tests/test_oracle_control.py, bit-exact on the GPU;
* a reused Result too small for a new grid is refused (the C-ABI carries no buffer sizes).
"""
import numpy as np
import pytest

import oracle
import test_oracle_control as toc
import workloads as W
from gpu_parity import compare_summaries, full_check, run_gpu
from paper_2601_03197_b200 import sdas

pytestmark = pytest.mark.gpu

OBJS = list(sdas.OBJECTIVES)


def _sync():
    import torch
    torch.cuda.synchronize()


def _grid_for(obj):
    if obj == "large_under_slo":                       # config-4 slice: MMPP-2 + model selection
        p, g = W.config4(n_seeds=2, n_requests=300, candidates=W.config4_candidates()[::509])
        return p, g, 6_000_000
    if obj == "p99_e2e_int":                           # classes + priority + admission gate
        p, g = W.config_prio(n_seeds=3, n_requests=300)
        return p, g, 0
    p, g = W.config1(n_seeds=3, n_requests=300, rates=[1, 4, 7])   # includes TOKEN overflow (bad cells)
    g["candidates"] += [W.adaptive(["function"], lo=200, hi=600), W.adaptive(["function"], lo=500, hi=900, dwell=4)]
    return p, g, 0


@pytest.mark.parametrize("obj", OBJS)
def test_group_and_row_argmin_every_objective(obj):
    p, g, slo = _grid_for(obj)
    gg = run_gpu(p, g, objective=obj, objective_slo=slo)
    sdas.finalize(gg["P"], gg["gv"], gg["res"], objective=obj, objective_slo=slo)
    _sync()
    o = oracle.simulate(p, g)
    compare_summaries(gg["summary"], o["summary"], where=obj)
    cnt, hist = oracle.cells(p, g, o)
    np.testing.assert_array_equal(gg["best_group"], oracle.argmin_groups(p, g, o["summary"], obj, slo))
    np.testing.assert_array_equal(gg["res"].best_row(), oracle.argmin_rows(p, g, cnt, hist, obj, slo))
    # re-rank the same summaries / cells under every other objective (sdas_group_argmin, sdas_finalize)
    for other in OBJS:
        sdas.group_argmin(gg["P"], gg["gv"], gg["res"], objective=other, objective_slo=slo)
        sdas.finalize(gg["P"], gg["gv"], gg["res"], objective=other, objective_slo=slo)
        _sync()
        np.testing.assert_array_equal(gg["res"].best_group(), oracle.argmin_groups(p, g, o["summary"], other, slo),
                                      err_msg=other)
        np.testing.assert_array_equal(gg["res"].best_row(), oracle.argmin_rows(p, g, cnt, hist, other, slo),
                                      err_msg=other)


def _host(res):
    return {n: res.t[n].cpu().numpy() for n in ("summary", "cell_cnt", "cell_hist", "best_group", "best_row")
            if n in res.t}


def _rel(a, b):
    return abs(a - b) <= 1e-12 * abs(b)


@pytest.mark.parametrize("which", ["config1", "prio", "truncated"])
def test_metrics_cell_group_row_scopes(which):
    if which == "prio":
        p, g = W.config_prio(n_seeds=2, n_requests=250)
    else:
        p, g = W.config1(n_seeds=2, n_requests=300, rates=[1, 6, 7])
        if which == "truncated":
            g["max_ticks"] = 120_000_000
    gg = run_gpu(p, g, objective="p99_e2e")
    sdas.finalize(gg["P"], gg["gv"], gg["res"], objective="p99_e2e")
    _sync()
    o = oracle.simulate(p, g)
    cnt, hist = oracle.cells(p, g, o)
    F = {n: i for i, n in enumerate(sdas.CELL_FIELDS)}
    host = _host(gg["res"])
    for cell in range(len(cnt)):
        m = sdas.metrics(gg["P"], gg["gv"], host, "cell", cell)
        q = cnt[cell]
        st = 1 if q[F["n_overflow"]] else 2 if q[F["n_truncated"]] else 0
        assert m["status"] == st
        for name, f in (("n_replicas", "n_replicas"), ("admitted", "admitted"), ("dropped", "dropped"),
                        ("completed", "completed"), ("sum_e2e", "sum_e2e"), ("sum_ff", "sum_ff"),
                        ("makespan", "makespan_sum"), ("int_nsys", "int_nsys"), ("good", "good"),
                        ("arrivals", "arrivals"), ("deliveries", "deliveries"), ("recv_steps", "recv_steps"),
                        ("decode_steps", "decode_steps"), ("window_closes", "window_closes"),
                        ("mode_switches", "mode_switches"), ("tokens", "tokens"), ("completed_int", "completed_int"),
                        ("rejected", "rejected"), ("sum_e2e_int", "sum_e2e_int"), ("good_int", "good_int")):
            assert m[name] == int(q[F[f]]), (cell, name)
        for name, h, qq in (("p50_e2e", 0, 50), ("p99_e2e", 0, 99), ("p90_e2e", 0, 90), ("p50_ff", 1, 50),
                            ("p99_ff", 1, 99), ("p50_e2e_int", 2, 50), ("p99_e2e_int", 2, 99)):
            assert m[name] == oracle.pooled_pct(hist[cell, h], qq), (cell, name)
        n = int(q[F["completed"]])
        if n:
            assert _rel(m["mean_e2e"], float(q[F["sum_e2e"]]) / n) and _rel(m["mean_ff"], float(q[F["sum_ff"]]) / n)
        mk = int(q[F["makespan_sum"]])
        if mk:
            assert _rel(m["throughput"], float(n * 10 ** 6) / mk)
            assert _rel(m["goodput"], float(int(q[F["good"]]) * 10 ** 6) / mk)
    og = oracle.argmin_groups(p, g, o["summary"], "p99_e2e")
    for gi in range(len(og)):
        assert sdas.metrics(gg["P"], gg["gv"], host, "group", gi)["best"] == og[gi]
    orow = oracle.argmin_rows(p, g, cnt, hist, "p99_e2e")
    for r in range(len(orow)):
        assert sdas.metrics(gg["P"], gg["gv"], host, "row", r)["best"] == orow[r]
    # REPLICA scope: goodput and the ff bins now stored in the summary
    for x in range(len(o["summary"])):
        s = o["summary"][x]
        m = sdas.metrics(gg["P"], gg["gv"], host, "replica", x)
        if int(s["status"]) == 1 or int(s["makespan"]) == 0:
            continue
        assert _rel(m["goodput"], float(int(s["good"]) * 10 ** 6) / float(s["makespan"]))
        assert (m["bin_p50_ff"], m["bin_p99_ff"]) == (int(s["bin_p50_ff"]) & 0xFFFF, int(s["bin_p99_ff"]) & 0xFFFF)


KNOBS = [("agent:1/max_num_seqs", 4, lambda p: p["roles"][1].__setitem__("max_num_seqs", 4)),
         ("agent:0/n_functions", 2, lambda p: p["roles"][0].__setitem__("n_functions", 2)),
         ("link:0->1/comm_mode", 2, lambda p: p["links"][0].__setitem__("mode", "token")),
         ("link:0->1/chunk_tokens", 8, lambda p: p["links"][0].__setitem__("chunk", 8)),
         ("link:0->1/net_delay", 30000, lambda p: p["links"][0].__setitem__("net", 30000)),
         ("link:0->1/pacing_gap", 100000, lambda p: p["links"][0].__setitem__("pacing_gap", 100000))]


@pytest.mark.parametrize("knob,value,edit", KNOBS, ids=[k[0] for k in KNOBS])
def test_knob_set_reaches_the_launch_and_reset_restores(knob, value, edit):
    import copy
    p, g = W.config1(n_seeds=2, n_requests=200, rates=[1, 5])
    g["candidates"] = [W.static(None), W.adaptive([None], lo=300, hi=700)]   # modes from the link knob
    P = sdas.Pipeline(p)
    gv = sdas.GridView(p, g, flags=sdas.FLAG_RECORDS)
    base = sdas.simulate(P, gv)
    _sync()
    base_bytes = base.summary().tobytes()
    P.set(knob, value)
    assert P.get(knob) == value
    r = sdas.simulate(P, gv)
    _sync()
    p2 = copy.deepcopy(p)
    edit(p2)
    o = oracle.simulate(p2, g)
    compare_summaries(r.summary(), o["summary"], where=knob)
    assert r.summary().tobytes() != base_bytes                  # the knob changed the model
    P.reset(knob)
    r2 = sdas.simulate(P, gv)
    _sync()
    assert r2.summary().tobytes() == base_bytes


def test_knob_errors():
    P = sdas.Pipeline(W.p2_x())
    with pytest.raises(sdas.SdasError) as e:
        P.set("agent:1/max_num_seqs", 0)
    assert e.value.code == sdas.E_OUT_OF_RANGE
    with pytest.raises(sdas.SdasError) as e:
        P.set("agent:1/no_such_knob", 1)
    assert e.value.code == sdas.E_UNKNOWN_PARAM
    with pytest.raises(sdas.SdasError) as e:
        P.set("link:1->0/comm_mode", 1)
    assert e.value.code == sdas.E_UNKNOWN_PARAM


# ------------------------------------------------------------------ encodings
def test_batch_changes_beyond_u16():
    # fast / slow instances of one source role under RR, both under batch control (B default 2), one request
    # per window: e2e alternates 100 (fast: calm -> reset both to 2) and 300 (slow: viol, Q = 0 -> halve
    # both to 1), so every window close after the first changes both instances: 2 (N - 2) changes
    N = 40000
    fast = W.cost(h=0, alpha=1, beta=0, tau0=99, gamma=0)
    slow = W.cost(h=0, alpha=1, beta=0, tau0=299, gamma=0)
    p = toc.srv(2, B=2, inst_cost=[fast, slow], route="rr")
    g = W.grid([toc.batch_cand(250)], [W.arr_list([1000 * j for j in range(N)], prompt=(1, 1), output=(1, 1))],
               n_requests=N)
    gg, o = full_check(p, g, objective=None)
    assert int(o["summary"][0]["batch_changes"]) == 2 * (N - 2) > 65535
    assert int(gg["summary"][0]["batch_changes"]) == 2 * (N - 2)


def test_select_changes_beyond_u16():
    # one request on LARGE decoding for 1.4e8 ticks: LARGE busy 1000 / window -> SMALL, SMALL idle -> LARGE,
    # ... every one of the 140000 window closes switches (rule M16(iii))
    large = dict(W.cost(h=0, alpha=1, beta=0, tau0=139_999_999, gamma=0), large=1)
    p = toc.srv(2, inst_cost=[large, toc.SMALL], route="select")
    g = W.grid([toc.sel_cand(10 ** 12)], [W.arr_list([0], prompt=(1, 1), output=(1, 1))], n_requests=1)
    gg, o = full_check(p, g, objective=None)
    assert int(o["summary"][0]["select_changes"]) == 140000 == int(gg["summary"][0]["select_changes"])


def test_saturated_latencies_exact_sums():
    s_ = (2 ** 32 - 1) // 3                             # e2e = s, 2s, 2^32 - 1, 4s (tests/test_oracle_control.py)
    g = W.grid([W.static()], [W.arr_list([0] * 4, prompt=(0, 0), output=(0, 0))], n_requests=4)
    gg, o = full_check(W.tool1(s_), g, objective=None)
    s = gg["summary"][0]
    assert int(s["n_saturated"]) == 2 and int(s["sum_e2e"]) == int(s["sum_ff"]) == 10 * s_
    assert gg["records"][0, :, 0].tolist() == [s_, 2 * s_, 0xFFFFFFFF, 0xFFFFFFFF]


def test_admission_gate_with_one_class():
    # a gate on a single-class workload rejects every arrival while closed (M28) -- the kernel
    # must run it (CLS instantiation) although no arrival profile has interactive requests
    p, g = W.config_prio(n_seeds=2, n_requests=300)
    for a in g["arrivals"]:
        a[0]["interactive"] = 0
    gg, o = full_check(p, g)
    assert (o["summary"]["rejected"] > 0).any()


@pytest.mark.parametrize("name", ["batch_seq", "batch_dwell", "select_busy", "select_viol", "rr", "load",
                                  "trunc", "ovf"])
def test_hand_scenarios_on_gpu(name):
    cases = {
        "batch_seq": (toc.srv(B=4), toc.batch_cand(250), toc.bursts(toc.KS), 10),
        "batch_dwell": (toc.srv(B=4), toc.batch_cand(250, dwell=2), toc.bursts(toc.KS), 10),
        "select_busy": (toc.srv(2, inst_cost=[toc.LARGE, toc.SMALL], route="select"), toc.sel_cand(10 ** 9),
                        [0, 400, 1000, 1100, 2300, 2700, 3200, 4000, 4400] + [5000 + 100 * i for i in range(7)] +
                        [6000, 8000], 9),
        "select_viol": (toc.srv(2, inst_cost=[dict(toc.LARGE, tau0=199), toc.SMALL], route="select"),
                        toc.sel_cand(150, dwell=2), [0, 1000, 2000, 3000], 4),
    }
    if name in cases:
        p, cand, ticks, nw = cases[name]
        g = W.grid([cand], [W.arr_list(ticks, prompt=(1, 1), output=(1, 1))], n_requests=len(ticks),
                   series_stride=1, series_slots=1, series_windows=nw)
        full_check(p, g, series=True, objective=None)
    elif name == "rr":
        for mode in ("function", "token", "batch"):
            g = W.grid([W.static(mode)], [W.arr_list([0, 1000, 2000, 3000], prompt=(1, 1), output=(4, 4))],
                       n_requests=4)
            full_check(toc.rr_pipe(mode), g, objective=None)
    elif name == "load":
        S = W.role("S", 1, W.cost(h=0, alpha=100, beta=0, tau0=1, gamma=0))
        T = W.role("T", 1, W.cost(h=0, alpha=200, beta=0, tau0=1, gamma=0), out=(0, 0, 1))
        p = W.pipeline([S, T], [W.link(0, 1, net=300, mode="function")], window=1000)
        cands = [W.adaptive(["function"], metric=m, lo=300, hi=500) for m in ("load", "busy")]
        g = W.grid(cands, [W.arr_list([0, 1000, 1050, 3000], prompt=(0, 0), output=(0, 0))], n_requests=4,
                   series_stride=1, series_slots=2, series_windows=4)
        full_check(p, g, series=True, objective=None)
    elif name == "trunc":
        for mt in (100, 113, 126, 127):
            g = W.grid([W.static("batch")], [W.arr_list([0, 3])], n_requests=2, max_ticks=mt)
            full_check(W.toy_ht("batch"), g, objective=None)
    else:
        p = W.tool1(10)
        p["roles"][0]["inbox_cap"] = 2
        for ticks in ([5, 5, 6, 7], [5, 5, 5, 9]):
            g = W.grid([W.static()], [W.arr_list(ticks, prompt=(0, 0), output=(0, 0))], n_requests=4)
            gg, o = full_check(p, g, objective=None)
            assert int(gg["summary"][0]["status"]) == 1


def test_reused_result_too_small_is_refused():
    p, g = W.config1(n_seeds=1, n_requests=100, rates=[0])
    P = sdas.Pipeline(p)
    small = sdas.simulate(P, sdas.GridView(p, g))
    p2, g2 = W.config1(n_seeds=4, n_requests=100)
    with pytest.raises(sdas.SdasError) as e:
        sdas.simulate(P, sdas.GridView(p2, g2), result=small)
    assert e.value.code == sdas.E_BUFFER
