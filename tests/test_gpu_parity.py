"""GPU (libsdas sm_100a, through the C-ABI) vs CPU oracle parity.

Bar (BASELINE.json north_star): histograms, event counts, percentiles and controller decisions
bit-exact (time is integer); derived fp64 means to 1e-12 relative.  Sizes here span several
waves of the persistent kernel and ragged tails; test_gpu_fullsize.py covers the bench
configuration at full size on sampled replicas.
"""
import numpy as np
import pytest

import oracle
import workloads as W
from gpu_parity import compare_records, compare_summaries, first_divergence, full_check, run_gpu, sorted_trace

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", ["token", "function", "batch"])
def test_ht0_spec_trace(mode):
    p = W.p2_spec(mode=mode, chunk=16, n_functions=2)
    g = W.grid([W.static(mode)], [W.arr_list([0], prompt=(100, 100), output=(32, 32))], n_requests=1)
    gg, o = full_check(p, g)
    assert int(gg["summary"][0]["p50_e2e"]) == {"token": 780800, "function": 657800, "batch": 786600}[mode]


@pytest.mark.parametrize("mode", ["batch", "function", "token"])
def test_ht13(mode):
    p = W.toy_ht(mode)
    g = W.grid([W.static(mode)], [W.arr_list([0, 3])], n_requests=2, series_stride=1, series_slots=1,
               series_windows=1)
    full_check(p, g, series=True)


@pytest.mark.parametrize("mode", ["batch", "function", "token"])
def test_trace_equivalence(mode):
    p = W.p2_x(mode=mode)
    g = W.grid([W.static(mode)], [W.poisson(570571)], n_seeds=2, n_requests=150)
    gg = run_gpu(p, g, trace_replica=1)
    o = oracle.simulate(p, g, trace_id=1)
    a, b = sorted_trace(gg["trace"]), sorted_trace(o["trace"])
    # an overflowed replica is discarded (rule M14); compare the traces up to the overflow tick
    t_ovf = min([r[0] for r in a + b if r[1] == 12] + [1 << 63])
    a, b = [r for r in a if r[0] < t_ovf], [r for r in b if r[0] < t_ovf]
    assert first_divergence(a, b) is None, first_divergence(a, b)
    assert int(gg["summary"][1]["status"]) == int(o["summary"][1]["status"])


@pytest.mark.parametrize("svc", ["det", "exp"])
def test_tools_lindley_tandem(svc):
    p = W.tool1(70000, svc=svc)
    g = W.grid([W.static()], [W.poisson(100000, output=(0, 0))], n_seeds=37, n_requests=700)
    full_check(p, g)
    p = W.tandem(60000, 70000, 1000, svc=svc)
    g = W.grid([W.static("batch")], [W.poisson(100000, output=(0, 0))], n_seeds=37, n_requests=700)
    full_check(p, g)


def test_config1_reduced():
    # all 8 rates x 3 modes x 3 seeds, N = 1500 (includes TOKEN overflow at high load)
    p, g = W.config1(n_seeds=3, n_requests=1500)
    gg, o = full_check(p, g, objective="p99_e2e")
    st = gg["summary"]["status"]
    assert (st == 1).any() and (st == 0).any()


@pytest.mark.parametrize("obj", ["p50_e2e", "p99_ff", "throughput", "goodput"])
def test_objectives(obj):
    p, g = W.config1(n_seeds=2, n_requests=400)
    full_check(p, g, objective=obj)


def test_config2_controller_reduced():
    p, g = W.config2(n_seeds=3, n_requests=400, series_stride=7, series_windows=64)
    gg, o = full_check(p, g, series=True)
    assert gg["summary"]["mode_switches"].sum() > 0


def test_config3_routing_batch_control_reduced():
    p, g = W.config3(n_seeds=2, n_requests=250)
    gg, o = full_check(p, g)
    s = gg["summary"]
    assert s["batch_changes"].sum() > 0 and s["mode_switches"].sum() > 0


def test_config4_mmpp_model_selection_reduced():
    cands = W.config4_candidates()[::331]
    p, g = W.config4(n_seeds=1, n_requests=300, candidates=cands)
    gg, o = full_check(p, g, objective="large_under_slo", objective_slo=6_000_000)
    s = gg["summary"]
    assert s["select_changes"].sum() > 0 and s["large_items"].sum() > 0


def test_config5_policy_mappings_reduced():
    p, g = W.config5(n_seeds=2, n_requests=300, n_rates=6, n_candidates=70)
    full_check(p, g)


def test_truncation_and_load_metric():
    p = W.p2_x()
    cands = [W.adaptive(["function"], metric="load", lo=2000, hi=6000), W.static("batch")]
    g = W.grid(cands, [W.poisson(m) for m in (998500, 399400)], n_seeds=3, n_requests=600,
               max_ticks=150_000_000)
    gg, o = full_check(p, g)
    assert (gg["summary"]["status"] == 2).any()


def test_rank_partition_matches_full_grid():
    p, g = W.config1(n_seeds=3, n_requests=300)
    full = run_gpu(p, g)
    ids = []
    for rank in range(3):
        part = run_gpu(p, g, rank=rank, world=3)
        L = part["res"].layout
        C = len(g["candidates"])
        for lg in range(L.n_local_groups):
            gidx = rank + lg * 3
            for c in range(C):
                a = part["summary"][lg * C + c]
                b = full["summary"][gidx * C + c]
                assert a.tobytes() == b.tobytes()
                ids.append(gidx * C + c)
    assert sorted(ids) == list(range(len(full["summary"])))


def test_metrics_derived_fp64():
    p, g = W.config1(n_seeds=2, n_requests=300, rates=[1, 6])
    gg = run_gpu(p, g)
    from paper_2601_03197_b200 import sdas
    host = {"summary": gg["res"].t["summary"].cpu().numpy()}
    o = oracle.simulate(p, g)
    for x in range(len(gg["summary"])):
        m = sdas.metrics(gg["P"], gg["gv"], host, "replica", x)
        s = o["summary"][x]
        if s["status"] != 0:
            continue
        n = float(s["completed"])
        for got, want in ((m["mean_e2e"], float(s["sum_e2e"]) / n), (m["mean_ff"], float(s["sum_ff"]) / n),
                          (m["throughput"], float(int(s["completed"]) * 10 ** 6) / float(s["makespan"]))):
            assert abs(got - want) <= 1e-12 * abs(want)


# ------------------------------------------------------------------ f1: KV transfer + hints (M21-M24)
@pytest.mark.parametrize("kv", ["off", "affinity", "recompute", "posthoc", "hint"])
def test_kv_single_request(kv):
    import json
    import os
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "ht_kv.json")))
    p = W.p2_kv(home_skew=1000)
    p["roles"][1]["route"] = "fixed"
    p["roles"][1]["route_fixed"] = 1
    g = W.grid([W.with_kv(W.static("batch"), kv)], [W.arr_list([0], prompt=(100, 100), output=(32, 32))],
               n_requests=1)
    gg, _ = full_check(p, g)
    want = gold["single_request_fixed_to_tester1"][kv]
    assert int(gg["summary"][0]["p50_e2e"]) == want["e2e"] and int(gg["summary"][0]["kv_transfers"]) == want[
        "kv_transfers"]


def test_kv_fig6_grid():
    p, g = W.config_kv(n_seeds=3, n_requests=400)
    gg, o = full_check(p, g, objective="goodput")
    assert gg["summary"]["kv_transfers"].sum() > 0


def test_kv_with_function_mode_and_rr():
    p = W.p2_kv(ctx_tokens=1500, home_skew=500)
    p["links"][0]["mode"] = "function"
    cands = [W.with_kv(W.static("function"), k) for k in ("affinity", "hint", "posthoc")]
    cands.append(W.with_kv(dict(W.static("token"), route="rr"), "recompute"))
    g = W.grid(cands, [W.poisson(m) for m in (600000, 280000)], n_seeds=3, n_requests=300)
    full_check(p, g)


# ------------------------------------------------------------------ silent-run coalescing
@pytest.mark.parametrize("cfg", ["config1", "config2", "config3", "config4", "kv", "trunc"])
def test_coalesced_runs_equal_stepwise(cfg):
    """SDAS_FLAG_STEPWISE (one event per DECODE step) and the default coalesced runs give identical bytes:
    summaries, records, series and cells."""
    if cfg == "config1":
        p, g = W.config1(n_seeds=3, n_requests=800)
    elif cfg == "config2":
        p, g = W.config2(n_seeds=3, n_requests=400, series_stride=5, series_windows=64)
    elif cfg == "config3":
        p, g = W.config3(n_seeds=2, n_requests=250)
    elif cfg == "config4":
        p, g = W.config4(n_seeds=1, n_requests=300, candidates=W.config4_candidates()[::97])
    elif cfg == "kv":
        p, g = W.config_kv(n_seeds=3, n_requests=300)
    else:
        p = W.p2_x()
        cands = [W.adaptive(["function"], metric="load", lo=2000, hi=6000), W.static("batch"), W.static("token")]
        g = W.grid(cands, [W.poisson(m) for m in (998500, 399400)], n_seeds=3, n_requests=600,
                   max_ticks=150_000_000)
    series = g.get("series_stride", 0) > 0
    a = run_gpu(p, g, series=series)
    b = run_gpu(p, g, series=series, stepwise=True)
    assert a["summary"].tobytes() == b["summary"].tobytes()
    for x, n in enumerate(a["summary"]["completed"]):   # records past `completed` are never written
        assert np.array_equal(a["records"][x, :n], b["records"][x, :n])
    assert np.array_equal(a["cells"][0], b["cells"][0]) and np.array_equal(a["cells"][1], b["cells"][1])
    if series:
        assert a["series"].tobytes() == b["series"].tobytes()


# ------------------------------------------------------------------ f3: compiled intents, guard M25, p90
def test_guard_alternation_toy():
    p = W.toy_ht("token")
    p["window"] = 1000
    p["roles"][1]["cost"]["h"] = 40
    cands = []
    for bound, dwell in ((131, 1), (131, 2), (0, 1), (215, 1)):
        c = W.static("token")
        c.update(kind="adaptive", dwell=dwell, policy_slo=bound, guard_links=[0], guard_pct=90)
        cands.append(c)
    g = W.grid(cands, [W.arr_list([j * 1000 for j in range(7)], prompt=(4, 4), output=(4, 4))], n_requests=7,
               series_stride=1, series_slots=4, series_windows=7)
    gg, o = full_check(p, g, series=True)
    assert [int(v) for v in gg["summary"]["mode_switches"]] == [6, 3, 1, 0]


@pytest.mark.parametrize("objective", ["p90_e2e", "throughput"])
def test_compiled_intent_grid(objective):
    from paper_2601_03197_b200 import sdas
    p = W.p2_x()
    P = sdas.Pipeline(p)
    cands = []
    for obj in ("max_throughput", "min_p90_latency"):
        for k in ([], [("e2e_p90", 3_000_000, [])], [("e2e_p99", 6_000_000, [])]):
            cands.append(sdas.compile_intent(P, obj, constraints=k)[0])
    cands.append(sdas.compile_intent(P, rules=W.static("batch"), constraints=[("e2e_p90", 2_500_000, [])])[0])
    g = W.grid(cands, [W.poisson(m) for m in (1597600, 726182, 469882)], n_seeds=3, n_requests=300)
    gg, o = full_check(p, g, objective=objective)
    s = gg["summary"]
    assert s["mode_switches"].sum() > 0 and (s["p90_e2e"][s["status"] == 0] > 0).all()


# ------------------------------------------------------------------ f2: classes, priority, admission (M26-M29)
@pytest.mark.parametrize("prio", [False, True])
def test_prio_single_server_trace(prio):
    rng = np.random.default_rng(5)
    ticks = np.cumsum(rng.integers(100, 1300, size=300)).tolist()
    p = W.tool1(700)
    g = W.grid([W.with_prio(W.static(), prio)], [W.with_classes(W.arr_list(ticks, prompt=(0, 0), output=(0, 0)),
                                                                400)], n_requests=300)
    gg, o = full_check(p, g)
    tr = run_gpu(p, g, trace_replica=0)["trace"]
    assert first_divergence(sorted_trace(tr), sorted_trace(oracle.simulate(p, g, trace_id=0)["trace"])) is None


def test_config_prio_grid():
    p, g = W.config_prio(n_seeds=3, n_requests=300, gaps=(1597600, 726182, 469882))
    gg, o = full_check(p, g, objective="p99_e2e_int")
    s = gg["summary"]
    assert s["rejected"].sum() > 0 and s["gate_changes"].sum() > 0 and s["completed_int"].sum() > 0


def test_prio_with_function_mode_jsq_and_controller():
    # config-3 DAG (routing over 2 instances, SLO batch control) with classes and priority service
    p, g = W.config3(n_seeds=2, n_requests=200)
    g["arrivals"] = [[W.with_classes(a, 250) for a in row] for row in g["arrivals"]]
    g["candidates"] = [W.with_prio(c, True, k % 2 == 1, (300, 700)) for k, c in enumerate(g["candidates"][:6])]
    full_check(p, g, objective="p99_e2e_int")


def test_prio_gate_window_series_and_stepwise():
    p, g = W.config_prio(n_seeds=2, n_requests=300, gaps=(399400,))
    g.update(series_stride=3, series_slots=6, series_windows=40)
    full_check(p, g, series=True)
    a = run_gpu(p, g, series=True)
    b = run_gpu(p, g, series=True, stepwise=True)
    assert a["summary"].tobytes() == b["summary"].tobytes()


# ------------------------------------------------------------------ f4: data-plane pacing (M30)
def test_pacing_spec_example_trace():
    p = W.toy_ht("batch")
    p["links"][0].update(net=1, pacing_gap=5)
    g = W.grid([W.static("batch")], [W.arr_list([0, 0], prompt=(4, 4), output=(1, 1))], n_requests=2)
    full_check(p, g)
    gg = run_gpu(p, g, trace_replica=0)
    assert first_divergence(sorted_trace(gg["trace"]), sorted_trace(oracle.simulate(p, g, trace_id=0)["trace"])) is None


@pytest.mark.parametrize("svc", ["det", "exp"])
def test_paced_tandem(svc):
    p = W.tandem(60000, 70000, 1000, svc=svc)
    p["links"][0]["pacing_gap"] = 90000
    g = W.grid([W.static("batch"), W.with_pacing(W.static("batch"), 50000), W.with_pacing(W.static("batch"), 0)],
               [W.poisson(100000, output=(0, 0))], n_seeds=9, n_requests=700)
    full_check(p, g)


def test_config_pace_grid():
    p, g = W.config_pace(n_seeds=3, n_requests=300)
    gg, o = full_check(p, g, objective="p99_e2e")
    a = run_gpu(p, g)
    b = run_gpu(p, g, stepwise=True)
    assert a["summary"].tobytes() == b["summary"].tobytes()


def test_pacing_with_fanout_routing_and_classes():
    # config-3 DAG: fan-out (MAXOUT 2), JSQ over two instances, paced links, and request classes
    p, g = W.config3(n_seeds=2, n_requests=200)
    for k, L in enumerate(p["links"]):
        L["pacing_gap"] = 3000 * (k + 1)
    g["arrivals"] = [[W.with_classes(a, 300) for a in row] for row in g["arrivals"]]
    g["candidates"] = [W.with_prio(c, k % 2 == 0) for k, c in enumerate(g["candidates"][:6])]
    full_check(p, g)


# ------------------------------------------------------------------ f4: snapshot (stale) JSQ routing (M31)
def _fanout2(window=400_000):
    dev = W.role("dev", c=W.cost(h=0), max_num_seqs=8, n_functions=2)
    tester = W.role("tester", 2, W.cost(h=2000), max_num_seqs=4, out=(0, 1, 1), route="jsq")
    return W.pipeline([dev, tester], [W.link(0, 1, net=500, chunk=8, mode="function")], window=window)


def test_stale_jsq_trace_and_grid():
    p = _fanout2()
    g = W.grid([W.with_stale_jsq(W.static(m)) for m in ("function", "token", "batch")] + [W.static("function")],
               [W.poisson(150_000, output=(32, 64)), W.poisson(90_000, output=(16, 64))], n_seeds=4,
               n_requests=300)
    full_check(p, g, series=False)
    gg = run_gpu(p, g, trace_replica=0)
    assert first_divergence(sorted_trace(gg["trace"]), sorted_trace(oracle.simulate(p, g, trace_id=0)["trace"])) is None


def test_stale_jsq_config3_with_controller_and_stepwise():
    # config-3 DAG (JSQ coder x 2, tester x 2) with stale JSQ on every other candidate
    p, g = W.config3(n_seeds=2, n_requests=250)
    g["candidates"] = [W.with_stale_jsq(c, k % 2 == 0) for k, c in enumerate(g["candidates"])]
    full_check(p, g, objective="p99_e2e")
    a = run_gpu(p, g)
    b = run_gpu(p, g, stepwise=True)
    assert a["summary"].tobytes() == b["summary"].tobytes()


# ------------------------------------------------------------------ K1 specialisation levels
def _same_results(a, b, series):
    assert a["summary"].tobytes() == b["summary"].tobytes()
    compare_records(a["records"], b["records"], a["summary"])   # slots past `completed` are never written
    if series:
        assert a["series"].tobytes() == b["series"].tobytes()
    for x, y in zip(a["cells"], b["cells"]):
        assert x.tobytes() == y.tobytes()


@pytest.mark.parametrize("cfg", ["config1", "config2", "config5", "tools", "truncated_mmpp"])
def test_lean_kernel_equals_generic(cfg):
    if cfg == "config1":
        p, g = W.config1(n_seeds=2, n_requests=400)
    elif cfg == "truncated_mmpp":               # MMPP-2 arrivals and max_ticks truncation on LEAN
        p = W.p2_x()
        g = W.grid([W.static("token"), W.static("batch"), W.adaptive(["function"], dwell=2)],
                   [W.mmpp2(900_000, 200_000, 20_000_000, 8_000_000)], n_seeds=6, n_requests=300,
                   max_ticks=160_000_000)
    elif cfg == "config2":
        p, g = W.config2(n_seeds=2, n_requests=300, series_stride=7, series_windows=64)
    elif cfg == "config5":
        p, g = W.config5(n_seeds=1, n_requests=200, n_rates=8, n_candidates=64)
    else:
        p = W.tandem(60000, 70000, 1000, svc="exp")
        g = W.grid([W.static("batch"), W.static("token")], [W.poisson(100000, output=(0, 0))], n_seeds=5,
                   n_requests=400)
    series = cfg == "config2"
    a = run_gpu(p, g, series=series)
    assert a["res"].layout.k1_variant == (0 if cfg == "truncated_mmpp" else 2)   # levels >= 1 never truncate
    b = run_gpu(p, g, series=series, generic=True)
    assert b["res"].layout.k1_variant == 0
    m = run_gpu(p, g, series=series, mid=True)
    assert m["res"].layout.k1_variant == (0 if cfg == "truncated_mmpp" else 1)
    _same_results(a, b, series)
    _same_results(m, b, series)
    o = oracle.simulate(p, g, series=series)
    compare_summaries(a["summary"], o["summary"])
    compare_records(a["records"], o["records"], a["summary"])


@pytest.mark.parametrize("cfg", ["config3", "fanout_stale", "config4_select"])
def test_mid_kernel_equals_generic(cfg):
    # routed / model-selecting pipelines without KV / pacing / classes / truncation run the level-1 kernel
    if cfg == "config3":
        p, g = W.config3(n_seeds=2, n_requests=250)
    elif cfg == "config4_select":
        cands = W.config4_candidates()
        p, g = W.config4(n_seeds=2, n_requests=250, candidates=cands[::1024] + cands[7::1531])
    else:
        p, g = W.config3(n_seeds=2, n_requests=200)
        g["candidates"] = [W.with_stale_jsq(c, k % 3 == 0) for k, c in enumerate(g["candidates"])]
    a = run_gpu(p, g)
    assert a["res"].layout.k1_variant == 1
    b = run_gpu(p, g, generic=True)
    assert b["res"].layout.k1_variant == 0
    _same_results(a, b, False)
    o = oracle.simulate(p, g)
    compare_summaries(a["summary"], o["summary"])
    compare_records(a["records"], o["records"], a["summary"])
