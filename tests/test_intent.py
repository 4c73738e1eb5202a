"""f3 host logic: sdas_compile_intent (SPEC.md:432-436 Intent, 475-483 compile_intent;
PAPER.md:63, 188, 220).  CPU only: compilation is host code behind the C-ABI (no GPU call)."""
import pytest

import workloads as W
from paper_2601_03197_b200 import sdas


def _pipe(window=1_000_000, n_links=1):
    if n_links == 1:
        p = W.p2_x()
    else:
        p, _ = W.config3(n_seeds=1, n_requests=10)
    p["window"] = window
    return sdas.Pipeline(p)


def test_max_throughput_one_link_is_the_three_band_template():
    # SPEC.md:482 "objective max_throughput, 1 link -> 3 rules (hi-band, lo-band, mid-band) on comm_mode";
    # SPEC.md:479 ">= 0.8 -> batch_all; <= 0.4 -> token_stream(16); otherwise per_function; dwell 1000 ms"
    c, obj = sdas.compile_intent(_pipe(), "max_throughput")
    assert obj == "throughput"
    assert c["kind"] == "adaptive" and c["ctl_links"] == [0] and c["metric"] == "busy"
    assert (c["lo"], c["hi"]) == (400, 800)
    assert c["band"] == ["token", "function", "batch"]        # low / mid / high band
    assert c["dwell"] == 1                                    # 1000 ms at W = 1 s
    assert c["guard_links"] == []


def test_dwell_is_one_second_in_windows():
    c, _ = sdas.compile_intent(_pipe(window=250_000), "max_throughput")
    assert c["dwell"] == 4
    c, _ = sdas.compile_intent(_pipe(window=300_000), "max_throughput")
    assert c["dwell"] == 4                                    # ceil(1e6 / 3e5)


def test_every_link_is_controlled():
    c, _ = sdas.compile_intent(_pipe(n_links=3), "max_throughput")
    assert c["ctl_links"] == [0, 1, 2]


def test_min_p90_streams_everywhere():
    c, obj = sdas.compile_intent(_pipe(n_links=3), "min_p90_latency")
    assert obj == "p90_e2e" and c["kind"] == "static"
    assert c["modes"] == ["token"] * 3 and c["ctl_links"] == []


def test_constraint_becomes_one_p90_guard():
    # SPEC.md:483 'constraint "e2e_latency_p90_ms <= 2000, scope interactive" -> one guard rule referencing
    # p90 aggregation' (the scope here is a set of links; priority classes are f2)
    c, obj = sdas.compile_intent(_pipe(), "min_p90_latency", constraints=[("e2e_p90", 2_000_000, [])])
    assert obj == "p90_e2e"
    assert c["kind"] == "adaptive" and c["guard_links"] == [0] and c["guard_pct"] == 90
    assert c["policy_slo"] == 2_000_000 and c["modes"] == ["token"] and c["ctl_links"] == []
    c, _ = sdas.compile_intent(_pipe(n_links=3), "max_throughput", constraints=[("e2e_p99", 5_000_000, [1])])
    assert c["guard_links"] == [1] and c["guard_pct"] == 99 and c["ctl_links"] == [0, 1, 2]


def test_explicit_rules_pass_through_unchanged():
    rules = W.adaptive(["function"], ctl_links=[0], lo=300, hi=900, dwell=3, batch_roles=[1], q_hi=5,
                       policy_slo=7_000_000)
    c, obj = sdas.compile_intent(_pipe(), rules=rules)
    assert obj == "p99_e2e"
    for k in ("kind", "modes", "ctl_links", "lo", "hi", "dwell", "band", "batch_roles", "q_hi", "policy_slo"):
        assert c[k] == rules[k], k


def test_empty_intent_is_invalid():
    with pytest.raises(sdas.SdasError) as e:
        sdas.compile_intent(_pipe())
    assert e.value.code == sdas.E_INVALID_ARG and "InvalidIntent" in str(e.value)


def test_one_bound_per_policy():
    with pytest.raises(sdas.SdasError) as e:
        sdas.compile_intent(_pipe(), "min_p90_latency",
                            constraints=[("e2e_p90", 2_000_000, []), ("e2e_p90", 3_000_000, [])])
    assert e.value.code == sdas.E_LIMIT
    c, _ = sdas.compile_intent(_pipe(n_links=3), "min_p90_latency",
                               constraints=[("e2e_p90", 2_000_000, [0]), ("e2e_p90", 2_000_000, [2])])
    assert c["guard_links"] == [0, 2]
    with pytest.raises(sdas.SdasError) as e:   # the rules' batch controller already uses another SLO
        sdas.compile_intent(_pipe(), rules=W.adaptive(["batch"], batch_roles=[1], policy_slo=1),
                            constraints=[("e2e_p90", 2_000_000, [])])
    assert e.value.code == sdas.E_LIMIT


def test_bad_enums():
    with pytest.raises(sdas.SdasError):
        sdas.compile_intent(_pipe(), "min_p90_latency", constraints=[("e2e_p90", 1, [3])])   # no link 3


def test_compiled_candidates_validate_in_a_grid():
    p = W.p2_x()
    P = sdas.Pipeline(p)
    cands = [sdas.compile_intent(P, o, constraints=k)[0] for o in ("max_throughput", "min_p90_latency")
             for k in ([], [("e2e_p90", 3_000_000, [])])]
    g = W.grid(cands, [W.poisson(m) for m in (998500, 570571)], n_seeds=2, n_requests=50)
    L = sdas.results_layout(P, sdas.GridView(p, g))
    assert L.n_replicas == 16
