"""Pins for the f1 extension (rules M21-M24): KV-cache transfer with controller hints and load
balancing (Fig. 6).  Expected values: tests/golden/ht_kv.json
(hand-derived), SPEC.md:291-302 lead-time arithmetic, the skewed-home composition of pinned
samplers, and the paper's direction (hints > post-hoc > no hooks; load balancing >> affinity)."""
import json
import os

import numpy as np
import pytest

import workloads as W

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "ht_kv.json")))


def _one_request(kv, net=1000, ctx=4000):
    p = W.p2_kv(ctx_tokens=ctx, home_skew=1000)          # every request's KV lives on tester 0
    p["roles"][1]["route"] = "fixed"
    p["roles"][1]["route_fixed"] = 1                     # ... and the router sends it to tester 1
    p["links"][0]["net"] = net
    g = W.grid([W.with_kv(W.static("batch"), kv)], [W.arr_list([0], prompt=(100, 100), output=(32, 32))],
               n_requests=1)
    return p, g


@pytest.mark.parametrize("kv", ["off", "affinity", "recompute", "posthoc", "hint"])
def test_kv_single_request_hand_trace(orc, kv):
    want = GOLD["single_request_fixed_to_tester1"][kv]
    p, g = _one_request(kv)
    s = orc.simulate(p, g)["summary"][0]
    assert s["status"] == 0
    assert int(s["p50_e2e"]) == want["e2e"] and int(s["p50_ff"]) == want["ff"]
    assert int(s["kv_transfers"]) == want["kv_transfers"]


def test_kv_hint_lead_spec_arithmetic(orc):
    # hint lead >= transfer -> no wait; lead 5 ms vs transfer 20 ms -> 15 ms; post-hoc 20 ms
    base = {}
    for net in (1000, 5000, 100000):
        p, g = _one_request("off", net=net, ctx=1000)
        base[net] = int(orc.simulate(p, g)["summary"][0]["p50_e2e"])
        p, g = _one_request("hint", net=net, ctx=1000)
        hint = int(orc.simulate(p, g)["summary"][0]["p50_e2e"])
        assert hint - base[net] == GOLD["hint_lead_ctx1000"]["_net_ticks_to_wait"][str(net)]
    p, g = _one_request("posthoc", net=1000, ctx=1000)
    assert int(orc.simulate(p, g)["summary"][0]["p50_e2e"]) - base[1000] == GOLD["hint_lead_ctx1000"]["posthoc_wait"]


def test_kv_home_skew_fraction(orc):
    # home = tester 0 with prob skew + (1 - skew)/2 (M21: BER(skew) then UNI over 2 testers)
    p = W.p2_kv(home_skew=600)
    p["roles"][1]["route"] = "fixed"
    p["roles"][1]["route_fixed"] = 1
    g = W.grid([W.with_kv(W.static("batch"), "posthoc")], [W.poisson(2_000_000)], n_seeds=8, n_requests=2000)
    s = orc.simulate(p, g, records=False)["summary"]
    frac = s["kv_transfers"].astype(np.int64).sum() / s["completed"].astype(np.int64).sum()
    assert abs(frac - (0.6 + 0.4 / 2)) < 0.015


def test_kv_directional_fig6(orc):
    # hints beat post-hoc transfer and no load balancing at high load
    p, g = W.config_kv(n_seeds=4, n_requests=1200, gaps=(240000, 210000))
    s = orc.simulate(p, g, records=False)["summary"]
    C, S = 4, 4
    for i in range(2):
        gp = []
        for c in range(C):
            xs = [s[(i * S + k) * C + c] for k in range(S)]
            gp.append(np.mean([x["good"] * 1e6 / x["makespan"] for x in xs]))
        aff, rec, post, hint = gp
        assert hint > post > rec and hint > 1.5 * aff, gp
