"""Edge cases of the hot path on the GPU, bit-exact against the oracle (both K1 levels that apply):
the smallest grid (one replica, one request), request_cap 1 (every concurrent arrival dropped), rings
so small that replicas overflow in every mode (R-OVF: status, overflow tick and id only), a replica
count that leaves a ragged last wave, zero-token outputs everywhere, and simultaneous arrivals."""
import numpy as np
import pytest

import oracle
import workloads as W
from gpu_parity import compare_records, compare_summaries, full_check, run_gpu

pytestmark = pytest.mark.gpu


def _both_levels(p, g):
    gg, o = full_check(p, g)
    b = run_gpu(p, g, generic=True)
    assert gg["summary"].tobytes() == b["summary"].tobytes()
    return gg, o


def test_single_replica_single_request():
    p = W.p2_x()
    g = W.grid([W.static("token")], [W.poisson(500_000)], n_seeds=1, n_requests=1)
    gg, o = _both_levels(p, g)
    s = gg["summary"][0]
    assert int(s["completed"]) == 1 and int(s["p50_e2e"]) == int(s["p99_e2e"]) == int(s["max_e2e"])


def test_request_cap_one_drops():
    p = W.p2_x()
    p["request_cap"] = 1
    g = W.grid([W.static(m) for m in ("batch", "function", "token")], [W.poisson(200_000), W.poisson(2_000_000)],
               n_seeds=3, n_requests=150)
    gg, o = _both_levels(p, g)
    s = gg["summary"]
    assert (s["dropped"] > 0).any() and (s["completed"] + s["dropped"] == 150).all()


@pytest.mark.parametrize("ring", ["inbox", "flight", "wait"])
def test_tiny_rings_overflow(ring):
    p = W.p2_x()
    cap = {"inbox": ("inbox_cap", 2), "flight": ("flight_cap", 2), "wait": ("wait_cap", 2)}[ring]
    p["roles"][1][cap[0]] = cap[1]
    g = W.grid([W.static(m) for m in ("batch", "function", "token")] + [W.adaptive(["function"])],
               [W.poisson(300_000), W.poisson(3_000_000)], n_seeds=3, n_requests=120)
    gg, o = _both_levels(p, g)
    assert (gg["summary"]["status"] == 1).any()          # some replicas overflowed ...
    assert (gg["summary"]["status"] == 0).any() or ring == "flight"


def test_ragged_last_wave():
    # 3 x 1 x 1 x 997 = 2991 replicas: not a multiple of any resident-warp count
    p, g = W.config1(n_seeds=997, n_requests=40, rates=[3])
    _both_levels(p, g)


def test_zero_token_outputs_and_simultaneous_arrivals():
    p = W.p2_spec(mode="function", chunk=4, n_functions=3)
    g = W.grid([W.static(m) for m in ("batch", "function", "token")],
               [W.arr_list([0] * 5 + [10, 10, 10, 500_000] + [600_000] * 7, prompt=(1, 9), output=(0, 3))],
               n_seeds=2, n_requests=16)
    gg, o = _both_levels(p, g)
    assert (gg["summary"]["completed"] > 0).all()
