"""Pins for the oracle's simulation model (rules M4-M16, M19).

Expected values come from: SURVEY.md hand traces HT-0..HT-3, HT-8, HT-9
(tests/golden/), textbook recursions (Lindley, tandem queue) evaluated here in
plain Python, closed-form queueing results (Pollaczek-Khinchine), Little's law
and conservation identities.
"""
import json
import math
import os

import numpy as np
import pytest

import workloads as W

GOLD = os.path.join(os.path.dirname(__file__), "golden")
HT = json.load(open(os.path.join(GOLD, "ht_traces.json")))
RNG = json.load(open(os.path.join(GOLD, "ht8_rng.json")))


def des_events(s):
    return int(s["arrivals"]) + int(s["deliveries"]) + int(s["recv_steps"]) + int(s["decode_steps"]) + int(
        s["window_closes"])


# ------------------------------------------------------------------ HT-8 arrivals (M2-M5)
def test_ht8_poisson_and_crn(orc):
    for s in (0, 1):
        want = RNG["poisson_M399400_s%d" % s]
        t, pr, _ = orc.arrivals(W.poisson(399400), s, 5)
        assert t.tolist() == want["A"] and pr.tolist() == want["P"]
    t, _, _ = orc.arrivals(W.poisson(3994000), 0, 1)
    assert int(t[0]) == RNG["poisson_M3994000_s0_j0"]   # common random numbers across rates


def test_ht8_mmpp_epoch_crossing(orc):
    m = RNG["mmpp2"]
    t, _, _ = orc.arrivals(W.mmpp2(*m["gap"], *m["sojourn"]), m["s"], 120)
    assert t[:3].tolist() == m["A_0_2"]
    assert t[62:66].tolist() == m["A_62_65"]


def test_poisson_count_spec122(orc):
    # rate 10/s for 100 s -> count in [850, 1150]; mean over 100 seeds within 2 %
    counts = []
    for s in range(100):
        t, _, _ = orc.arrivals(W.poisson(100000), s, 1400)
        c = int((t <= 100_000_000).sum())
        assert 850 <= c <= 1150
        counts.append(c)
    assert abs(np.mean(counts) / 1000 - 1) < 0.02


# ------------------------------------------------------------------ HT-0
@pytest.mark.parametrize("mode", ["token", "function", "batch"])
def test_ht0_spec_trace(orc, mode):
    want = HT["HT0"][mode]
    p = W.p2_spec(mode=mode, chunk=16, n_functions=2)
    g = W.grid([W.static(mode)], [W.arr_list([0], prompt=(100, 100), output=(32, 32))], n_requests=1)
    r = orc.simulate(p, g, trace_id=0)
    s = r["summary"][0]
    assert s["status"] == 0 and s["completed"] == 1
    assert int(s["p50_e2e"]) == want["e2e"] and int(s["p50_ff"]) == want["ff"]
    assert des_events(s) == want["des_events"]
    tr = r["trace"]
    deliv = sorted(int(x["tick"]) for x in tr if x["code"] == 7)
    assert deliv == want["deliveries"]   # 267 ms first chunk / 523 ms batch


# ------------------------------------------------------------------ HT-1..HT-3
@pytest.mark.parametrize("mode", ["batch", "function", "token"])
def test_ht13_contention(orc, mode):
    want = HT["HT13"][mode]
    inv = HT["HT13"]["_invariants"]
    p = W.toy_ht(mode)
    g = W.grid([W.static(mode)], [W.arr_list([0, 3])], n_requests=2, series_stride=1, series_slots=1,
               series_windows=1)
    r = orc.simulate(p, g, series=True)
    s = r["summary"][0]
    assert r["records"][0, :, 0].tolist() == want["e2e"]
    assert r["records"][0, :, 1].tolist() == want["ff"]
    assert des_events(s) == want["des_events"]
    assert int(s["arrivals"]) + int(s["deliveries"]) == want["msg_events"]
    assert int(s["int_nsys"]) == want["int_nsys"] == int(s["sum_e2e"])   # Little's law
    ser = r["series"][0, 0]
    assert int(ser[0]["busy"]) == inv["dev_busy"] and int(ser[1]["busy"]) == want["tester_busy"]
    assert int(s["tokens"]) == inv["dev_tokens"] + inv["tester_tokens"]


# ------------------------------------------------------------------ HT-5 sequential JSQ
def test_ht5_two_openings_same_tick(orc):
    # two requests admitted together to one dev batch emit BATCH messages in the same DECODE
    # completion; the tester role has 2 idle instances: first -> A, second -> B (in-flight counts)
    p = W.p2_spec(mode="batch")
    p["roles"][1]["n_instances"] = 2
    g = W.grid([W.static("batch")], [W.arr_list([0, 0], prompt=(10, 10), output=(8, 8))], n_requests=2)
    r = orc.simulate(p, g, trace_id=0)
    emits = [x for x in r["trace"] if x["code"] == 6]
    assert len(emits) == 2 and emits[0]["tick"] == emits[1]["tick"]
    assert [int(e["a"]) for e in emits] == [1, 2]
    assert [int(e["b"]) for e in emits] == [0, 1]


# ------------------------------------------------------------------ HT-6 exact recursions
def _svc(orc, j, s, role, ordinal, mean):
    w = orc.philox([j, s, (3 << 16) | role, ordinal], [W.MASTER_SEED & 0xFFFFFFFF, W.MASTER_SEED >> 32])
    return max(1, orc.exp_sample(mean, w[0]))


@pytest.mark.parametrize("svc", ["det", "exp"])
def test_lindley_single_tool(orc, svc):
    N, S, M = 3000, 70000, 100000
    p = W.tool1(S, svc=svc)
    g = W.grid([W.static()], [W.poisson(M, output=(0, 0))], n_seeds=3, n_requests=N)
    r = orc.simulate(p, g)
    for x in range(3):
        A, _, _ = orc.arrivals(W.poisson(M, output=(0, 0)), x, N)
        C_prev, e2e = 0, []
        for j in range(N):
            Sj = S if svc == "det" else _svc(orc, j, x, 0, 0, S)
            C_prev = max(int(A[j]), C_prev) + Sj          # Lindley: C_j = max(A_j, C_{j-1}) + S_j
            e2e.append(C_prev - int(A[j]))
        s = r["summary"][x]
        assert s["dropped"] == 0 and s["completed"] == N
        assert r["records"][x, :, 0].tolist() == e2e
        assert int(s["makespan"]) == C_prev


@pytest.mark.parametrize("svc", ["det", "exp"])
def test_tandem_recursion(orc, svc):
    # C1_j = max(A_j, C1_{j-1}) + S1_j ;  C2_j = max(C1_j + d, C2_{j-1}) + S2_j   (HT-6)
    N, S1, S2, d, M = 2000, 60000, 70000, 1000, 100000
    p = W.tandem(S1, S2, d, svc=svc)
    g = W.grid([W.static("batch")], [W.poisson(M, output=(0, 0))], n_seeds=2, n_requests=N)
    r = orc.simulate(p, g)
    for x in range(2):
        A, _, _ = orc.arrivals(W.poisson(M, output=(0, 0)), x, N)
        c1 = c2 = 0
        e2e = []
        for j in range(N):
            s1 = S1 if svc == "det" else _svc(orc, j, x, 0, 0, S1)
            s2 = S2 if svc == "det" else _svc(orc, j, x, 1, 1, S2)
            c1 = max(int(A[j]), c1) + s1
            c2 = max(c1 + d, c2) + s2
            e2e.append(c2 - int(A[j]))
        assert r["records"][x, :, 0].tolist() == e2e


def test_tandem_small_example(orc):
    # SURVEY.md HT-6 example: A=(0,2,3,10), S1=4, S2=3, d=1 -> e2e=(8,10,13,10)
    p = W.tandem(4, 3, 1)
    g = W.grid([W.static("batch")], [W.arr_list([0, 2, 3, 10], prompt=(0, 0), output=(0, 0))], n_requests=4)
    r = orc.simulate(p, g)
    assert r["records"][0, :, 0].tolist() == [8, 10, 13, 10]


# ------------------------------------------------------------------ statistics (P-K)
def _mean_wait(orc, p, g, S_mean):
    r = orc.simulate(p, g, records=False, hists=False)
    s = r["summary"]
    assert (s["dropped"] == 0).all()
    return (s["sum_e2e"].astype(np.float64).sum() / s["completed"].sum()) - S_mean


def test_md1_mean_wait(orc):
    S, M = 100000, 200000
    g = W.grid([W.static()], [W.poisson(M, output=(0, 0))], n_seeds=8, n_requests=100000)
    wq = _mean_wait(orc, W.tool1(S), g, S)
    lam = 1.0 / (M - 0.5)                  # effective mean gap (floor bias)
    rho = lam * S
    assert abs(wq / (rho * S / (2 * (1 - rho))) - 1) < 0.015


def test_mm1_mean_wait(orc):
    S, M = 100000, 200000
    g = W.grid([W.static()], [W.poisson(M, output=(0, 0))], n_seeds=16, n_requests=100000)
    r = orc.simulate(W.tool1(S, svc="exp"), g, records=False, hists=False)
    s = r["summary"]
    ES = S - 0.5                            # floor bias of the service draw
    lam = 1.0 / (M - 0.5)
    rho = lam * ES
    mean_e2e = s["sum_e2e"].astype(np.float64).sum() / s["completed"].sum()
    assert abs((mean_e2e - ES) / (rho * ES / (1 - rho)) - 1) < 0.04


def test_mg1_mean_wait(orc):
    # S = alpha + beta P, P ~ U[64,256]: E[S]=13000, E[S^2]=1.7676e8 (SURVEY c.5)
    for M, want in ((26000, 6798.46), (16250, 27193.85)):
        p = W.tool1(5000, beta=50)
        g = W.grid([W.static()], [W.poisson(M, prompt=(64, 256), output=(0, 0))], n_seeds=8, n_requests=100000)
        wq = _mean_wait(orc, p, g, 13000)
        tol = 0.02 if M == 26000 else 0.05
        assert abs(wq / want - 1) < tol, (M, wq, want)


# ------------------------------------------------------------------ identities
@pytest.mark.parametrize("mode", ["batch", "function", "token"])
def test_little_and_conservation(orc, mode):
    p = W.p2_x(mode=mode)
    g = W.grid([W.static(mode)], [W.poisson(m) for m in (3994000, 998500, 570571)], n_seeds=2, n_requests=800)
    r = orc.simulate(p, g)
    per_item = {"batch": 1, "function": 4, "token": 32}[mode]
    for x, s in enumerate(r["summary"]):
        if s["status"] != 0:
            continue
        assert s["admitted"] + s["dropped"] == 800
        assert s["completed"] == s["admitted"]
        assert int(s["int_nsys"]) == int(s["sum_e2e"])                    # Little's law, exact
        assert s["msgs_emitted"] == s["msgs_received"] == s["deliveries"]
        assert s["tokens_emitted"] == s["tokens_received"] == 128 * s["completed"]
        assert s["msgs_emitted"] == per_item * s["completed"]             # BATCH 1, FUNCTION F, TOKEN ceil(out/c)
        assert s["tokens"] == 256 * s["completed"]                        # dev 128 + tester out = n_in
        e2e = r["records"][x, : s["completed"], 0]
        ff = r["records"][x, : s["completed"], 1]
        assert (ff <= e2e).all()


def test_ht9_window_accounting(orc):
    # four arrivals at 990000 to a tool with a 15000-tick service; W = 1e6
    p = W.tool1(15000)
    g = W.grid([W.static()], [W.arr_list([990000] * 4, prompt=(0, 0), output=(0, 0))], n_requests=4,
               series_stride=1, series_slots=1, series_windows=3)
    r = orc.simulate(p, g, series=True)
    s = r["summary"][0]
    ser = r["series"][0]
    assert s["window_closes"] == 1 and s["makespan"] == 1050000
    assert [int(ser[k, 0]["busy"]) for k in range(2)] == [10000, 50000]
    assert [int(ser[k, 0]["qint"]) for k in range(2)] == [30000, 3 * 5000 + 2 * 15000 + 1 * 15000]
    assert [int(ser[k, 0]["maxq"]) for k in range(2)] == [3, 3]
    # a step [999000, 1015000) splits 1000 / 15000 across the boundary
    g2 = W.grid([W.static()], [W.arr_list([999000], prompt=(0, 0), output=(0, 0))], n_requests=1,
                series_stride=1, series_slots=1, series_windows=2)
    r2 = orc.simulate(W.tool1(16000), g2, series=True)
    assert [int(r2["series"][0, k, 0]["busy"]) for k in range(2)] == [1000, 15000]


def test_overflow_is_deterministic_and_zeroed(orc):
    p = W.p2_x(mode="token")
    g = W.grid([W.static("token")], [W.poisson(399400)], n_seeds=2, n_requests=3000)
    a = orc.simulate(p, g)
    b = orc.simulate(p, g, threads=1)
    for x in range(2):
        assert a["summary"][x]["status"] == 1 and a["summary"][x]["completed"] == 0
        assert a["summary"][x].tobytes() == b["summary"][x].tobytes()
        assert a["hists"][x].sum() == 0


def test_determinism_and_thread_independence(orc):
    p, g = W.config1(n_seeds=2, n_requests=600, rates=[0, 4, 7])
    a = orc.simulate(p, g, threads=1)
    b = orc.simulate(p, g, threads=5)
    assert a["summary"].tobytes() == b["summary"].tobytes()
    assert a["records"].tobytes() == b["records"].tobytes()
