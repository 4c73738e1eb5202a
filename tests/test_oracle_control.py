"""Pins for the oracle's controller and routing rules that configs 3-5 rank by (rules M11, M14, M16(ii),
M16(iii), M15 LOAD metric, max_ticks truncation, R-OVF, R-SAT).

Every expected value below is derived by hand from the rule's statement, with the derivation in the
comments: toy pipelines with unit-cost RECV steps, constant DECODE steps and explicit (LIST) arrival
ticks make every timeline short enough to write out.  None of the expectations is computed by code that
re-implements the rule.

Rules pinned (statements from DESIGN.md §2 / SURVEY.md §8(c) M16):
  * M16(ii) SLO batch size (PAPER.md:217 `set('max_num_seqs', 4)`): at the close of a window with n >= 1
    completions, viol <=> #(e2e <= slo) < ceil(0.99 n), calm <=> #(2 e2e <= slo) >= ceil(0.99 n);
    viol -> B <- min(32, 2B) if the instance's integral Q dt > q_hi * W else max(1, B/2); calm -> reset
    to the default; dwell D and no-op suppression.
  * M16(iii) model selection: SMALL iff 1000 busy(selected) >= hi W or viol; LARGE iff
    1000 busy(selected) <= lo W and not viol; dwell and no-op suppression.
  * M11 RR: the k-th opening message into a role goes to instance
    k mod n (per-role counter); a candidate's route override replaces JSQ/RR, never FIXED/SELECT.
  * M15/M16(i) LOAD metric: the band decision uses the integral of L = in-flight + inbox + [RECV] + wait
    + batch over the destination's instances instead of busy time.
  * M1/M12 truncation: events at ticks <= max_ticks are processed; the replica stops before the first
    event tick > max_ticks, with status TRUNCATED and makespan = the last processed tick.
  * M14 + R-OVF: a push into a full inbox / wait / in-flight ring sets OVERFLOW at that tick; only the
    status, the overflow tick and the replica id are reported.
  * M18/M19 + R-SAT: record fields saturate at 2^32-1; a record holding the sentinel counts as saturated;
    the sums stay exact.
"""
import pytest

import oracle
import workloads as W

TR_EMIT = 6


@pytest.fixture(scope="module")
def orc():
    return oracle


def srv(n_instances=1, B=4, tau0=100, alpha=1, inst_cost=None, route="jsq", caps=64):
    """A one-role pipeline: RECV costs alpha (h = beta = 0), DECODE costs tau0 (gamma = 0), out = O_j."""
    r = W.role("srv", n_instances, W.cost(h=0, alpha=alpha, beta=0, tau0=tau0, gamma=0), inst_cost=inst_cost,
               max_num_seqs=B, route=route, inbox_cap=caps, wait_cap=caps, flight_cap=caps)
    return W.pipeline([r], [], feedback_role=0, request_cap=caps, window=1000)


def bursts(ks, W_=1000):
    """k_w requests at the start tick of window w."""
    return [w * W_ for w, k in enumerate(ks) for _ in range(k)]


def batch_cand(slo, q_hi=1, dwell=1):
    c = W.adaptive([], ctl_links=[], batch_roles=[0], q_hi=q_hi, policy_slo=slo, dwell=dwell)
    return c


def run(orc, p, cand, ticks, n_windows=0, **kw):
    g = W.grid([cand], [W.arr_list(ticks, prompt=(1, 1), output=(1, 1))], n_requests=len(ticks),
               series_stride=1 if n_windows else 0, series_slots=1 if n_windows else 0,
               series_windows=n_windows, **kw)
    return orc.simulate(p, g, series=bool(n_windows), trace_id=0)


# ------------------------------------------------------------------ M16(ii) SLO-aware batch size
# One instance, RECV 1 tick, DECODE 100 ticks (gamma = 0), out = 1 token: a burst of k requests at a
# window start T0 is received in k ticks (Q = inbox + wait = k-1 throughout), then decoded in waves of B:
# wave m (1-based) completes at T0 + k + 100 m, so e2e = k + 100 m.  Integral Q over the window =
# k(k-1) + 100 * sum_m max(0, k - m B).  W = 1000, q_hi = 1 (threshold 1000), policy slo = 250.
KS = [8, 12, 12, 20, 2, 9, 1, 0, 1, 1]


def _waves(k, B):
    """e2e of a burst of k with batch size B (hand formula above), in completion order."""
    return [k + 100 * (1 + i // B) for i in range(k)]


def test_batch_control_sequence(orc):
    # window: k, B in force -> e2e waves, integral Q, decision at the close (q = window + 1)
    # w0: 8, B=4 -> 108 x4, 208 x4; Q = 56 + 400 = 456;  max 208 <= 250 no viol; #(<=125) = 4 < 8 not calm
    # w1: 12, B=4 -> 112/212/312 x4; Q = 132 + 800 + 400 = 1332; #(<=250) = 8 < ceil(11.88) = 12 viol;
    #     1332 > 1000 -> B = min(32, 8) = 8 at q = 2
    # w2: 12, B=8 -> 112 x8, 212 x4; Q = 132 + 400 = 532; no viol, #(<=125) = 8 < 12 not calm -> stay 8
    # w3: 20, B=8 -> 120 x8, 220 x8, 320 x4; Q = 380 + 1200 + 400 = 1980; #(<=250) = 16 < 20 viol;
    #     1980 > 1000 -> B = 16 at q = 4
    # w4: 2, B=16 -> 102 x2; Q = 2; no viol; #(<=125) = 2 >= ceil(1.98) = 2 calm -> reset to 4 at q = 5
    # w5: 9, B=4 -> 109 x4, 209 x4, 309; Q = 72 + 500 + 100 = 672; #(<=250) = 8 < ceil(8.91) = 9 viol;
    #     672 <= 1000 -> B = max(1, 2) = 2 at q = 6
    # w6: 1, B=2 -> 101; calm -> reset to 4 at q = 7
    # w7: no completion -> no action;  w8: 1 -> 101, calm but B is the default: no-op;  w9: final partial
    r = run(orc, srv(B=4), batch_cand(250), bursts(KS), n_windows=10)
    s = r["summary"][0]
    Bs = [4, 4, 8, 8, 16, 4, 2, 4, 4, 4]
    assert [int(r["series"][0, w, 0]["B"]) for w in range(10)] == Bs
    assert [int(r["series"][0, w, 0]["qint"]) for w in range(10)] == [456, 1332, 532, 1980, 2, 672, 0, 0, 0, 0]
    assert int(s["batch_changes"]) == 5 and int(s["window_closes"]) == 9
    want = [e for k, B in zip(KS, Bs) for e in _waves(k, B)]
    assert r["records"][0, :, 0].tolist() == want
    assert int(s["makespan"]) == 9101 and int(s["decode_steps"]) == 17 and int(s["recv_steps"]) == 66


def test_batch_control_dwell_two(orc):
    # dwell 2: q=2 double to 8 (q_last 2); q=4 double to 16 (4-2 >= 2); q=5 calm reset wanted but 5-4 < 2:
    # held, so window 5 (k = 9) runs at B = 16: one wave, e2e 109 x9, calm -> reset to 4 at q = 6;
    # q=7 and q=9 calm no-ops
    r = run(orc, srv(B=4), batch_cand(250, dwell=2), bursts(KS), n_windows=10)
    s = r["summary"][0]
    Bs = [4, 4, 8, 8, 16, 16, 4, 4, 4, 4]
    assert [int(r["series"][0, w, 0]["B"]) for w in range(10)] == Bs
    assert int(s["batch_changes"]) == 3
    assert r["records"][0, :, 0].tolist() == [e for k, B in zip(KS, Bs) for e in _waves(k, B)]


@pytest.mark.parametrize("B0,k,q_hi,want_B1,changes", [
    (32, 40, 1, 32, 0),   # viol, Q = 1560 + 800 = 2360 > 1000 -> min(32, 64) = 32: no change
    (1, 3, 1, 1, 0),      # viol, Q = 6 + 300 = 306 <= 1000 -> max(1, 0) = 1: no change
    (1, 3, 0, 2, 1),      # q_hi 0: 306 > 0 -> double to 2
])
def test_batch_control_limits(orc, B0, k, q_hi, want_B1, changes):
    # slo 50: every e2e (>= k + 100) violates; one more request in window 1 makes window 0 close
    r = run(orc, srv(B=B0), batch_cand(50, q_hi=q_hi), bursts([k, 1]), n_windows=2)
    s = r["summary"][0]
    assert int(r["series"][0, 1, 0]["B"]) == want_B1 and int(s["batch_changes"]) == changes
    assert r["records"][0, :k, 0].tolist() == _waves(k, B0)


# ------------------------------------------------------------------ M16(iii) model selection
LARGE = dict(W.cost(h=0, alpha=1, beta=0, tau0=399, gamma=0), large=1)   # RECV 1 + DECODE 399 = 400
SMALL = dict(W.cost(h=0, alpha=1, beta=0, tau0=99, gamma=0), large=0)    # 100


def sel_cand(slo, lo=300, hi=700, dwell=1):
    return W.adaptive([], ctl_links=[], lo=lo, hi=hi, dwell=dwell, select_role=0, policy_slo=slo)


def test_model_selection_by_busy(orc):
    # instance 0 LARGE (400 ticks per request), instance 1 SMALL (100); selection starts on LARGE.
    # w0: 0, 400 on L -> busy 800: 800000 >= 700 W -> SMALL at q=1
    # w1: 1000, 1100 on S -> busy(S) 200 <= 300 W, no viol -> LARGE at q=2
    # w2: 2300, 2700 on L -> [2300,2700) + [2700,3000) = 700: 700000 >= 700000 (inclusive) -> SMALL at q=3
    # w3: L finishes [3000,3100) (busy 100, not selected); 3200 on S -> busy(S) 100 <= 300 -> LARGE at q=4
    # w4: 4000, 4400 on L -> 800 -> SMALL at q=5
    # w5: 5000..5600 (7) on S -> busy(S) 700 (busy(L) 0): SMALL = current, no-op
    # w6: 6000 on S -> busy(S) 100 -> LARGE at q=7;  w7: idle, LARGE = current: no-op;  8000 -> L
    ticks = [0, 400, 1000, 1100, 2300, 2700, 3200, 4000, 4400] + [5000 + 100 * i for i in range(7)] + [6000, 8000]
    p = srv(2, inst_cost=[LARGE, SMALL], route="select")
    r = run(orc, p, sel_cand(10 ** 9), ticks, n_windows=9)
    s = r["summary"][0]
    busy = [[int(r["series"][0, w, i]["busy"]) for i in range(2)] for w in range(9)]
    assert busy == [[800, 0], [0, 200], [700, 0], [100, 100], [800, 0], [0, 700], [0, 100], [0, 0], [400, 0]]
    assert int(s["select_changes"]) == 6 and int(s["large_items"]) == 7
    assert r["records"][0, :, 0].tolist() == [400, 400, 100, 100, 400, 400, 100, 400, 400] + [100] * 8 + [400]


@pytest.mark.parametrize("dwell,want,changes", [
    # slo 150, LARGE = 200 ticks: a window with a LARGE completion violates even at busy 200 <= lo
    (1, [200, 100, 200, 100], 3),   # q1 SMALL (viol), q2 LARGE (busy 100, no viol), q3 SMALL (viol)
    (2, [200, 100, 100, 200], 2),   # q2 LARGE held (2-1 < 2); window 2 on SMALL: no viol -> LARGE at q3
])
def test_model_selection_by_violation(orc, dwell, want, changes):
    large = dict(LARGE, tau0=199)
    p = srv(2, inst_cost=[large, SMALL], route="select")
    r = run(orc, p, sel_cand(150, dwell=dwell), [0, 1000, 2000, 3000])
    assert r["records"][0, :, 0].tolist() == want
    assert int(r["summary"][0]["select_changes"]) == changes


# ------------------------------------------------------------------ M11 round robin
def rr_pipe(mode, n=3, route="rr", route_fixed=0):
    gen = W.role("gen", 1, W.cost(h=0, alpha=1, beta=0, tau0=10, gamma=0), n_functions=2)
    rev = W.role("rev", n, W.cost(h=5, alpha=0, beta=0, tau0=1, gamma=0), out=(0, 0, 1), route=route,
                 route_fixed=route_fixed)
    return W.pipeline([gen, rev], [W.link(0, 1, net=1, chunk=1, mode=mode)])


def opening_dests(r):
    return [int(e["a"]) for e in r["trace"] if e["code"] == TR_EMIT and (int(e["c"]) >> 16) & 1]


@pytest.mark.parametrize("mode,per_req", [("function", 2), ("token", 1), ("batch", 1)])
def test_rr_rotates_per_opening(orc, mode, per_req):
    # spaced requests (out = 4 tokens): FUNCTION emits 2 opening messages per request, TOKEN(1) one
    # opening stream (continuations sticky), BATCH one message; the k-th opening goes to instance k mod 3
    g = W.grid([W.static(mode)], [W.arr_list([0, 1000, 2000, 3000], prompt=(1, 1), output=(4, 4))], n_requests=4)
    r = orc.simulate(rr_pipe(mode), g, trace_id=0)
    assert opening_dests(r) == [1 + k % 3 for k in range(4 * per_req)]
    # continuations follow their stream's instance
    emits = [(int(e["b"]), int(e["a"])) for e in r["trace"] if e["code"] == TR_EMIT]
    first = {}
    for j, d in emits:
        first.setdefault(j, d)
    if mode == "token":
        assert all(d == first[j] for j, d in emits)


@pytest.mark.parametrize("role_route,override,want", [
    ("jsq", None, [1, 1, 1, 1]),        # idle instances, loads all 0: JSQ picks the lowest
    ("jsq", "rr", [1, 2, 3, 1]),        # the candidate's override turns JSQ into RR
    ("rr", "jsq", [1, 1, 1, 1]),        # ... and RR into JSQ
    ("fixed", "rr", [3, 3, 3, 3]),      # FIXED (instance 2) is never overridden
])
def test_route_override(orc, role_route, override, want):
    c = W.static("batch")
    c["route"] = override
    g = W.grid([c], [W.arr_list([0, 1000, 2000, 3000], prompt=(1, 1), output=(4, 4))], n_requests=4)
    r = orc.simulate(rr_pipe("batch", route=role_route, route_fixed=2), g, trace_id=0)
    assert opening_dests(r) == want


def test_rr_counter_is_per_role(orc):
    # gen -> A (2 instances, RR) -> B (2 instances, RR): each role's openings rotate over its own
    # instances in its own emission order, whatever the other role did
    gen = W.role("gen", 1, W.cost(h=0, alpha=1, beta=0, tau0=10, gamma=0), n_functions=3)
    A = W.role("A", 2, W.cost(h=3, alpha=1, beta=0, tau0=7, gamma=0), out=(0, 1, 1), route="rr")
    B = W.role("B", 2, W.cost(h=5, alpha=0, beta=0, tau0=1, gamma=0), out=(0, 0, 1), route="rr")
    p = W.pipeline([gen, A, B], [W.link(0, 1, net=1, mode="function"), W.link(1, 2, net=2, mode="batch")])
    g = W.grid([W.static("function", "batch")], [W.arr_list([0, 500, 900], prompt=(1, 1), output=(6, 6))],
               n_requests=3)
    r = orc.simulate(p, g, trace_id=0)
    ev = [e for e in r["trace"] if e["code"] == TR_EMIT and (int(e["c"]) >> 16) & 1]
    to_a = [int(e["a"]) for e in ev if (int(e["c"]) >> 20) == 0]
    to_b = [int(e["a"]) for e in ev if (int(e["c"]) >> 20) == 1]
    assert len(to_a) == 9 and len(to_b) == 9     # 3 requests x 3 functions; one BATCH message per A item
    assert to_a == [1 + k % 2 for k in range(9)] and to_b == [3 + k % 2 for k in range(9)]


# ------------------------------------------------------------------ M16(i) with the LOAD metric
def test_load_metric_band(orc):
    # tool S (100 ticks) -> net 300 -> tool T (200 ticks).  For T, L = in-flight + inbox + [RECV] + wait + batch.
    # w0: request 0: in flight [100, 400), RECV [400, 600): integral L = 500, busy 200
    # w1: requests at 1000 and 1050: S [1000,1100), [1100,1200); in flight [1100,1400), [1200,1500);
    #     T RECV [1400,1600), inbox [1500,1600), RECV [1600,1800): integral L = 600 + 100 + 400 = 1100,
    #     busy 400
    # w2: idle (0, 0);  w3: request at 3000 (final partial window)
    # lo 300 / hi 500 permille, bands TOKEN / FUNCTION / BATCH, initial FUNCTION, dwell 1:
    #   LOAD: 500 >= 500 -> BATCH (q1), 1100 -> BATCH (no-op), 0 -> TOKEN (q3)     modes F, B, B, T
    #   BUSY: 200 <= 300 -> TOKEN (q1), 400 -> FUNCTION (q2), 0 -> TOKEN (q3)       modes F, T, F, T
    S = W.role("S", 1, W.cost(h=0, alpha=100, beta=0, tau0=1, gamma=0))
    T = W.role("T", 1, W.cost(h=0, alpha=200, beta=0, tau0=1, gamma=0), out=(0, 0, 1))
    p = W.pipeline([S, T], [W.link(0, 1, net=300, mode="function")], window=1000)
    M = oracle.MODES
    for metric, modes, switches in (("load", "FBBT", 2), ("busy", "FTFT", 3)):
        c = W.adaptive(["function"], ctl_links=[0], metric=metric, lo=300, hi=500, dwell=1)
        g = W.grid([c], [W.arr_list([0, 1000, 1050, 3000], prompt=(0, 0), output=(0, 0))], n_requests=4,
                   series_stride=1, series_slots=1, series_windows=4)
        r = orc.simulate(p, g, series=True)
        got = [int(r["series"][0, w, 1]["mode"]) for w in range(4)]
        assert got == [M[{"F": "function", "B": "batch", "T": "token"}[x]] for x in modes], metric
        assert int(r["summary"][0]["mode_switches"]) == switches
        assert [int(r["series"][0, w, 1]["busy"]) for w in range(4)] == [200, 400, 0, 200]
        assert r["records"][0, :, 0].tolist() == [600, 1600 - 1000, 1800 - 1050, 600]


# ------------------------------------------------------------------ truncation (max_ticks)
@pytest.mark.parametrize("max_ticks,status,makespan,decode_steps,tokens,int_nsys", [
    (100, 2, 99, 4, 8, 99 + 96),     # last processed tick 99 (tester RECV r1 -> DECODE start); next 113
    (113, 2, 113, 5, 10, 113 + 110),  # 113 processed (tester step 1: first feedback); next 127
    (126, 2, 113, 5, 10, 113 + 110),
    (127, 0, 127, 6, 12, 127 + 124),  # 127 processed: both complete
])
def test_truncation_ht1(orc, max_ticks, status, makespan, decode_steps, tokens, int_nsys):
    # SURVEY HT-1 (BATCH) timeline: dev RECV [0,9), [9,18), DECODE b=2 ends 32, 46, 60, 74 (emit, deliver 75);
    # tester RECV [75,87), [87,99), DECODE [99,113), [113,127)
    g = W.grid([W.static("batch")], [W.arr_list([0, 3])], n_requests=2, max_ticks=max_ticks)
    s = orc.simulate(W.toy_ht("batch"), g)["summary"][0]
    assert int(s["status"]) == status and int(s["makespan"]) == makespan
    assert int(s["decode_steps"]) == decode_steps and int(s["tokens"]) == tokens
    assert int(s["int_nsys"]) == int_nsys
    assert int(s["arrivals"]) == 2 and int(s["deliveries"]) == 2 and int(s["recv_steps"]) == 4
    assert int(s["completed"]) == (2 if status == 0 else 0)
    if status:
        assert int(s["p99_e2e"]) == 0xFFFFFFFF and int(s["sum_e2e"]) == 0


# ------------------------------------------------------------------ M14 overflow tick (R-OVF)
def _ovf(orc, p, ticks, out=(0, 0)):
    g = W.grid([W.static("batch")], [W.arr_list(ticks, prompt=(0, 0), output=out)], n_requests=len(ticks))
    return orc.simulate(p, g)["summary"][0]


@pytest.mark.parametrize("ticks,tick", [([5, 5, 6, 7], 7), ([5, 5, 5, 9], 5)])
def test_overflow_inbox(orc, ticks, tick):
    # inbox cap 2, service 10: at 5 two arrivals fill the inbox, START takes one; the next arrival that
    # finds 2 waiting overflows (tick 7; or at once when a third arrives at 5, before START)
    p = W.tool1(10)
    p["roles"][0]["inbox_cap"] = 2
    s = _ovf(orc, p, ticks)
    assert int(s["status"]) == 1 and int(s["stop_tick"]) == tick
    assert int(s["completed"]) == 0 and int(s["arrivals"]) == 0 and int(s["sum_e2e"]) == 0


def test_overflow_wait_and_flight(orc):
    # wait cap 1: RECV [0,1) puts j0 in wait; RECV-first takes j1 [1,2); its item finds wait full at 2
    p = srv(B=1)
    p["roles"][0]["wait_cap"] = 1
    s = _ovf(orc, p, [0, 0], out=(1, 1))
    assert int(s["status"]) == 1 and int(s["stop_tick"]) == 2
    # in-flight cap 2 at the destination, net 100: tool emissions at 1, 2, 3 -> the third overflows at 3
    p = W.tandem(1, 1000, 100)
    p["roles"][1]["flight_cap"] = 2
    s = _ovf(orc, p, [0, 0, 0])
    assert int(s["status"]) == 1 and int(s["stop_tick"]) == 3


# ------------------------------------------------------------------ R-SAT: saturated records, exact sums
def test_saturated_latencies(orc):
    # four requests at 0 on one tool with service s = (2^32 - 1) / 3: e2e = s, 2s, 3s = 2^32 - 1, 4s
    s_ = (2 ** 32 - 1) // 3
    g = W.grid([W.static()], [W.arr_list([0] * 4, prompt=(0, 0), output=(0, 0))], n_requests=4)
    r = orc.simulate(W.tool1(s_), g)
    s = r["summary"][0]
    sat = 0xFFFFFFFF
    assert r["records"][0, :, 0].tolist() == [s_, 2 * s_, sat, sat]
    assert r["records"][0, :, 1].tolist() == [s_, 2 * s_, sat, sat]   # a tool's first feedback = completion
    assert int(s["n_saturated"]) == 2
    assert int(s["sum_e2e"]) == 10 * s_ and int(s["sum_ff"]) == 10 * s_          # exact u64 sums (M19)
    assert int(s["max_e2e"]) == sat and int(s["p99_e2e"]) == sat and int(s["p50_e2e"]) == 2 * s_
    assert int(s["bin_p99_e2e"]) == 463


def test_batch_changes_every_window(orc):
    # fast (100) / slow (300) instances of the source role under RR, both under batch control (B default 2),
    # one request per window (j at 1000 j): window j holds request j on instance j mod 2.  Slow windows
    # violate (300 > 250, Q = 0) -> both instances halve to 1; fast windows are calm (200 <= 250) -> both
    # reset to 2.  Window 0 (fast, B already 2) changes nothing; windows 1..N-2 change both: 2 (N - 2).
    N = 50
    fast = W.cost(h=0, alpha=1, beta=0, tau0=99, gamma=0)
    slow = W.cost(h=0, alpha=1, beta=0, tau0=299, gamma=0)
    r = run(orc, srv(2, B=2, inst_cost=[fast, slow], route="rr"), batch_cand(250), [1000 * j for j in range(N)],
            n_windows=N)
    s = r["summary"][0]
    assert int(s["batch_changes"]) == 2 * (N - 2)
    assert r["records"][0, :, 0].tolist() == [100 if j % 2 == 0 else 300 for j in range(N)]
    assert [int(r["series"][0, w, i]["B"]) for w in range(4) for i in range(2)] == [2, 2, 2, 2, 1, 1, 2, 2]


def test_select_changes_every_window(orc):
    # one request on LARGE decoding for 1.4e8 ticks: busy(LARGE) = W -> SMALL; busy(SMALL) = 0 -> LARGE; ...
    # every one of the 140000 window closes before the completion at 1.4e8 switches
    large = dict(W.cost(h=0, alpha=1, beta=0, tau0=139_999_999, gamma=0), large=1)
    r = run(orc, srv(2, inst_cost=[large, SMALL], route="select"), sel_cand(10 ** 12), [0])
    s = r["summary"][0]
    assert int(s["select_changes"]) == 140000 == int(s["window_closes"])
    assert r["records"][0, :, 0].tolist() == [140_000_000]
