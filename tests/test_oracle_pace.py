"""Oracle pins for f4: data-plane pacing M30 -- PAPER.md:261 ("the data plane substrate
must support different message granularities ..., priorities, and pacing strategies")
(pacing_gap: minimum ms between envelope emissions), 188-191 (dispatch: "consecutive emissions on one link
are >= pacing_gap apart"; "pacing_gap=5, two ready envelopes at now=0 -> arrivals at 1 ms and 6 ms with
network_delay=1").
"""
import numpy as np
import pytest

import oracle
import workloads as W

KEY = [W.MASTER_SEED & 0xFFFFFFFF, W.MASTER_SEED >> 32]


def _svc(j, s, role, mean):
    w = oracle.philox([j, s, (3 << 16) | role, role], KEY)   # SVC stream; ordinal = the request's item index
    return max(1, oracle.exp_sample(mean, w[0]))


def test_spec_example_two_envelopes():
    # two requests in one decode batch finish together at tick T: their BATCH envelopes leave at T and T+5
    p = W.toy_ht("batch")
    p["links"][0].update(net=1, pacing_gap=5)
    g = W.grid([W.static("batch")], [W.arr_list([0, 0], prompt=(4, 4), output=(1, 1))], n_requests=2)
    tr = oracle.simulate(p, g, trace_id=0)["trace"]
    emits = sorted(int(r["tick"]) for r in tr if r["code"] == 6)          # TR_EMIT
    deliv = sorted(int(r["tick"]) for r in tr if r["code"] == 7)          # TR_DELIVER
    assert len(emits) == 2 and emits[0] == emits[1]
    T = emits[0]
    assert deliv == [T + 1, T + 6]
    p["links"][0]["pacing_gap"] = 0
    tr0 = oracle.simulate(p, g, trace_id=0)["trace"]
    assert sorted(int(r["tick"]) for r in tr0 if r["code"] == 7) == [T + 1, T + 1]


@pytest.mark.parametrize("svc", ["det", "exp"])
@pytest.mark.parametrize("gap", [0, 50000, 90000])
def test_paced_tandem_recursion(svc, gap):
    # C1 = max(A, C1') + S1 ; D = max(C1, D' + g) (dispatch) ; C2 = max(D + d, C2') + S2
    N, S1, S2, d, M = 1500, 60000, 70000, 1000, 100000
    p = W.tandem(S1, S2, d, svc=svc)
    p["links"][0]["pacing_gap"] = gap
    g = W.grid([W.static("batch")], [W.poisson(M, output=(0, 0))], n_seeds=2, n_requests=N)
    r = oracle.simulate(p, g)
    for x in range(2):
        A, _, _ = oracle.arrivals(W.poisson(M, output=(0, 0)), x, N)
        c1 = c2 = 0
        dprev = None
        e2e = []
        for j in range(N):
            s1 = S1 if svc == "det" else _svc(j, x, 0, S1)
            s2 = S2 if svc == "det" else _svc(j, x, 1, S2)
            c1 = max(int(A[j]), c1) + s1
            dj = c1 if (gap == 0 or dprev is None) else max(c1, dprev + gap)
            dprev = dj
            c2 = max(dj + d, c2) + s2
            e2e.append(c2 - int(A[j]))
        assert r["summary"][x]["status"] == 0
        assert r["records"][x, :, 0].tolist() == e2e


def test_candidate_override_and_zero():
    p, g = W.config_pace(n_seeds=2, n_requests=200, gaps=(726182,), pacing=(0, 4000))
    o = oracle.simulate(p, g)
    s = o["summary"].reshape(-1, len(g["candidates"]))
    # override 4000 on every link == the pipeline's link knob set to 4000
    p2 = W.p2_x()
    p2["links"][0]["pacing_gap"] = 4000
    g2 = W.grid([W.static(m) for m in ("token", "function", "batch")], g["arrivals"], n_seeds=2, n_requests=200)
    o2 = oracle.simulate(p2, g2)["summary"].reshape(-1, 3)
    for k in range(3):
        assert (s[:, 2 * k + 1]["sum_e2e"] == o2[:, k]["sum_e2e"]).all()
        assert (s[:, 2 * k + 1]["makespan"] == o2[:, k]["makespan"]).all()
    # override 0 == unpaced even when the link knob paces
    g3 = W.grid([W.with_pacing(W.static("token"), 0)], g["arrivals"], n_seeds=2, n_requests=200)
    o3 = oracle.simulate(p2, g3)["summary"]
    assert (o3["sum_e2e"] == s[:, 0]["sum_e2e"]).all()


def test_pacing_bounds_link_rate_and_conserves():
    # TOKEN(c=4) emits ~32 messages per request on dev->tester; a 20000-tick gap caps the link at 50 msg/s
    p, g = W.config_pace(n_seeds=2, n_requests=150, gaps=(1597600,), pacing=(0, 20000))
    o = oracle.simulate(p, g)
    s = o["summary"]
    assert (s["msgs_emitted"] == s["msgs_received"]).all() and (s["tokens_emitted"] == s["tokens_received"]).all()
    cs = s.reshape(-1, len(g["candidates"]))
    for k in range(0, len(g["candidates"]), 2):
        paced, free = cs[:, k + 1], cs[:, k]
        ok = (paced["status"] == 0) & (free["status"] == 0)
        assert ok.any()
        assert (paced["makespan"][ok] >= (paced["deliveries"][ok].astype(np.int64) - 1) * 20000).all()
        assert (paced["sum_e2e"][ok] >= free["sum_e2e"][ok]).all()


# ------------------------------------------------------------------ M31 snapshot (stale) JSQ routing
def _fanout2(route="jsq", window=1_000_000):
    # dev -> tester x 2 (SPEC.md:469 route(): least_queue_depth on the latest Snapshot, ties -> lowest id)
    dev = W.role("dev", c=W.cost(h=0), max_num_seqs=8, n_functions=2)
    tester = W.role("tester", 2, W.cost(h=2000), max_num_seqs=4, out=(0, 1, 1), route=route, route_fixed=0)
    return W.pipeline([dev, tester], [W.link(0, 1, net=500, chunk=8, mode="function")], window=window)


def test_stale_jsq_without_a_poll_is_fixed_zero():
    g = W.grid([dict(W.static("function"), stale_jsq=True)], [W.poisson(300_000, output=(32, 64))], n_seeds=3,
               n_requests=200)
    a = oracle.simulate(_fanout2(window=10 ** 12), g)["summary"]   # no window closes before the end
    gf = W.grid([W.static("function")], g["arrivals"], n_seeds=3, n_requests=200)
    b = oracle.simulate(_fanout2(route="fixed", window=10 ** 12), gf)["summary"]
    for f in ("status", "completed", "sum_e2e", "sum_ff", "makespan", "deliveries", "decode_steps"):
        assert (a[f] == b[f]).all(), f


def test_stale_jsq_sends_each_window_to_one_instance():
    Wn = 400_000
    p = _fanout2(window=Wn)
    g = W.grid([dict(W.static("function"), stale_jsq=True), W.static("function")],
               [W.poisson(150_000, output=(32, 64))], n_requests=150)
    dests = {}
    for rid in (0, 1):
        tr = oracle.simulate(p, g, trace_id=rid)["trace"]
        per_w = {}
        for r in tr:
            if r["code"] == 6 and (int(r["c"]) >> 16) & 1:          # TR_EMIT of an opening message
                per_w.setdefault(int(r["tick"]) // Wn, set()).add(int(r["a"]))
        dests[rid] = per_w
    assert all(len(v) == 1 for v in dests[0].values())                # stale: one instance per window
    assert {d for v in dests[0].values() for d in v} == {1, 2}       # ... that changes between windows
    assert any(len(v) == 2 for v in dests[1].values())                # live JSQ splits within a window
