"""Oracle pins for f2: request classes (M26), interactive-first service (M27), the
admission gate (M28) and per-class metrics (M29) -- PAPER.md:49, 126 ("pipeline-wide prioritization of
interactive or latency-sensitive requests"), PAPER.md:212 ("admit only high-priority requests under
load"); SPEC.md:27-31 (Priority), 159-164 (strictly higher priority first, FIFO within a priority).
"""
import numpy as np
import pytest

import oracle
import workloads as W

THR = lambda pm: (pm << 32) // 1000        # noqa: E731  M26 threshold floor(permille * 2^32 / 1000)


def classes(n, permille, s=0, master_seed=W.MASTER_SEED):
    """M26 from the Philox primitive (pinned by its KATs in test_oracle_primitives.py)."""
    key = (master_seed & 0xFFFFFFFF, master_seed >> 32)
    return [1 if oracle.philox((j, s, 2 << 16, 1), key)[0] < THR(permille) else 0 for j in range(n)]


def _tool_grid(ticks, permille, cands, service=700):
    p = W.tool1(service)
    g = W.grid(cands, [W.with_classes(W.arr_list(ticks, prompt=(0, 0), output=(0, 0)), permille)],
               n_requests=len(ticks))
    return p, g


def test_class_draw_counts():
    n = 2000
    p, g = _tool_grid([j * 1000 for j in range(n)], 300, [W.static()], service=10)
    s = oracle.simulate(p, g)["summary"][0]
    cls = classes(n, 300)
    assert int(s["completed_int"]) == sum(cls)
    assert abs(sum(cls) - 600) < 4 * np.sqrt(n * 0.3 * 0.7)        # binomial(2000, 0.3)


@pytest.mark.parametrize("permille", [0, 1000])
def test_one_class_limits(permille):
    p, g = W.config1(n_seeds=2, n_requests=300, rates=[2, 4])
    g["arrivals"] = [[W.with_classes(a, permille) for a in row] for row in g["arrivals"]]
    base = g["candidates"]
    g["candidates"] = base + [W.with_prio(c) for c in base]
    o = oracle.simulate(p, g)
    s = o["summary"].reshape(-1, 2, len(base))
    # priority service with a single class is FIFO: identical replicas
    for f in ("status", "completed", "sum_e2e", "p99_e2e", "p50_ff", "makespan", "decode_steps"):
        assert (s[:, 0][f] == s[:, 1][f]).all(), f
    ok = o["summary"]["status"] == 0
    if permille == 0:
        assert (o["summary"]["completed_int"] == 0).all() and (o["summary"]["p99_e2e_int"] == 0xFFFFFFFF).all()
    else:
        x = o["summary"][ok]
        assert (x["completed_int"] == x["completed"]).all() and (x["sum_e2e_int"] == x["sum_e2e"]).all()
        assert (x["p99_e2e_int"] == x["p99_e2e"]).all() and (x["p50_e2e_int"] == x["p50_e2e"]).all()


def _priority_queue_model(ticks, cls, S, prio):
    """Brute force: one deterministic server (service S), non-preemptive; START picks the earliest
    interactive waiting request if prio, else the earliest; arrivals at a tick join before START."""
    n = len(ticks)
    done = [None] * n
    waiting, t, j, busy_until, cur = [], 0, 0, None, None
    while any(d is None for d in done):
        cands = [x for x in (busy_until, ticks[j] if j < n else None) if x is not None]
        t = min(cands)
        if busy_until == t:
            done[cur] = t
            busy_until = cur = None
        while j < n and ticks[j] == t:
            waiting.append(j)
            j += 1
        if busy_until is None and waiting:
            pick = next((k for k in waiting if cls[k]), waiting[0]) if prio else waiting[0]
            waiting.remove(pick)
            cur, busy_until = pick, t + S
    return [done[k] - ticks[k] for k in range(n)]


@pytest.mark.parametrize("prio", [False, True])
def test_nonpreemptive_priority_single_server(prio):
    rng = np.random.default_rng(5)
    ticks = np.cumsum(rng.integers(100, 1300, size=300)).tolist()
    cls = classes(300, 400)
    p, g = _tool_grid(ticks, 400, [W.with_prio(W.static(), prio)], service=700)
    o = oracle.simulate(p, g)
    want = _priority_queue_model(ticks, cls, 700, prio)
    got = sorted(int(v) for v in o["records"][0, :, 0])
    assert got == sorted(want)
    s = o["summary"][0]
    assert int(s["sum_e2e_int"]) == sum(w for w, c in zip(want, cls) if c)


def test_cobham_md1_class_means():
    # non-preemptive priority M/D/1 (Cobham 1954): W0 = lambda S^2 / 2, W_int = W0 / (1 - rho_1),
    # W_bg = W0 / ((1 - rho_1)(1 - rho)); sojourn = W + S.  rho = 0.75, 30% interactive.
    S, gap, pm = 750, 1000, 300
    p = W.tool1(S, request_cap=4096)
    g = W.grid([W.with_prio(W.static())], [W.with_classes(W.poisson(gap, output=(0, 0)), pm)], n_seeds=24,
               n_requests=20000)
    s = oracle.simulate(p, g, records=False, hists=False)["summary"]
    lam, rho = 1.0 / gap, S / gap
    rho1 = rho * pm / 1000
    W0 = lam * S * S / 2
    want_int, want_bg = S + W0 / (1 - rho1), S + W0 / ((1 - rho1) * (1 - rho))
    n_int = s["completed_int"].astype(float).sum()
    got_int = s["sum_e2e_int"].astype(float).sum() / n_int
    got_bg = (s["sum_e2e"].astype(float).sum() - s["sum_e2e_int"].astype(float).sum()) / (
        s["completed"].astype(float).sum() - n_int)
    assert abs(got_int / want_int - 1) < 0.03 and abs(got_bg / want_bg - 1) < 0.05, (got_int, want_int, got_bg,
                                                                                     want_bg)


def test_admission_gate_limits():
    n, G = 400, 1000
    ticks = [j * 700 for j in range(n)]
    cls = classes(n, 300)
    p = W.tool1(300, request_cap=4096)
    p["window"] = G
    cands = [W.with_prio(W.static(), False, True, (0, 10 ** 9)),   # never closes == no gate
             W.static(),
             W.with_prio(W.static(), False, True, (0, 0))]         # closes at the first close, never reopens
    g = W.grid(cands, [W.with_classes(W.arr_list(ticks, prompt=(0, 0), output=(0, 0)), 300)], n_requests=n)
    s = oracle.simulate(p, g)["summary"]
    for f in ("completed", "sum_e2e", "makespan", "dropped"):
        assert s[0][f] == s[1][f], f
    assert s[0]["gate_changes"] == 0 and s[0]["rejected"] == 0
    # gate closed from tick G on (WINDOW precedes ARRIVE): every background arrival at t >= G is rejected
    rej = sum(1 for j in range(n) if ticks[j] >= G and not cls[j])
    assert int(s[2]["rejected"]) == rej and int(s[2]["dropped"]) == rej and int(s[2]["gate_changes"]) == 1
    assert int(s[2]["completed_int"]) == sum(cls) and int(s[2]["completed"]) == n - rej


def test_gate_opens_again_under_low_load():
    # bursty: a dense burst closes the gate, a long quiet tail reopens it (busy 0 <= lo)
    ticks = [j * 310 for j in range(60)] + [60 * 310 + 5000 * k for k in range(1, 200)]
    p = W.tool1(300, request_cap=4096)
    p["window"] = 2000
    g = W.grid([W.with_prio(W.static(), False, True, (100, 900))],
               [W.with_classes(W.arr_list(ticks, prompt=(0, 0), output=(0, 0)), 300)], n_requests=len(ticks))
    s = oracle.simulate(p, g)["summary"][0]
    assert int(s["gate_changes"]) >= 2 and 0 < int(s["rejected"]) < 60


def test_interactive_objective_argmin_brute_force():
    p, g = W.config_prio(n_seeds=2, n_requests=250, gaps=(726182, 399400))
    o = oracle.simulate(p, g)
    best = oracle.argmin_groups(p, g, o["summary"], "p99_e2e_int")
    C = len(g["candidates"])
    for gg, b in enumerate(best):
        rows = o["summary"][gg * C:(gg + 1) * C]
        keys = [(int(r["status"] != 0), int(r["p99_e2e_int"]), int(r["sum_e2e_int"]), c) for c, r in enumerate(rows)]
        assert b == min(keys)[-1]


def test_prio_helps_interactive_and_cells_hold_interactive_hist():
    # candidates: (batch|token) x (fifo|prio) x (no gate|gate); fifo vs prio without the gate, each mode at a
    # load it sustains (P2-X capacity: BATCH 2.5 req/s, TOKEN 0.98 req/s)
    for base, gap in ((0, 469882), (4, 1300000)):
        p, g = W.config_prio(n_seeds=4, n_requests=400, gaps=(gap,))
        o = oracle.simulate(p, g)
        s = o["summary"].reshape(-1, len(g["candidates"]))
        m = (s["status"][:, base] == 0) & (s["status"][:, base + 2] == 0)
        assert m.sum() >= 3
        mean = lambda k: (s[m, k]["sum_e2e_int"] / s[m, k]["completed_int"]).mean()   # noqa: E731
        assert mean(base + 2) < mean(base)
        cnt, hist = oracle.cells(p, g, o)
        assert (hist[:, 2].sum(axis=1) == cnt[:, 24]).all()
