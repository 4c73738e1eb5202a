"""Oracle pins for f3: the constraint-guard control rule M25 that compiled intents use,
the exact nearest-rank p90 (min_p90_latency objective) and its argmin (M20).

M25 ("min_p90_latency: token_stream(16) everywhere plus a
constraint-guard rule per constraint that flips the scoped links to batch_all when the constraint metric
violates its bound"; "ensure the end-to-end latency of 90% of interactive requests is within a
specified SLO ... demote ... to synchronous mode"): at each window close with n >= 1 completions, a guarded
link is set to BATCH iff fewer than ceil(pct * n / 100) of them met the bound, else reset to its initial
mode; dwell D and no-op suppression as M16.
"""
import numpy as np
import pytest

import oracle
import workloads as W


@pytest.fixture(scope="module")
def orc():
    return oracle


G = 1000   # one request per window: arrival j at j*G, window length G


def _toy(n, cand):
    p = W.toy_ht("token")
    p["window"] = G
    p["roles"][1]["cost"]["h"] = 40     # per-message cost: a lone request is slower under TOKEN than BATCH
    g = W.grid([cand], [W.arr_list([j * G for j in range(n)], prompt=(4, 4), output=(4, 4))], n_requests=n,
               series_stride=1, series_slots=1, series_windows=n)
    return p, g


def _single(orc, mode):
    p, g = _toy(1, W.static(mode))
    return int(orc.simulate(p, g)["records"][0, 0, 0])


def _guarded(bound, dwell=1, pct=90):
    c = W.static("token")
    c["kind"] = "adaptive"
    c["dwell"] = dwell
    c["policy_slo"] = bound
    c["guard_links"] = [0]
    c["guard_pct"] = pct
    return c


def test_guard_alternates_batch_and_reset(orc):
    e_t, e_b = _single(orc, "token"), _single(orc, "batch")
    assert e_b < e_t < G            # precondition of the hand derivation (requests never overlap)
    n = 7
    p, g = _toy(n, _guarded(bound=e_b))
    r = orc.simulate(p, g, series=True)
    s = r["summary"][0]
    # window k holds request k only: TOKEN violates (e_t > bound) -> BATCH for request k+1, whose e_b meets
    # the bound -> reset to TOKEN for request k+2 ...
    assert [int(v) for v in r["records"][0, :, 0]] == [e_t if j % 2 == 0 else e_b for j in range(n)]
    assert int(s["mode_switches"]) == n - 1 and int(s["window_closes"]) == n - 1
    modes = [int(r["series"][0, k, 1]["mode"]) for k in range(n)]      # tester's in-link mode per window
    assert modes == [oracle.MODES["token"] if k % 2 == 0 else oracle.MODES["batch"] for k in range(n)]


def test_guard_dwell_two(orc):
    e_t, e_b = _single(orc, "token"), _single(orc, "batch")
    n = 7
    p, g = _toy(n, _guarded(bound=e_b, dwell=2))
    r = orc.simulate(p, g)
    # close of window q-1 decides request q's mode.  q=1: TOKEN violated -> BATCH (q_last 1); q=2: reset
    # wanted, 2-1 < 2 held; q=3: reset (q_last 3); q=4: violated, 4-3 < 2 held; q=5: BATCH; q=6: held
    want = [e_t, e_b, e_b, e_t, e_t, e_b, e_b]
    assert [int(v) for v in r["records"][0, :, 0]] == want
    assert int(r["summary"][0]["mode_switches"]) == 3


@pytest.mark.parametrize("bound_kind", ["never", "always"])
def test_guard_limits(orc, bound_kind):
    e_t, e_b = _single(orc, "token"), _single(orc, "batch")
    n = 5
    if bound_kind == "never":          # every request meets the bound: nothing ever fires == static TOKEN
        p, g = _toy(n, _guarded(bound=e_t))
        r = orc.simulate(p, g)
        assert [int(v) for v in r["records"][0, :, 0]] == [e_t] * n
        assert int(r["summary"][0]["mode_switches"]) == 0
    else:                              # bound 0: violated at the first close, then BATCH never meets it
        p, g = _toy(n, _guarded(bound=0))
        r = orc.simulate(p, g)
        assert [int(v) for v in r["records"][0, :, 0]] == [e_t] + [e_b] * (n - 1)
        assert int(r["summary"][0]["mode_switches"]) == 1


def test_guard_pct_rank(orc):
    # pct 0: ceil(0) = 0 completions needed -> never violated, even with bound 0
    e_t = _single(orc, "token")
    p, g = _toy(4, _guarded(bound=0, pct=0))
    r = orc.simulate(p, g)
    assert [int(v) for v in r["records"][0, :, 0]] == [e_t] * 4


def test_guard_on_a_real_grid_only_switches_guarded_links(orc):
    # config-1 pipeline under load: the guard fires, and a static-token twin with the guard off differs
    p, g = W.config1(n_seeds=2, n_requests=300, rates=[1, 2])
    p["links"][0]["mode"] = "token"
    g["candidates"] = [W.static("token"), _guarded(bound=2_000_000)]
    o = orc.simulate(p, g)
    s = o["summary"].reshape(-1, 2)
    assert (s[:, 0]["mode_switches"] == 0).all()
    assert (s["status"] == 0).all()
    assert (s[:, 1]["mode_switches"] > 0).any()
    assert (s[:, 1]["p90_e2e"] <= s[:, 0]["p90_e2e"]).all()     # demoting to BATCH under overload helps p90


def test_p90_is_nearest_rank_of_records(orc):
    p, g = W.config1(n_seeds=2, n_requests=500, rates=[0, 3, 6])
    o = orc.simulate(p, g)
    for x, s in enumerate(o["summary"]):
        n = int(s["completed"])
        if s["status"] != 0 or n == 0:
            assert int(s["p90_e2e"]) == 0xFFFFFFFF
            continue
        e2e = np.sort(o["records"][x, :n, 0].astype(np.int64))
        assert int(s["p90_e2e"]) == int(e2e[-(-90 * n // 100) - 1])      # rank ceil(0.9 n), 1-based
        assert int(s["p50_e2e"]) <= int(s["p90_e2e"]) <= int(s["p99_e2e"])


def test_p90_argmin_brute_force(orc):
    p, g = W.config1(n_seeds=3, n_requests=300, rates=[2, 5])
    o = orc.simulate(p, g)
    best = orc.argmin_groups(p, g, o["summary"], "p90_e2e")
    C = len(g["candidates"])
    for gg, b in enumerate(best):
        rows = o["summary"][gg * C:(gg + 1) * C]
        keys = [(int(r["status"] != 0), int(r["dropped"]), int(r["p90_e2e"]), int(r["sum_e2e"]), c)
                for c, r in enumerate(rows)]
        assert b == min(keys)[-1]
