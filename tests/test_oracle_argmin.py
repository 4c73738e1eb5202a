"""Pins for the oracle's argmin (rule M20 with the DESIGN.md readings R-KEYS and R-RATE0), every objective,
per group (orc_argmin_groups) and per pooled cell row (orc_argmin_rows).

The brute force here is written from the key definitions in DESIGN.md §2 (R-KEYS), not from the oracle:
each candidate gets a Python tuple key and the winner is min() over the tuples -- a total order, so the
scan order cannot matter.  Rates are exact fractions (Fraction), never cross-multiplied.  Pooled row
percentiles are taken from the sorted multiset of samples (np.repeat of the histogram, or the union of
the cell's raw records), not from a cumulative scan.  Inputs: random summaries / cells with tiny value
ranges (ties on every field are frequent, so every tie-break is exercised) and real simulations.

R-KEYS (ties -> lowest c, the last key component):
  latency objective q (p50 / p90 / p99 e2e, p99 ff):  (bad, dropped, p_q, sum, c)
  MAX_THROUGHPUT / MAX_GOODPUT:                       (bad, -completed/makespan | -good/makespan, p99, c)
  MAX_LARGE_FRAC_UNDER_SLO (feasible = dropped == 0 and p99 <= slo):
                                                      (bad, not feasible, -large if feasible else dropped, p99, c)
  MIN_P99_E2E_INTERACTIVE:                            (bad, p99 interactive, sum interactive e2e, c)
bad = status != OK (group) or n_ok != n_replicas (row); a zero makespan is rate 0 (R-RATE0).
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle
import workloads as W

OBJS = list(oracle.OBJECTIVES)
P_FIELD = {"p99_e2e": "p99_e2e", "p50_e2e": "p50_e2e", "p99_ff": "p99_ff", "p90_e2e": "p90_e2e",
           "p99_e2e_int": "p99_e2e_int"}
SUM_FIELD = {"p99_ff": "sum_ff", "p99_e2e_int": "sum_e2e_int"}


def rate(n, m):
    return Fraction(int(n), int(m)) if m else Fraction(0)


def key(obj, c, bad, dropped, p, p99, s, completed, makespan, good, large, slo):
    if obj in ("throughput", "goodput"):
        return (bad, -rate(good if obj == "goodput" else completed, makespan), p99, c)
    if obj == "large_under_slo":
        feas = dropped == 0 and p99 <= slo
        return (bad, not feas, -large if feas else dropped, p99, c)
    if obj == "p99_e2e_int":
        return (bad, p, s, c)
    return (bad, dropped, p, s, c)


def brute_groups(summ, C, obj, slo):
    best = []
    for g in range(len(summ) // C):
        keys = []
        for c in range(C):
            x = summ[g * C + c]
            keys.append(key(obj, c, int(x["status"] != 0), int(x["dropped"]), int(x[P_FIELD.get(obj, "p99_e2e")]),
                            int(x["p99_e2e"]), int(x[SUM_FIELD.get(obj, "sum_e2e")]), int(x["completed"]),
                            int(x["makespan"]), int(x["good"]), int(x["large_items"]), slo))
        best.append(min(keys)[-1])
    return best


def _grid(C, I, K, S):
    return W.grid([W.static()] * C, [[W.poisson(1000)] * K for _ in range(I)], n_seeds=S)


@pytest.mark.parametrize("obj", OBJS)
def test_group_argmin_brute_force_random(obj):
    rng = np.random.default_rng(20260103 + OBJS.index(obj))
    C, I, K, S = 7, 3, 2, 50
    g = _grid(C, I, K, S)
    n = C * I * K * S
    s = np.zeros(n, dtype=oracle.SUMMARY_DTYPE)
    s["status"] = rng.choice([0, 0, 0, 1, 2], n)
    s["dropped"] = rng.integers(0, 3, n)
    for f in ("p50_e2e", "p99_e2e", "p99_ff", "p90_e2e", "p99_e2e_int"):
        s[f] = rng.integers(5, 8, n)
    for f in ("sum_e2e", "sum_ff", "sum_e2e_int"):
        s[f] = rng.integers(10, 12, n)
    s["completed"] = rng.integers(0, 4, n)
    s["makespan"] = rng.choice([0, 2, 3, 4, 6], n)
    s["good"] = rng.integers(0, 3, n)
    s["large_items"] = rng.integers(0, 4, n)
    best = oracle.argmin_groups(W.p2_x(), g, s, obj, slo=6)
    assert best.tolist() == brute_groups(s, C, obj, 6)


def _pooled(counts, q):
    """Lower bin edge of the nearest-rank q-percentile of the multiset holding counts[b] copies of bin b."""
    samples = np.repeat(np.arange(len(counts)), counts)          # sorted by construction
    if len(samples) == 0:
        return 0xFFFFFFFF
    k = -(-q * len(samples) // 100)                               # ceil(q n / 100), 1-based
    return int(oracle.bin_lo(int(samples[k - 1])))


def test_pooled_percentile_brute_force():
    # orc_pooled_pct against the sorted multiset of bins (random histograms, every quantile used)
    rng = np.random.default_rng(11)
    for _ in range(300):
        h = np.zeros(oracle.NBINS, dtype=np.int64)
        if rng.random() > 0.05:
            bins = rng.integers(0, oracle.NBINS, size=int(rng.integers(1, 40)))
            np.add.at(h, bins, rng.integers(1, 4, size=len(bins)))
        for q in (50, 90, 99):
            assert oracle.pooled_pct(h, q) == _pooled(h, q)


HIST = {"p99_ff": 1, "p99_e2e_int": 2}
Q = {"p50_e2e": 50, "p90_e2e": 90}
CNT = {n: i for i, n in enumerate(oracle.CELL_FIELDS + ["completed_int", "rejected", "sum_e2e_int", "good_int"])}


def brute_rows(cnt, hist, C, obj, slo, pooled=None):
    best = []
    for row in range(len(cnt) // C):
        keys = []
        for c in range(C):
            cell = row * C + c
            q = cnt[cell]
            p = pooled[cell] if pooled is not None else _pooled(hist[cell, HIST.get(obj, 0)], Q.get(obj, 99))
            p99 = pooled[cell] if pooled is not None else _pooled(hist[cell, 0], 99)
            sf = {"p99_ff": "sum_ff", "p99_e2e_int": "sum_e2e_int"}.get(obj, "sum_e2e")
            keys.append(key(obj, c, int(q[CNT["n_ok"]] != q[CNT["n_replicas"]]), int(q[CNT["dropped"]]), p, p99,
                            int(q[CNT[sf]]), int(q[CNT["completed"]]), int(q[CNT["makespan_sum"]]),
                            int(q[CNT["good"]]), int(q[CNT["large_items"]]), slo))
        best.append(min(keys)[-1])
    return best


@pytest.mark.parametrize("obj", OBJS)
def test_row_argmin_brute_force_random(obj):
    rng = np.random.default_rng(7 + OBJS.index(obj))
    C, I, K = 6, 5, 4
    g = _grid(C, I, K, 1)
    n_cells = C * I * K
    cnt = np.zeros((n_cells, oracle.NCNT), dtype=np.int64)
    cnt[:, CNT["n_replicas"]] = 3
    cnt[:, CNT["n_ok"]] = rng.choice([3, 3, 2], n_cells)
    for f, hi in (("dropped", 2), ("sum_e2e", 3), ("sum_ff", 3), ("sum_e2e_int", 3), ("completed", 4),
                  ("makespan_sum", 4), ("good", 3), ("large_items", 3)):
        cnt[:, CNT[f]] = rng.integers(0, hi, n_cells)
    hist = np.zeros((n_cells, oracle.NHIST, oracle.NBINS), dtype=np.int64)
    for cell in range(n_cells):
        for h in range(oracle.NHIST):
            if rng.random() < 0.15:
                continue                                          # an empty histogram: p = UINT32_MAX
            bins = rng.choice([17, 40, 41, 300], size=int(rng.integers(1, 6)))
            np.add.at(hist[cell, h], bins, 1)
    slo = int(oracle.bin_lo(40))
    best = oracle.argmin_rows(W.p2_x(), g, cnt, hist, obj, slo=slo)
    assert best.tolist() == brute_rows(cnt, hist, C, obj, slo)


# ------------------------------------------------------------------ real simulations
def _sim_grid():
    # P2-X at an overloaded and a moderate rate: TOKEN overflows at the high rate (bad), the adaptive
    # policies differ in drops, percentiles and throughput
    p, g = W.config1(n_seeds=3, n_requests=250, rates=[2, 7])
    g["candidates"] += [W.adaptive(["function"], lo=200, hi=600, dwell=1),
                        W.adaptive(["function"], lo=500, hi=900, dwell=4)]
    return p, g


@pytest.mark.parametrize("obj", ["p99_e2e", "p50_e2e", "p99_ff", "p90_e2e", "throughput", "goodput",
                                 "large_under_slo"])
def test_group_argmin_brute_force_simulated(obj):
    p, g = _sim_grid()
    o = oracle.simulate(p, g)
    slo = 6_000_000
    assert oracle.argmin_groups(p, g, o["summary"], obj, slo=slo).tolist() == \
        brute_groups(o["summary"], len(g["candidates"]), obj, slo)


@pytest.mark.parametrize("obj", ["p99_e2e", "p50_e2e", "p99_ff", "p90_e2e", "throughput", "goodput"])
def test_row_argmin_pooled_records(obj):
    # pooled row percentile = lower edge of the bin of the k-th smallest record of the whole cell (the union
    # of the records of its non-overflowed replicas), computed here by sorting that union
    p, g = _sim_grid()
    o = oracle.simulate(p, g)
    cnt, hist = oracle.cells(p, g, o)
    C, S = len(g["candidates"]), g["n_seeds"]
    field = 1 if obj == "p99_ff" else 0
    q = Q.get(obj, 99)
    pooled = []
    for cell in range(len(cnt)):
        ik, c = divmod(cell, C)
        vals = []
        for s in range(S):
            r = (ik * S + s) * C + c
            x = o["summary"][r]
            if x["status"] != 1:
                vals += o["records"][r, : int(x["completed"]), field].tolist()
        vals.sort()
        pooled.append(0xFFFFFFFF if not vals else
                      int(oracle.bin_lo(oracle.bin_of(vals[-(-q * len(vals) // 100) - 1]))))
    # (throughput / goodput break rate ties by the e2e p99: the same pooled list, field 0, q = 99)
    got = oracle.argmin_rows(p, g, cnt, hist, obj)
    assert got.tolist() == brute_rows(cnt, hist, C, obj, 0, pooled=pooled)
    assert (cnt[:, CNT["n_ok"]] != cnt[:, CNT["n_replicas"]]).any()     # the grid has bad cells
