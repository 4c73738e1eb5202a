"""Pins for the oracle's primitives (rules M2, M3, M11, M16(i), M17, M18).

Every expected value here is fixed by something other than the oracle's code:
published Random123 KATs, closed forms computed with Python's decimal/math,
brute-force definitions, or the SURVEY.md hand-traced tables (HT-4, HT-5, HT-7).
"""
import json
import math
import os
import random
from decimal import Decimal, getcontext

import numpy as np
import pytest

import workloads as W

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _h(x):
    return int(x, 16) if isinstance(x, str) else int(x)


def test_philox_kat(orc):
    kat = json.load(open(os.path.join(GOLD, "ht8_rng.json")))["philox_kat"]
    for v in kat:
        out = orc.philox([_h(x) for x in v["ctr"]], [_h(x) for x in v["key"]])
        assert [f"{x:08x}" for x in out] == v["out"]


def test_log2_table_closed_form(orc):
    # T[i] = round(2^32 log2(1 + i/256)), recomputed with 50-digit decimals (rule M3)
    getcontext().prec = 50
    ln2 = Decimal(2).ln()
    for i in range(257):
        v = (Decimal(256 + i) / Decimal(256)).ln() / ln2 * (Decimal(2) ** 32)
        assert orc.log2_table(i) == int(v.to_integral_value()), i
    spots = json.load(open(os.path.join(GOLD, "ht8_rng.json")))["log2_table_spots"]
    for k, v in spots.items():
        assert orc.log2_table(int(k)) == v


def test_exp_sampler_edges_and_closed_form(orc):
    edges = json.load(open(os.path.join(GOLD, "ht8_rng.json")))["exp_edges_M1e5"]
    for x, v in edges.items():
        assert orc.exp_sample(100000, int(x)) == v
    # |EXP(M;x) - (-M ln U)| <= 1 + M*ln2*2.8e-6 with U = (x+1)/2^32: floor (<1) plus the
    # chord-below-concave-log2 interpolation error (<= 2.74e-6 in log2 units, SURVEY c.5)
    rng = random.Random(1)
    for M in (1, 7, 1000, 100000, 3994000, 60000000):
        bound = 1.0 + M * math.log(2) * 2.8e-6
        for _ in range(400):
            x = rng.getrandbits(32)
            exact = -M * math.log((x + 1) / 2 ** 32)
            got = orc.exp_sample(M, x)
            assert exact - bound <= got <= exact + M * math.log(2) * 2.8e-6 + 1e-6, (M, x, got, exact)


def test_exp_sampler_stratified_mean(orc):
    # mean over stratified U approaches E[floor(M Exp(1))] ~= M - 1/2 (floor bias), SURVEY c.5
    M = 100000
    n = 1 << 14
    xs = [(k << 18) + (1 << 17) for k in range(n)]
    mean = sum(orc.exp_sample(M, x) for x in xs) / n
    assert abs(mean / M - (1 - 0.5 / M)) < 2e-3


def test_uni(orc):
    assert orc.uni(64, 256, 0) == 64
    assert orc.uni(64, 256, 2 ** 32 - 1) == 256
    assert orc.uni(5, 5, 12345) == 5
    rng = random.Random(2)
    for _ in range(200):
        lo = rng.randrange(0, 1000)
        hi = lo + rng.randrange(0, 1000)
        x = rng.getrandbits(32)
        assert orc.uni(lo, hi, x) == lo + (x * (hi - lo + 1)) // 2 ** 32


def test_bins_ht7(orc):
    assert orc.bin_of(100000) == 216 and orc.bin_lo(216) == 98304 and orc.bin_lo(217) == 102400
    assert orc.bin_of(266000) == 240 and orc.bin_lo(240) == 262144 and orc.bin_lo(241) == 278528
    for v in range(32):
        assert orc.bin_of(v) == v
    assert orc.bin_of(2 ** 32 - 1) == 463
    # containment and relative width <= 1/16 on random values (M17 by its defining property)
    rng = random.Random(3)
    prev = 0
    for v in sorted(rng.getrandbits(rng.randrange(1, 33)) for _ in range(3000)):
        b = orc.bin_of(v)
        assert orc.bin_lo(b) <= v < orc.bin_lo(b + 1)
        assert b >= prev
        prev = b
        if v >= 32:
            assert (orc.bin_lo(b + 1) - orc.bin_lo(b)) * 16 <= orc.bin_lo(b)


def test_jsq_ht5(orc):
    assert orc.jsq([5, 1]) == 1
    assert orc.jsq([2, 2]) == 0
    rng = random.Random(4)
    for _ in range(200):
        loads = [rng.randrange(0, 50) for _ in range(rng.randrange(1, 8))]
        i = orc.jsq(loads)
        assert loads[i] == min(loads) and i == loads.index(min(loads))
        k = rng.randrange(1, 100)
        assert orc.jsq([k * x for x in loads]) == i  # scaling invariance


def test_controller_ht4(orc):
    B, F, T = 0, 1, 2
    band = [T, F, B]
    busy = [812345, 350000, 400000, 799999, 800000]
    for dwell, expect, switches in ((2, [B, B, T, T, B], 3), (1, [B, T, T, F, B], 4)):
        cur, q_last, got, n = F, -(1 << 62), [], 0
        for k, u in enumerate(busy):
            new, q_last = orc.mode_step(u, 400, 800, 10 ** 6, 1, band, dwell, k + 1, cur, q_last)
            n += new != cur
            cur = new
            got.append(cur)
        assert got == expect and n == switches


def test_band_inclusive_edges(orc):
    W_ = 10 ** 6
    assert orc.band(800000, 400, 800, W_, 1) == 2   # 1000u >= hi W n
    assert orc.band(799999, 400, 800, W_, 1) == 1
    assert orc.band(400000, 400, 800, W_, 1) == 0   # 1000u <= lo W n
    assert orc.band(400001, 400, 800, W_, 1) == 1
    assert orc.band(1600000, 400, 800, W_, 2) == 2  # n instances scale the threshold


def test_percentiles_nearest_rank(orc):
    # p90(1..100)=90, p99(1..1000)=990 -- the definition k = ceil(q n)
    def nearest(vals, q_num):
        k = -(-q_num * len(vals) // 100)
        return sorted(vals)[k - 1]
    assert nearest(list(range(1, 101)), 90) == 90
    assert nearest(list(range(1, 1001)), 99) == 990
    # the oracle's p50/p99 equal the definition applied to its own records, and the bin
    # of the value is the histogram bin (M18)
    p = W.p2_x()
    g = W.grid([W.static("batch"), W.static("function")], [W.poisson(570571)], n_seeds=3, n_requests=700)
    r = orc.simulate(p, g)
    for x in range(len(r["ids"])):
        s = r["summary"][x]
        n = int(s["completed"])
        e2e = r["records"][x, :n, 0].astype(np.int64).tolist()
        ff = r["records"][x, :n, 1].astype(np.int64).tolist()
        assert s["p50_e2e"] == nearest(e2e, 50) and s["p99_e2e"] == nearest(e2e, 99)
        assert s["p50_ff"] == nearest(ff, 50) and s["p99_ff"] == nearest(ff, 99)
        assert s["bin_p99_e2e"] == orc.bin_of(int(s["p99_e2e"]))
        assert s["bin_p50_ff"] == orc.bin_of(int(s["p50_ff"]))
        assert r["hists"][x, 0].sum() == n and r["hists"][x, 1].sum() == n
        assert s["sum_e2e"] == sum(e2e) and s["max_e2e"] == max(e2e)
