"""Pins for the oracle's cell-summed window series (SURVEY.md M15 "plus cell-summed series"; PAPER.md:231-238
"flexible aggregation functions"; reading R-CSER): per cell (i, k, c), window w and instance
{sum integral Q, sum busy, replicas that closed w, sum max Q, sum B, replicas per in-link mode}.

Pinned by: the HT-9 window-accounting hand trace (one replica: the cell series IS its window record), the
invariant cell series == the sum over the cell's seeds of the per-replica series (every replica sampled,
stride 1; the per-replica series are pinned by HT-9 and tests/test_oracle_control.py), and a replica
that overflows after two window closes (its two closed windows count, R-CSER)."""
import numpy as np

import oracle
import workloads as W


def test_ht9_cell_series_hand_values():
    # four arrivals at 990000 on one tool (15000 ticks each), W = 1e6 (tests/test_oracle_model.py HT-9):
    # window 0: busy 10000, integral Q 30000, max Q 3; window 1: busy 50000, Q 60000, max Q 3
    p = W.tool1(15000)
    g = W.grid([W.static()], [W.arr_list([990000] * 4, prompt=(0, 0), output=(0, 0))], n_requests=4,
               series_windows=3)
    cs = oracle.simulate(p, g, cell_series=True)["cell_series"]
    assert cs.shape == (1, 3, 1, 8)
    B = p["roles"][0]["max_num_seqs"]
    assert cs[0, 0, 0].tolist() == [30000, 10000, 1, 3, B, 0, 0, 0]     # no in-link: no mode counts
    assert cs[0, 1, 0].tolist() == [60000, 50000, 1, 3, B, 0, 0, 0]
    assert cs[0, 2, 0].tolist() == [0] * 8                              # the replica ended in window 1


def test_cell_series_is_the_sum_of_replica_series():
    p, g = W.config2(n_seeds=5, n_requests=250, series_stride=1, series_windows=80)
    g["arrivals"] = g["arrivals"][:5]                     # rates that never overflow (TOKEN at high load would)
    R = W.grid_size(g)
    g["series_slots"] = R                                 # every replica keeps its own series
    o = oracle.simulate(p, g, series=True, cell_series=True)
    ser, cs, s = o["series"], o["cell_series"], o["summary"]
    C, S = len(g["candidates"]), g["n_seeds"]
    assert (s["status"] == 0).all()                       # no overflow: every window a replica closed is in its series
    for cell in range(cs.shape[0]):
        ik, c = divmod(cell, C)
        rids = [(ik * S + x) * C + c for x in range(S)]
        reached = np.array([[w <= int(s[r]["window_closes"]) for w in range(80)] for r in rids])   # + final
        for i in range(2):
            rs = ser[rids, :, i]
            assert cs[cell, :, i, 0].tolist() == rs["qint"].astype(np.uint64).sum(0).tolist()
            assert cs[cell, :, i, 1].tolist() == rs["busy"].astype(np.uint64).sum(0).tolist()
            assert cs[cell, :, i, 2].tolist() == reached.sum(0).tolist()
            assert cs[cell, :, i, 3].tolist() == rs["maxq"].astype(np.uint64).sum(0).tolist()
            assert cs[cell, :, i, 4].tolist() == (rs["B"].astype(np.uint64) * reached).sum(0).tolist()
            for m in range(3):
                want = ((rs["mode"] == m) & reached).sum(0) if i == 1 else np.zeros(80, np.int64)
                assert cs[cell, :, i, 5 + m].tolist() == want.tolist()


def test_cell_series_keeps_windows_closed_before_an_overflow():
    # inbox cap 2, service 10: requests at 5, 5, 6 are served; three arrivals at 2000007 overflow there.
    # Windows 0 and 1 were closed (at 1e6, 2e6) before the overflow: they count (R-CSER), window 2 does not
    p = W.tool1(10)
    p["roles"][0]["inbox_cap"] = 2
    g = W.grid([W.static()], [W.arr_list([5, 5, 6] + [2_000_007] * 3, prompt=(0, 0), output=(0, 0))], n_requests=6,
               series_windows=4)
    o = oracle.simulate(p, g, cell_series=True)
    assert int(o["summary"][0]["status"]) == 1
    cs = o["cell_series"][0, :, 0]
    assert cs[:, 2].tolist() == [1, 1, 0, 0] and cs[:, 1].tolist() == [30, 0, 0, 0]
