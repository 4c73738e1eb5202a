"""Two-level rings: on the specialised K1 levels a ring whose capacity exceeds the planner's
shared-memory bound keeps its oldest entries in shared memory and spills the rest to the warp's extension
area of `work`.  SDAS_FLAG_SPILL forces the smallest bound (32 entries), so every queue longer than 32
(overloaded replicas: deep tester inboxes / decode-wait queues, fan-out in-flight bursts) goes through
the extension.  Results must be bit-exact with the oracle and byte-identical to whole rings."""
import numpy as np
import pytest

import workloads as W
from gpu_parity import compare_records, full_check, run_gpu
from random_cases import make_case

pytestmark = pytest.mark.gpu


def _spill_equals_whole(p, g, series=False):
    gg, o = full_check(p, g, series=series, spill=True)
    assert gg["res"].layout.ring_s == 32 and gg["res"].layout.k1_variant >= 1
    whole = run_gpu(p, g, records=True, series=series, objective="p99_e2e")
    assert whole["summary"].tobytes() == gg["summary"].tobytes()
    compare_records(gg["records"], whole["records"], gg["summary"])   # the completed records of every replica
    for a, b in zip(whole["cells"], gg["cells"]):
        assert a.tobytes() == b.tobytes()
    return gg, o


def test_spill_config1_overloaded():
    # rates up to 1.15x the BATCH capacity: FUNCTION's tester wait queue reaches hundreds of items
    p, g = W.config1(n_seeds=3, n_requests=1200)
    gg, o = _spill_equals_whole(p, g)
    assert (o["summary"]["status"] == 0).any()


def test_spill_config2_controller_series():
    p, g = W.config2(n_seeds=2, n_requests=500, series_stride=5, series_windows=96)
    _spill_equals_whole(p, g, series=True)


def test_spill_config3_routing():
    p, g = W.config3(n_seeds=2, n_requests=300)
    gg, _ = _spill_equals_whole(p, g)
    assert gg["res"].layout.k1_variant == 1


def test_spill_config4_model_selection():
    p, g = W.config4(n_seeds=1, n_requests=400, candidates=W.config4_candidates()[::701])
    _spill_equals_whole(p, g)


def test_spill_fanout_bursts():
    # dev -> (tester, reviewer) fan-out with TOKEN(1) streams: in-flight bursts well past 32 per instance
    dev = W.role("dev", 1, W.cost(h=0), max_num_seqs=16, n_functions=4, inbox_cap=128, wait_cap=128)
    t = W.role("tester", 1, W.cost(h=2000), out=(0, 1, 1), inbox_cap=512, flight_cap=256, wait_cap=512)
    rv = W.role("reviewer", 1, W.cost(h=1000), out=(8, 0, 1), inbox_cap=512, flight_cap=256, wait_cap=512)
    p = W.pipeline([dev, t, rv], [W.link(0, 1, net=5000, chunk=1, mode="token"),
                                  W.link(0, 2, net=20000, chunk=2, mode="token")], feedback_role=1)
    g = W.grid([W.static("token", "token"), W.static("function", "batch")],
               [W.poisson(m) for m in (300000, 600000)], n_seeds=3, n_requests=300)
    _spill_equals_whole(p, g)


@pytest.mark.parametrize("seed", range(40))
def test_spill_random_cases(seed):
    p, g, obj = make_case(seed)
    gg = run_gpu(p, g, records=True, objective=obj, spill=True)
    if gg["res"].layout.k1_variant == 0:
        pytest.skip("level-0 grid (KV / classes / pacing / LOAD / truncation): rings stay whole")
    full_check(p, g, objective=obj, spill=True)
