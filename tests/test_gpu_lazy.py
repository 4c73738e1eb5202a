"""LEAN K1's lazy deliveries, emit-ahead source runs, RECV chains, advance first feedback and
chained resume (§5.8: full batches with waiting items, window closes and B changes inside chunk RECVs)
against the oracle and against the
generic kernel (which delivers every message as its own event and ends every run at an emission point):
P2-X / P2-SPEC variants that exercise every branch -- TOKEN / FUNCTION / BATCH, deep batches (B = 32) whose
emit-ahead steps do not fit the destination's in-flight ring (room-limited runs), in-flight rings smaller
than the batch (emit-ahead off), a net delay longer than a DECODE step (emit-ahead off), tester inboxes
near full (lazy deliveries become events), arrivals landing exactly on step boundaries, adaptive control
with waiting items (window-bounded runs), the two-level-ring kernel, and the bench's config-2 grid."""
import copy

import pytest

import workloads as W
from gpu_parity import compare_records, full_check, run_gpu

pytestmark = pytest.mark.gpu


def _lean_vs_generic(p, g, series=False, spill=False):
    a, o = full_check(p, g, series=series, spill=spill)
    assert a["res"].layout.k1_variant == 2
    b = run_gpu(p, g, series=series, generic=True, objective="p99_e2e")
    assert a["summary"].tobytes() == b["summary"].tobytes()
    compare_records(a["records"], b["records"], a["summary"])
    for x, y in zip(a["cells"], b["cells"]):
        assert x.tobytes() == y.tobytes()
    if series:
        assert a["series"].tobytes() == b["series"].tobytes()
    return a, o


CANDS = [W.static("token"), W.static("function"), W.static("batch"), W.adaptive(["function"], dwell=1),
         W.adaptive(["token"], lo=600, hi=900, dwell=2)]


@pytest.mark.parametrize("variant", ["base", "b32_room", "tiny_flight", "slow_net", "small_inbox", "det_boundary",
                                     "spec_chunk1", "series", "slow_recv", "fast_recv", "tiny_inbox",
                                     "chain_full_batch", "chain_window_b"])
def test_lazy_and_ahead_variants(variant):
    p = W.p2_x()
    g = W.grid(copy.deepcopy(CANDS), [W.poisson(m) for m in (3994000, 998500, 469882, 347304)], n_seeds=3,
               n_requests=400)
    series = False
    if variant == "b32_room":          # 32 sequences x TOKEN(4): more ahead messages than the 64-slot ring
        p["roles"][0]["max_num_seqs"] = 32
    elif variant == "tiny_flight":     # ring smaller than the batch: emit-ahead off, overflows in TOKEN
        p["roles"][1]["flight_cap"] = 6
    elif variant == "slow_net":        # net delay > one DECODE step: emit-ahead off
        p["links"][0]["net"] = 40000
    elif variant == "small_inbox":     # the tester's inbox nearly full: lazy deliveries turn into events
        p["roles"][1]["inbox_cap"] = 40
    elif variant == "det_boundary":    # DET arrivals on a grid commensurate with the step costs
        g["arrivals"] = [[W.det(16000 * k)] for k in (40, 100, 250)]
    elif variant == "spec_chunk1":     # P2-SPEC with TOKEN(1): an emission every step
        p = W.p2_spec(mode="token", chunk=1, n_functions=4)
    elif variant == "slow_recv":       # chunk RECVs longer than the chunk spacing: chains break (hard ticks)
        p["roles"][1]["cost"]["h"] = 60000
    elif variant == "fast_recv":       # cheap chunk RECVs: long chains of non-closing chunks
        p["roles"][1]["cost"].update(h=500, beta=5)
        p["links"][0]["chunk"] = 2
    elif variant == "tiny_inbox":      # hard messages queue behind chains into a 3-slot inbox: overflow ticks
        p["roles"][1]["inbox_cap"] = 3
        p["roles"][1]["cost"]["h"] = 30000
    elif variant == "chain_full_batch":   # chained resume with a full batch and items waiting
        p["roles"][1]["max_num_seqs"] = 1
        p["roles"][1]["cost"].update(h=3000, beta=10)
        p["window"] = 37_000              # window closes (possible B changes) inside many chunk RECVs
    elif variant == "chain_window_b":     # SLO batch control on the tester: B changes at window closes
        p["roles"][1]["max_num_seqs"] = 2
        p["window"] = 53_000
        g["candidates"] = g["candidates"] + [
            W.adaptive(["token"], batch_roles=[1], q_hi=1, policy_slo=2_000_000, dwell=1),
            W.adaptive(["token"], lo=100, hi=200, batch_roles=[1], q_hi=3, policy_slo=800_000, dwell=1)]
    elif variant == "series":
        g["series_stride"], g["series_slots"], g["series_windows"] = 7, 9, 200
        series = True
    _lean_vs_generic(p, g, series=series)


def test_lazy_and_ahead_spill_kernel():
    p, g = W.config2(n_seeds=2, n_requests=400, series_stride=0)
    _lean_vs_generic(p, g, spill=True)


def test_lazy_and_ahead_config2_grid():
    p, g = W.config2(n_seeds=3, n_requests=500, series_stride=5, series_windows=128)
    _lean_vs_generic(p, g, series=True)
