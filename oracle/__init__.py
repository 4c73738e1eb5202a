"""CPU oracle for the SDAS strategy simulator -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2601_03197_b200``) never imports it and shares no code with it.

The oracle (``oracle.cpp``) is a plain event-heap DES of the model in DESIGN.md
§"Model" (rules M0-M20).  This wrapper only marshals the plain
dicts of ``workloads`` into the oracle's own ctypes structs.

Pins (tests/test_oracle_*.py), each independent of the oracle's own code:
  * Philox4x32-10: the three published Random123 known-answer vectors.
  * log2 table: closed form round(2^32 log2(1+i/256)) recomputed with mpmath-free
    Python integer/float math plus the spot values T[1..3], T[128] (SURVEY HT-8).
  * EXP sampler: edge values EXP(1e5; 2^31-1) = floor(1e5 ln 2) = 69314, the tail
    cap, and the stratified mean 1 - 0.5/M (closed form of the floor bias).
  * Arrivals: SURVEY.md HT-8 golden vectors (Poisson s=0/1, MMPP epoch crossing).
  * Mode semantics: SPEC.md:529 trace (267 / 523 ms) and the SURVEY.md HT-0..HT-3
    hand traces (e2e, ff, busy, event counts, integral of N_sys).
  * Queueing core: Lindley / tandem recursions computed independently in Python
    on the oracle's arrival ticks, exact for every request (HT-6).
  * Statistics: M/D/1 and M/M/1 mean waits (Pollaczek-Khinchine), M/G/1.
  * Little's law (integral N_sys dt == sum e2e) and message/token conservation.
  * Controller: HT-4 table; JSQ: HT-5; bins/percentiles: HT-7 + brute force.
  * Round 2 (tests/test_oracle_control.py, test_oracle_argmin.py, test_oracle_cellseries.py):
    hand-derived sequences for SLO batch control M16(ii), model selection M16(iii), RR and
    route overrides M11, the LOAD metric, max_ticks truncation, overflow ticks (R-OVF) and
    saturated latencies (R-SAT); every argmin objective per group and per pooled row against a
    tuple-key brute force (R-KEYS, R-RATE0); the cell-summed series (R-CSER).  Each of 28
    plausible slips in oracle.cpp turns one of them red (tools/mutate_oracle.py).
Parity unpinned: the full LLM-agent model (batching + RECV-first + modes) at scale
has no closed form; it is pinned only compositionally (DESIGN.md §"Parity pins").
"""

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.environ.get("ORACLE_LIB", os.path.join(_HERE, "liboracle.so"))   # ORACLE_LIB: mutation runs only

NBINS = 464
NCNT = 28
NHIST = 3
MAX_LINKS = 8

MODES = {"batch": 0, "function": 1, "token": 2}
KV_POLICIES = {"off": 0, "affinity": 1, "recompute": 2, "posthoc": 3, "hint": 4}


def _kv(pipe):
    kv = pipe.get("kv") or {}
    return (kv.get("role", 0), kv.get("ctx_tokens", 0), kv.get("tau_xfer", 0), kv.get("home_skew", 0))
ROUTES = {"jsq": 0, "rr": 1, "fixed": 2, "select": 3}
ARRIVALS = {"poisson": 0, "mmpp2": 1, "det": 2, "list": 3}
OBJECTIVES = {"p99_e2e": 0, "p50_e2e": 1, "p99_ff": 2, "throughput": 3, "goodput": 4, "large_under_slo": 5,
              "p90_e2e": 6, "p99_e2e_int": 7}
STATUS = {0: "ok", 1: "overflow", 2: "truncated"}
CELL_FIELDS = ["n_replicas", "n_ok", "n_overflow", "n_truncated", "admitted", "dropped", "completed",
               "sum_e2e", "sum_ff", "makespan_sum", "int_nsys", "good", "large_items", "arrivals",
               "deliveries", "recv_steps", "decode_steps", "window_closes", "mode_switches", "tokens",
               "batch_changes", "select_changes", "n_saturated", "kv_transfers"]


def build(force=False):
    src = os.path.join(_HERE, "oracle.cpp")
    if "ORACLE_LIB" in os.environ:              # a prebuilt (mutated) oracle under test: never rebuilt here
        return _LIB_PATH
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-o", _LIB_PATH, src,
                               "-lpthread"], cwd=_HERE)
    return _LIB_PATH


class Cost(C.Structure):
    _fields_ = [(n, C.c_uint32) for n in ("h", "alpha", "beta", "tau0", "gamma", "large")]


class Role(C.Structure):
    _fields_ = [("n_instances", C.c_uint32), ("cost", Cost), ("inst_cost", C.POINTER(Cost)),
                ("max_num_seqs", C.c_uint32), ("out_fixed", C.c_uint32), ("out_num", C.c_uint32),
                ("out_den", C.c_uint32), ("n_functions", C.c_uint32), ("svc_exp", C.c_uint32),
                ("route", C.c_uint32), ("route_fixed", C.c_uint32), ("inbox_cap", C.c_uint32),
                ("flight_cap", C.c_uint32), ("wait_cap", C.c_uint32)]


class Link(C.Structure):
    _fields_ = [(n, C.c_uint32) for n in ("src", "dst", "net", "chunk", "mode", "pacing_gap")]


class Arrival(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("gap", C.c_uint64 * 2), ("sojourn", C.c_uint64 * 2),
                ("list", C.POINTER(C.c_uint64)), ("list_len", C.c_uint32), ("p_lo", C.c_uint32),
                ("p_hi", C.c_uint32), ("o_lo", C.c_uint32), ("o_hi", C.c_uint32),
                ("interactive_permille", C.c_uint32)]


class Candidate(C.Structure):
    _fields_ = [("adaptive", C.c_uint32), ("mode", C.c_uint32 * MAX_LINKS), ("ctl_links", C.c_uint32),
                ("metric_load", C.c_uint32), ("lo", C.c_uint32), ("hi", C.c_uint32), ("dwell", C.c_uint32),
                ("band", C.c_uint32 * 3), ("route_override", C.c_uint32), ("batch_roles", C.c_uint32),
                ("q_hi", C.c_uint32), ("select_role", C.c_int32), ("policy_slo", C.c_uint64),
                ("kv_policy", C.c_uint32), ("guard_links", C.c_uint32), ("guard_pct", C.c_uint32),
                ("prio", C.c_uint32), ("admit", C.c_uint32), ("admit_lo", C.c_uint32), ("admit_hi", C.c_uint32),
                ("pacing_gap", C.c_uint32), ("stale_jsq", C.c_uint32)]


class Pipeline(C.Structure):
    _fields_ = [("n_roles", C.c_uint32), ("roles", C.POINTER(Role)), ("n_links", C.c_uint32),
                ("links", C.POINTER(Link)), ("feedback_role", C.c_uint32), ("request_cap", C.c_uint32),
                ("window", C.c_uint64), ("slo", C.c_uint64), ("kv_role", C.c_uint32),
                ("kv_ctx_tokens", C.c_uint32), ("kv_tau_xfer", C.c_uint32), ("kv_home_skew", C.c_uint32)]


class Grid(C.Structure):
    _fields_ = [("n_cand", C.c_uint32), ("cand", C.POINTER(Candidate)), ("n_rates", C.c_uint32),
                ("n_profiles", C.c_uint32), ("arr", C.POINTER(Arrival)), ("n_seeds", C.c_uint32),
                ("seed_offset", C.c_uint32), ("master_seed", C.c_uint64), ("n_requests", C.c_uint32),
                ("max_ticks", C.c_uint64), ("series_stride", C.c_uint32), ("series_slots", C.c_uint32),
                ("series_windows", C.c_uint32)]


SUMMARY_FIELDS = [
    ("status", np.uint32), ("admitted", np.uint32), ("dropped", np.uint32), ("completed", np.uint32),
    ("makespan", np.uint64), ("sum_e2e", np.uint64), ("sum_ff", np.uint64), ("int_nsys", np.uint64),
    ("p50_e2e", np.uint32), ("p99_e2e", np.uint32), ("p50_ff", np.uint32), ("p99_ff", np.uint32),
    ("bin_p50_e2e", np.uint32), ("bin_p99_e2e", np.uint32), ("bin_p50_ff", np.uint32), ("bin_p99_ff", np.uint32),
    ("max_e2e", np.uint32), ("n_saturated", np.uint32),
    ("arrivals", np.uint32), ("deliveries", np.uint32), ("recv_steps", np.uint32), ("decode_steps", np.uint32),
    ("window_closes", np.uint32), ("mode_switches", np.uint32), ("good", np.uint32), ("large_items", np.uint32),
    ("tokens", np.uint64), ("stop_tick", np.uint64), ("replica", np.uint64),
    ("batch_changes", np.uint32), ("select_changes", np.uint32), ("kv_transfers", np.uint32), ("p90_e2e", np.uint32),
    ("completed_int", np.uint32), ("rejected", np.uint32), ("good_int", np.uint32), ("gate_changes", np.uint32),
    ("sum_e2e_int", np.uint64), ("p50_e2e_int", np.uint32), ("p99_e2e_int", np.uint32),
    ("msgs_emitted", np.uint64), ("tokens_emitted", np.uint64), ("msgs_received", np.uint64),
    ("tokens_received", np.uint64),
]
SUMMARY_DTYPE = np.dtype(SUMMARY_FIELDS, align=True)
SERIES_DTYPE = np.dtype([("qint", np.uint64), ("busy", np.uint32), ("maxq", np.uint16), ("mode", np.uint8),
                         ("B", np.uint8)], align=True)
TRACE_DTYPE = np.dtype([("tick", np.uint64), ("code", np.uint32), ("a", np.uint32), ("b", np.uint32),
                        ("c", np.uint32)], align=True)

_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        L.orc_philox.argtypes = [C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        L.orc_log2_table.restype = C.c_uint64
        L.orc_log2_table.argtypes = [C.c_uint32]
        L.orc_exp_sample.restype = C.c_uint64
        L.orc_exp_sample.argtypes = [C.c_uint64, C.c_uint32]
        L.orc_uni.restype = C.c_uint32
        L.orc_uni.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32]
        L.orc_bin.restype = C.c_uint32
        L.orc_bin.argtypes = [C.c_uint32]
        L.orc_bin_lo.restype = C.c_uint64
        L.orc_bin_lo.argtypes = [C.c_uint32]
        L.orc_band.restype = C.c_uint32
        L.orc_band.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32]
        L.orc_jsq.restype = C.c_uint32
        L.orc_jsq.argtypes = [C.POINTER(C.c_uint32), C.c_uint32]
        L.orc_arrivals.restype = C.c_int
        L.orc_arrivals.argtypes = [C.POINTER(Arrival), C.c_uint64, C.c_uint32, C.c_uint32, C.c_void_p,
                                   C.c_void_p, C.c_void_p]
        L.orc_simulate.restype = C.c_int
        L.orc_simulate.argtypes = [C.POINTER(Pipeline), C.POINTER(Grid), C.c_void_p, C.c_uint64, C.c_uint32,
                                   C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p,
                                   C.c_uint64, C.POINTER(C.c_uint64), C.c_void_p]
        L.orc_cells.argtypes = [C.POINTER(Grid), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_argmin_groups.argtypes = [C.POINTER(Grid), C.c_void_p, C.c_uint32, C.c_uint64, C.c_void_p]
        L.orc_pooled_pct.restype = C.c_uint64
        L.orc_pooled_pct.argtypes = [C.c_void_p, C.c_uint32]
        L.orc_argmin_rows.argtypes = [C.POINTER(Grid), C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint64,
                                      C.c_void_p]
        _lib = L
    return _lib


# ------------------------------------------------------------------ marshalling
def _cost(d):
    return Cost(d["h"], d["alpha"], d["beta"], d["tau0"], d["gamma"], d.get("large", 0))


def _arrival(a, keep):
    x = Arrival()
    x.kind = ARRIVALS[a["kind"]]
    x.gap[0], x.gap[1] = a["gap"]
    x.sojourn[0], x.sojourn[1] = a["sojourn"]
    if a["list"]:
        arr = (C.c_uint64 * len(a["list"]))(*a["list"])
        keep.append(arr)
        x.list = C.cast(arr, C.POINTER(C.c_uint64))
        x.list_len = len(a["list"])
    x.p_lo, x.p_hi = a["prompt"]
    x.o_lo, x.o_hi = a["output"]
    x.interactive_permille = a.get("interactive", 0)
    return x


def _candidate(c, n_links):
    x = Candidate()
    x.adaptive = 1 if c["kind"] == "adaptive" else 0
    modes = list(c["modes"]) + [None] * MAX_LINKS
    for l in range(MAX_LINKS):
        m = modes[l] if l < len(c["modes"]) else (c["modes"][-1] if c["modes"] else None)
        x.mode[l] = 255 if m is None or l >= n_links else MODES[m]
    x.ctl_links = sum(1 << l for l in c["ctl_links"])
    x.metric_load = 1 if c["metric"] == "load" else 0
    x.lo, x.hi, x.dwell = c["lo"], c["hi"], c["dwell"]
    for b in range(3):
        x.band[b] = MODES[c["band"][b]]
    x.route_override = 255 if c["route"] is None else ROUTES[c["route"]]
    x.batch_roles = sum(1 << r for r in c["batch_roles"])
    x.q_hi = c["q_hi"]
    x.select_role = -1 if c["select_role"] is None else c["select_role"]
    x.policy_slo = c["policy_slo"]
    x.kv_policy = KV_POLICIES[c.get("kv", "off")]
    x.guard_links = sum(1 << l for l in c.get("guard_links", ()))
    x.guard_pct = c.get("guard_pct", 90)
    x.prio = 1 if c.get("prio") else 0
    x.admit = 1 if c.get("admit") else 0
    x.admit_lo, x.admit_hi = c.get("admit_band", (400, 800))
    x.pacing_gap = 0xFFFFFFFF if c.get("pacing_gap") is None else int(c["pacing_gap"])
    x.stale_jsq = 1 if c.get("stale_jsq") else 0
    return x


class Problem:
    """ctypes views of (pipeline, grid) dicts; keeps every buffer alive."""

    def __init__(self, pipe, grid):
        keep = []
        roles = (Role * len(pipe["roles"]))()
        for r, d in enumerate(pipe["roles"]):
            R = roles[r]
            R.n_instances = d["n_instances"]
            R.cost = _cost(d["cost"])
            if d["inst_cost"]:
                ic = (Cost * len(d["inst_cost"]))(*[_cost(x) for x in d["inst_cost"]])
                keep.append(ic)
                R.inst_cost = C.cast(ic, C.POINTER(Cost))
            R.max_num_seqs = d["max_num_seqs"]
            R.out_fixed, R.out_num, R.out_den = d["out"]
            R.n_functions = d["n_functions"]
            R.svc_exp = 1 if d["svc"] == "exp" else 0
            R.route = ROUTES[d["route"]]
            R.route_fixed = d["route_fixed"]
            R.inbox_cap, R.flight_cap, R.wait_cap = d["inbox_cap"], d["flight_cap"], d["wait_cap"]
        links = (Link * max(1, len(pipe["links"])))()
        for l, d in enumerate(pipe["links"]):
            links[l] = Link(d["src"], d["dst"], d["net"], d["chunk"], MODES[d["mode"]], d.get("pacing_gap", 0))
        self.pipe = Pipeline(len(pipe["roles"]), C.cast(roles, C.POINTER(Role)), len(pipe["links"]),
                             C.cast(links, C.POINTER(Link)), pipe["feedback_role"], pipe["request_cap"],
                             pipe["window"], pipe["slo"], *_kv(pipe))
        nl = len(pipe["links"])
        cands = (Candidate * len(grid["candidates"]))(*[_candidate(c, nl) for c in grid["candidates"]])
        I = len(grid["arrivals"])
        K = len(grid["arrivals"][0])
        arrs = (Arrival * (I * K))(*[_arrival(a, keep) for row in grid["arrivals"] for a in row])
        self.grid = Grid(len(grid["candidates"]), C.cast(cands, C.POINTER(Candidate)), I, K,
                         C.cast(arrs, C.POINTER(Arrival)), grid["n_seeds"], grid["seed_offset"],
                         grid["master_seed"], grid["n_requests"], grid["max_ticks"], grid["series_stride"],
                         grid["series_slots"], grid["series_windows"])
        self.keep = [roles, links, cands, arrs, keep]
        self.n_inst = sum(d["n_instances"] for d in pipe["roles"])
        self.C, self.I, self.K, self.S = len(grid["candidates"]), I, K, grid["n_seeds"]
        self.N = grid["n_requests"]
        self.R = self.C * I * K * self.S


CELL_SERIES_FIELDS = ["qint", "busy", "n", "maxq", "B", "n_batch", "n_function", "n_token"]


def simulate(pipe, grid, ids=None, threads=None, records=True, hists=True, series=False, trace_id=None,
             trace_cap=1 << 20, cell_series=False):
    """Run the oracle on replica ids (default: the whole grid).  Returns a dict of numpy arrays."""
    p = Problem(pipe, grid)
    if ids is None:
        ids = np.arange(p.R, dtype=np.uint64)
    ids = np.ascontiguousarray(np.asarray(ids, dtype=np.uint64))
    n = len(ids)
    threads = threads or os.cpu_count() or 1
    summ = np.zeros(n, dtype=SUMMARY_DTYPE)
    rec = np.zeros((n, p.N, 2), dtype=np.uint32) if records else None
    hst = np.zeros((n, NHIST, NBINS), dtype=np.uint32) if hists else None
    ser = None
    if series and grid["series_stride"]:
        ser = np.zeros((grid["series_slots"], grid["series_windows"], p.n_inst), dtype=SERIES_DTYPE)
    tr = np.zeros(trace_cap, dtype=TRACE_DTYPE) if trace_id is not None else None
    cser = None
    if cell_series and grid["series_windows"]:
        cser = np.zeros((p.I * p.K * p.C, grid["series_windows"], p.n_inst, 8), dtype=np.uint64)
    tn = C.c_uint64(0)
    rc = lib().orc_simulate(C.byref(p.pipe), C.byref(p.grid), ids.ctypes.data, n, threads, summ.ctypes.data,
                            rec.ctypes.data if rec is not None else None,
                            hst.ctypes.data if hst is not None else None,
                            ser.ctypes.data if ser is not None else None,
                            0 if trace_id is None else int(trace_id),
                            tr.ctypes.data if tr is not None else None, trace_cap, C.byref(tn),
                            cser.ctypes.data if cser is not None else None)
    if rc != 0:
        raise ValueError("oracle rejected the input (rc=%d)" % rc)
    out = {"summary": summ, "ids": ids, "records": rec, "hists": hst, "series": ser, "cell_series": cser}
    if tr is not None:
        out["trace"] = tr[: min(tn.value, trace_cap)]
    return out


def cells(pipe, grid, res):
    """Cell merge over a full-grid result (ids must be 0..R-1 in order)."""
    p = Problem(pipe, grid)
    assert len(res["ids"]) == p.R and res["hists"] is not None
    n_cells = p.I * p.K * p.C
    cnt = np.zeros((n_cells, NCNT), dtype=np.int64)
    hist = np.zeros((n_cells, NHIST, NBINS), dtype=np.int64)
    lib().orc_cells(C.byref(p.grid), res["summary"].ctypes.data, res["hists"].ctypes.data, cnt.ctypes.data,
                    hist.ctypes.data)
    return cnt, hist


def argmin_groups(pipe, grid, summary, objective="p99_e2e", slo=0):
    p = Problem(pipe, grid)
    best = np.zeros(p.I * p.K * p.S, dtype=np.int32)
    lib().orc_argmin_groups(C.byref(p.grid), summary.ctypes.data, OBJECTIVES[objective], slo, best.ctypes.data)
    return best


def argmin_rows(pipe, grid, cnt, hist, objective="p99_e2e", slo=0):
    p = Problem(pipe, grid)
    best = np.zeros(p.I * p.K, dtype=np.int32)
    lib().orc_argmin_rows(C.byref(p.grid), np.ascontiguousarray(cnt).ctypes.data,
                          np.ascontiguousarray(hist).ctypes.data, OBJECTIVES[objective], slo, best.ctypes.data)
    return best


def pooled_pct(hist, num):
    """M18 on one pooled histogram (NBINS counts): lower edge of the num-th percentile's bin."""
    h = np.ascontiguousarray(np.asarray(hist, dtype=np.int64))
    return lib().orc_pooled_pct(h.ctypes.data, num)


# ------------------------------------------------------------------ primitives
def philox(ctr, key):
    c = (C.c_uint32 * 4)(*ctr)
    k = (C.c_uint32 * 2)(*key)
    o = (C.c_uint32 * 4)()
    lib().orc_philox(c, k, o)
    return tuple(o)


def log2_table(i):
    return lib().orc_log2_table(i)


def exp_sample(mean, x):
    return lib().orc_exp_sample(mean, x)


def uni(lo, hi, x):
    return lib().orc_uni(lo, hi, x)


def bin_of(v):
    return lib().orc_bin(v)


def bin_lo(b):
    return lib().orc_bin_lo(b)


def band(u, lo, hi, window, n):
    return lib().orc_band(u, lo, hi, window, n)


def jsq(loads):
    a = (C.c_uint32 * len(loads))(*loads)
    return lib().orc_jsq(a, len(loads))


def arrivals(arr, s, n, master_seed=260103197):
    keep = []
    a = _arrival(arr, keep)
    t = np.zeros(n, dtype=np.uint64)
    pr = np.zeros(n, dtype=np.uint32)
    ou = np.zeros(n, dtype=np.uint32)
    rc = lib().orc_arrivals(C.byref(a), master_seed, s, n, t.ctypes.data, pr.ctypes.data, ou.ctypes.data)
    if rc:
        raise ValueError("bad arrival descriptor")
    return t, pr, ou


def mode_step(u, lo, hi, window, n, band, dwell, q, cur, q_last):
    """One window close of the M16(i) mode policy; returns (new_mode, new_q_last)."""
    L = lib()
    L.orc_mode_step.restype = C.c_uint32
    L.orc_mode_step.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32,
                                C.POINTER(C.c_uint32), C.c_uint32, C.c_int64, C.c_uint32, C.POINTER(C.c_int64)]
    b = (C.c_uint32 * 3)(*band)
    ql = C.c_int64(q_last)
    m = L.orc_mode_step(u, lo, hi, window, n, b, dwell, q, cur, C.byref(ql))
    return m, ql.value
