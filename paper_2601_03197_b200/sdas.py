"""Thin Python binding of libsdas (include/sdas.h): argument marshalling only.

Every step of the simulation runs in the sm_100a kernels of libsdas.so; PyTorch only provides
device memory, streams and (in ``parallel``) process groups.  There is no CPU fallback: if the
shared library or a CUDA device is missing, calls raise.

The function names follow the C-ABI: ``Pipeline`` wraps sdas_pipeline_create / sdas_set /
sdas_reset / sdas_get; ``results_layout``, ``simulate``, ``control_sweep``, ``finalize`` and
``metrics`` wrap the calls of the same names.  Inputs are the plain dicts of ``workloads``.
"""
import ctypes as C
import os

import numpy as np

from . import build as _build

_lib = None

OK, E_INVALID_ARG, E_INVALID_FIELD, E_UNKNOWN_PARAM, E_OUT_OF_RANGE, E_BUFFER, E_CUDA, E_STATE, E_LIMIT = \
    0, -1, -2, -3, -4, -5, -6, -7, -8
MODES = {"batch": 0, "function": 1, "token": 2}
ROUTES = {"jsq": 0, "rr": 1, "fixed": 2, "select": 3}
KV_POLICIES = {"off": 0, "affinity": 1, "recompute": 2, "posthoc": 3, "hint": 4}


def _kv_fields(pipe):
    kv = pipe.get("kv") or {}
    return (kv.get("role", 0), kv.get("ctx_tokens", 0), kv.get("tau_xfer", 0), kv.get("home_skew", 0))


ARRIVALS = {"poisson": 0, "mmpp2": 1, "det": 2, "list": 3}
OBJECTIVES = {"p99_e2e": 0, "p50_e2e": 1, "p99_ff": 2, "throughput": 3, "goodput": 4, "large_under_slo": 5,
              "p90_e2e": 6, "p99_e2e_int": 7}
INTENTS = {None: 0, "max_throughput": 1, "min_p90_latency": 2}
CONSTRAINT_METRICS = {"e2e_p90": 0, "e2e_p99": 1}
SCOPES = {"replica": 0, "cell": 1, "group": 2, "row": 3}
FLAG_RECORDS, FLAG_SERIES, FLAG_TRACE, FLAG_STEPWISE, FLAG_GENERIC, FLAG_MID, FLAG_SPILL = 1, 2, 4, 8, 16, 32, 64
FLAG_CELL_SERIES = 128
CELL_SERIES_FIELDS = ["qint", "busy", "n", "maxq", "B", "n_batch", "n_function", "n_token"]
NBINS, NCNT, NHIST = 464, 28, 3
ROUTE_NONE = 255

SUMMARY_DTYPE = np.dtype([
    ("status", "<u4"), ("admitted", "<u4"), ("dropped", "<u4"), ("completed", "<u4"),
    ("makespan", "<u8"), ("sum_e2e", "<u8"), ("sum_ff", "<u8"), ("int_nsys", "<u8"),
    ("p50_e2e", "<u4"), ("p99_e2e", "<u4"), ("p50_ff", "<u4"), ("p99_ff", "<u4"),
    ("bin_p50_e2e", "<u2"), ("bin_p99_e2e", "<u2"), ("p90_e2e", "<u4"), ("max_e2e", "<u4"), ("n_saturated", "<u4"),
    ("arrivals", "<u4"), ("deliveries", "<u4"), ("recv_steps", "<u4"), ("decode_steps", "<u4"),
    ("window_closes", "<u4"), ("mode_switches", "<u4"), ("good", "<u4"), ("large_items", "<u4"),
    ("tokens", "<u8"), ("batch_changes", "<u4"), ("kv_transfers", "<u4"),
    ("completed_int", "<u4"), ("rejected", "<u4"), ("sum_e2e_int", "<u8"), ("p50_e2e_int", "<u4"),
    ("p99_e2e_int", "<u4"), ("good_int", "<u4"), ("gate_changes", "<u4"), ("select_changes", "<u4"),
    ("bin_p50_ff", "<u2"), ("bin_p99_ff", "<u2"), ("reserved", "<u4", (2,))])
assert SUMMARY_DTYPE.itemsize == 176
SERIES_DTYPE = np.dtype([("qint", "<u8"), ("busy", "<u4"), ("maxq", "<u2"), ("mode", "u1"), ("B", "u1")])
TRACE_DTYPE = np.dtype([("tick", "<u8"), ("code", "<u4"), ("a", "<u4"), ("b", "<u4"), ("c", "<u4")])
CELL_FIELDS = ["n_replicas", "n_ok", "n_overflow", "n_truncated", "admitted", "dropped", "completed",
               "sum_e2e", "sum_ff", "makespan_sum", "int_nsys", "good", "large_items", "arrivals",
               "deliveries", "recv_steps", "decode_steps", "window_closes", "mode_switches", "tokens",
               "batch_changes", "select_changes", "n_saturated", "kv_transfers", "completed_int", "rejected",
               "sum_e2e_int", "good_int"]


class SdasError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__("sdas error %d: %s" % (code, msg))
        self.code = code


# ------------------------------------------------------------------ C structs (include/sdas.h)
class Cost(C.Structure):
    _fields_ = [(n, C.c_uint32) for n in ("h_msg", "alpha", "beta", "tau0", "gamma", "large")]


class RoleDesc(C.Structure):
    _fields_ = [("n_instances", C.c_uint32), ("cost", Cost), ("inst_cost", C.POINTER(Cost)),
                ("max_num_seqs", C.c_uint32), ("out_fixed", C.c_uint32), ("out_num", C.c_uint32),
                ("out_den", C.c_uint32), ("n_functions", C.c_uint32), ("svc", C.c_uint32), ("route", C.c_uint32),
                ("route_fixed", C.c_uint32), ("inbox_cap", C.c_uint32), ("flight_cap", C.c_uint32),
                ("wait_cap", C.c_uint32)]


class LinkDesc(C.Structure):
    _fields_ = [(n, C.c_uint32) for n in ("src_role", "dst_role", "net_delay", "chunk_tokens", "mode", "pacing_gap")]


class PipelineDesc(C.Structure):
    _fields_ = [("n_roles", C.c_uint32), ("roles", C.POINTER(RoleDesc)), ("n_links", C.c_uint32),
                ("links", C.POINTER(LinkDesc)), ("feedback_role", C.c_uint32), ("request_cap", C.c_uint32),
                ("window_ticks", C.c_uint64), ("slo_ticks", C.c_uint64), ("kv_role", C.c_uint32),
                ("kv_ctx_tokens", C.c_uint32), ("kv_tau_xfer", C.c_uint32), ("kv_home_skew", C.c_uint32)]


class Candidate(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("mode", C.c_uint8 * 8), ("ctl_links", C.c_uint32), ("metric", C.c_uint32),
                ("lo_permille", C.c_uint32), ("hi_permille", C.c_uint32), ("dwell_windows", C.c_uint32),
                ("band_mode", C.c_uint8 * 4), ("route_override", C.c_uint32), ("batch_roles", C.c_uint32),
                ("q_hi", C.c_uint32), ("select_role", C.c_int32), ("kv_policy", C.c_uint32),
                ("guard_links", C.c_uint32), ("guard_pct", C.c_uint32), ("prio", C.c_uint32), ("admit", C.c_uint32),
                ("admit_lo_permille", C.c_uint32), ("admit_hi_permille", C.c_uint32), ("pacing_gap", C.c_uint32),
                ("stale_jsq", C.c_uint32), ("policy_slo_ticks", C.c_uint64)]


class Constraint(C.Structure):
    _fields_ = [("metric", C.c_uint32), ("scope_links", C.c_uint32), ("bound_ticks", C.c_uint64)]


class Intent(C.Structure):
    _fields_ = [("objective", C.c_uint32), ("n_constraints", C.c_uint32),
                ("constraints", C.POINTER(Constraint)), ("rules", C.POINTER(Candidate))]


class ArrivalDesc(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("mean_gap", C.c_uint64 * 2), ("mean_sojourn", C.c_uint64 * 2),
                ("list", C.POINTER(C.c_uint64)), ("list_len", C.c_uint32), ("prompt_lo", C.c_uint32),
                ("prompt_hi", C.c_uint32), ("out_lo", C.c_uint32), ("out_hi", C.c_uint32),
                ("interactive_permille", C.c_uint32)]


class Grid(C.Structure):
    _fields_ = [("n_candidates", C.c_uint32), ("cand", C.POINTER(Candidate)), ("n_rates", C.c_uint32),
                ("n_profiles", C.c_uint32), ("arrivals", C.POINTER(ArrivalDesc)), ("n_seeds", C.c_uint32),
                ("seed_offset", C.c_uint32), ("master_seed", C.c_uint64), ("n_requests", C.c_uint32),
                ("max_ticks", C.c_uint64), ("flags", C.c_uint32), ("series_stride", C.c_uint32),
                ("series_slots", C.c_uint32), ("series_windows", C.c_uint32), ("group_begin", C.c_uint64),
                ("group_end", C.c_uint64), ("rank", C.c_uint32), ("world", C.c_uint32),
                ("trace_replica", C.c_uint64), ("trace_cap", C.c_uint32)]


class Layout(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "params_bytes", "work_bytes", "summary_bytes", "records_bytes", "series_bytes", "cell_cnt_bytes",
        "cell_hist_bytes", "best_group_bytes", "best_row_bytes", "trace_bytes", "n_local_replicas",
        "n_local_groups", "n_groups", "n_cells", "n_rows", "n_replicas")] + [
        ("n_instances", C.c_uint32), ("smem_per_replica", C.c_uint32), ("warps_per_block", C.c_uint32),
        ("blocks_per_sm", C.c_uint32), ("resident_replicas", C.c_uint64), ("k1_variant", C.c_uint32),
        ("ring_s", C.c_uint32), ("cell_series_bytes", C.c_uint64)]


BUFFER_NAMES = ["params", "work", "summary", "records", "series", "cell_cnt", "cell_hist", "best_group",
                "best_row", "trace", "cell_series"]


class Buffers(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in BUFFER_NAMES]


class MetricsOut(C.Structure):
    _fields_ = [("status", C.c_uint32), ("n_replicas", C.c_uint64), ("admitted", C.c_uint64),
                ("dropped", C.c_uint64), ("completed", C.c_uint64), ("p50_e2e", C.c_uint32),
                ("p99_e2e", C.c_uint32), ("p50_ff", C.c_uint32), ("p99_ff", C.c_uint32),
                ("bin_p50_e2e", C.c_uint32), ("bin_p99_e2e", C.c_uint32), ("bin_p50_ff", C.c_uint32),
                ("bin_p99_ff", C.c_uint32), ("p90_e2e", C.c_uint32), ("pad0", C.c_uint32), ("mean_e2e", C.c_double), ("mean_ff", C.c_double),
                ("throughput", C.c_double), ("goodput", C.c_double)] + [
        (n, C.c_uint64) for n in ("makespan", "sum_e2e", "sum_ff", "int_nsys", "good", "large_items", "arrivals",
                                  "deliveries", "recv_steps", "decode_steps", "window_closes", "mode_switches",
                                  "tokens", "message_events", "des_events", "completed_int", "rejected",
                                  "sum_e2e_int", "good_int")] + [("p50_e2e_int", C.c_uint32), ("p99_e2e_int", C.c_uint32),
        ("best", C.c_int32), ("series", C.c_void_p), ("series_len", C.c_uint64)]


EXPORTS = ["sdas_last_error", "sdas_version", "sdas_pipeline_create", "sdas_pipeline_destroy", "sdas_set",
           "sdas_reset", "sdas_get", "sdas_results_layout", "sdas_simulate", "sdas_control_sweep",
           "sdas_group_argmin", "sdas_finalize", "sdas_metrics", "sdas_compile_intent"]


def lib():
    """Load libsdas.so (building it in-tree if stale).  Raises if it cannot be loaded."""
    global _lib
    if _lib is None:
        path = _build.LIB
        if _build.needs_build() and "SDAS_LIB" not in os.environ:   # an explicit SDAS_LIB is never rebuilt
            _build.build()
        if not os.path.exists(path):
            raise ImportError("libsdas.so missing: run python -m paper_2601_03197_b200.build")
        L = C.CDLL(path)
        L.sdas_last_error.restype = C.c_char_p
        L.sdas_version.restype = C.c_char_p
        L.sdas_pipeline_create.argtypes = [C.POINTER(PipelineDesc), C.POINTER(C.c_void_p)]
        L.sdas_pipeline_destroy.argtypes = [C.c_void_p]
        L.sdas_pipeline_destroy.restype = None
        L.sdas_set.argtypes = [C.c_void_p, C.c_char_p, C.c_int64]
        L.sdas_reset.argtypes = [C.c_void_p, C.c_char_p]
        L.sdas_get.argtypes = [C.c_void_p, C.c_char_p, C.POINTER(C.c_int64)]
        L.sdas_results_layout.argtypes = [C.c_void_p, C.POINTER(Grid), C.POINTER(Layout)]
        L.sdas_simulate.argtypes = [C.c_void_p, C.POINTER(Grid), C.POINTER(Buffers), C.c_void_p]
        L.sdas_control_sweep.argtypes = [C.c_void_p, C.POINTER(Grid), C.c_uint32, C.c_uint64, C.POINTER(Buffers),
                                         C.c_void_p]
        L.sdas_finalize.argtypes = [C.c_void_p, C.POINTER(Grid), C.c_uint32, C.c_uint64, C.POINTER(Buffers),
                                    C.c_void_p]
        L.sdas_group_argmin.argtypes = [C.c_void_p, C.POINTER(Grid), C.c_uint32, C.c_uint64, C.POINTER(Buffers),
                                        C.c_void_p]
        L.sdas_metrics.argtypes = [C.c_void_p, C.POINTER(Grid), C.POINTER(Buffers), C.c_uint32, C.c_uint64,
                                   C.POINTER(MetricsOut)]
        L.sdas_compile_intent.argtypes = [C.c_void_p, C.POINTER(Intent), C.POINTER(Candidate),
                                          C.POINTER(C.c_uint32)]
        for f in EXPORTS:
            if f not in ("sdas_last_error", "sdas_version", "sdas_pipeline_destroy"):
                getattr(L, f).restype = C.c_int32
        _lib = L
    return _lib


def _check(rc):
    if rc != OK:
        raise SdasError(rc, lib().sdas_last_error().decode())


# ------------------------------------------------------------------ marshalling
def _cost(d):
    return Cost(d["h"], d["alpha"], d["beta"], d["tau0"], d["gamma"], d.get("large", 0))


def _candidate(c, n_links):
    x = Candidate()
    x.kind = 1 if c["kind"] == "adaptive" else 0
    for l in range(8):
        if l < n_links and c["modes"]:
            m = c["modes"][l] if l < len(c["modes"]) else c["modes"][-1]
            x.mode[l] = 255 if m is None else MODES[m]
        else:
            x.mode[l] = 255
    x.ctl_links = sum(1 << l for l in c["ctl_links"])
    x.metric = 1 if c["metric"] == "load" else 0
    x.lo_permille, x.hi_permille, x.dwell_windows = c["lo"], c["hi"], c["dwell"]
    for b in range(3):
        x.band_mode[b] = MODES[c["band"][b]]
    x.route_override = ROUTE_NONE if c["route"] is None else ROUTES[c["route"]]
    x.batch_roles = sum(1 << r for r in c["batch_roles"])
    x.q_hi = c["q_hi"]
    x.select_role = -1 if c["select_role"] is None else c["select_role"]
    x.policy_slo_ticks = c["policy_slo"]
    x.kv_policy = KV_POLICIES[c.get("kv", "off")]
    x.guard_links = sum(1 << l for l in c.get("guard_links", ()))
    x.guard_pct = c.get("guard_pct", 90)
    x.prio = 1 if c.get("prio") else 0
    x.admit = 1 if c.get("admit") else 0
    x.admit_lo_permille, x.admit_hi_permille = c.get("admit_band", (400, 800))
    x.pacing_gap = 0xFFFFFFFF if c.get("pacing_gap") is None else int(c["pacing_gap"])
    x.stale_jsq = 1 if c.get("stale_jsq") else 0
    return x


def _candidate_dict(x, n_links):
    """Inverse of _candidate: a ctypes sdas_candidate as a workloads candidate dict."""
    inv = {v: k for k, v in MODES.items()}
    kvinv = {v: k for k, v in KV_POLICIES.items()}
    rinv = {v: k for k, v in ROUTES.items()}
    return {"kind": "adaptive" if x.kind == 1 else "static",
            "modes": [None if x.mode[l] == 255 else inv[x.mode[l]] for l in range(n_links)],
            "ctl_links": [l for l in range(n_links) if (x.ctl_links >> l) & 1],
            "metric": "load" if x.metric == 1 else "busy", "lo": x.lo_permille, "hi": x.hi_permille,
            "dwell": x.dwell_windows, "band": [inv[x.band_mode[b]] for b in range(3)],
            "route": None if x.route_override == ROUTE_NONE else rinv[x.route_override],
            "batch_roles": [r for r in range(32) if (x.batch_roles >> r) & 1], "q_hi": x.q_hi,
            "select_role": None if x.select_role < 0 else x.select_role, "policy_slo": x.policy_slo_ticks,
            "kv": kvinv[x.kv_policy], "guard_links": [l for l in range(n_links) if (x.guard_links >> l) & 1],
            "guard_pct": x.guard_pct, "prio": bool(x.prio), "admit": bool(x.admit),
            "admit_band": (x.admit_lo_permille, x.admit_hi_permille),
            "pacing_gap": None if x.pacing_gap == 0xFFFFFFFF else x.pacing_gap, "stale_jsq": bool(x.stale_jsq)}


def compile_intent(pipeline, objective=None, constraints=(), rules=None):
    """sdas_compile_intent (f3): an intent -> (candidate dict, sweep objective name).

    objective: None | "max_throughput" | "min_p90_latency"; constraints: [(metric, bound_ticks, scope_links)]
    with metric "e2e_p90" | "e2e_p99" and scope_links a list of link ids ([] = every link); rules: an
    explicit candidate dict (passed through)."""
    nl = len(pipeline.desc["links"])
    cs = (Constraint * max(1, len(constraints)))()
    for k, (m, bound, scope) in enumerate(constraints):
        cs[k] = Constraint(CONSTRAINT_METRICS[m], sum(1 << l for l in scope), bound)
    it = Intent(INTENTS[objective], len(constraints), C.cast(cs, C.POINTER(Constraint)), None)
    keep = None
    if rules is not None:
        keep = _candidate(rules, nl)
        it.rules = C.pointer(keep)
    out, obj = Candidate(), C.c_uint32()
    _check(lib().sdas_compile_intent(pipeline.h, C.byref(it), C.byref(out), C.byref(obj)))
    return _candidate_dict(out, nl), {v: k for k, v in OBJECTIVES.items()}[obj.value]


class GridView:
    """ctypes sdas_grid for a workloads grid dict (keeps its arrays alive)."""

    def __init__(self, pipe, grid, flags=0, rank=0, world=1, group_range=None, trace_replica=None,
                 trace_cap=1 << 16):
        self.keep = []
        nl = len(pipe["links"])
        cands = (Candidate * len(grid["candidates"]))(*[_candidate(c, nl) for c in grid["candidates"]])
        I, K = len(grid["arrivals"]), len(grid["arrivals"][0])
        arrs = (ArrivalDesc * (I * K))()
        for x, a in enumerate(a for row in grid["arrivals"] for a in row):
            A = arrs[x]
            A.kind = ARRIVALS[a["kind"]]
            A.mean_gap[0], A.mean_gap[1] = a["gap"]
            A.mean_sojourn[0], A.mean_sojourn[1] = a["sojourn"]
            if a["list"]:
                buf = (C.c_uint64 * len(a["list"]))(*a["list"])
                self.keep.append(buf)
                A.list = C.cast(buf, C.POINTER(C.c_uint64))
                A.list_len = len(a["list"])
            A.prompt_lo, A.prompt_hi = a["prompt"]
            A.out_lo, A.out_hi = a["output"]
            A.interactive_permille = a.get("interactive", 0)
        if trace_replica is not None:
            flags |= FLAG_TRACE
        gb, ge = group_range if group_range is not None else (0, 0)
        self.g = Grid(len(grid["candidates"]), C.cast(cands, C.POINTER(Candidate)), I, K,
                      C.cast(arrs, C.POINTER(ArrivalDesc)), grid["n_seeds"], grid["seed_offset"],
                      grid["master_seed"], grid["n_requests"], grid["max_ticks"], flags, grid["series_stride"],
                      grid["series_slots"], grid["series_windows"], gb, ge, rank, world,
                      0 if trace_replica is None else int(trace_replica), trace_cap)
        self.keep += [cands, arrs]
        self.C, self.I, self.K, self.S = len(grid["candidates"]), I, K, grid["n_seeds"]
        self.N = grid["n_requests"]
        self.flags = flags

    def ref(self):
        return C.byref(self.g)


class Pipeline:
    """sdas_pipeline_create / set / reset / get (Table 1)."""

    def __init__(self, pipe):
        self.desc = pipe
        roles = (RoleDesc * len(pipe["roles"]))()
        self._keep = []
        for r, d in enumerate(pipe["roles"]):
            R = roles[r]
            R.n_instances = d["n_instances"]
            R.cost = _cost(d["cost"])
            if d["inst_cost"]:
                ic = (Cost * len(d["inst_cost"]))(*[_cost(x) for x in d["inst_cost"]])
                self._keep.append(ic)
                R.inst_cost = C.cast(ic, C.POINTER(Cost))
            R.max_num_seqs = d["max_num_seqs"]
            R.out_fixed, R.out_num, R.out_den = d["out"]
            R.n_functions = d["n_functions"]
            R.svc = 1 if d["svc"] == "exp" else 0
            R.route = ROUTES[d["route"]]
            R.route_fixed = d["route_fixed"]
            R.inbox_cap, R.flight_cap, R.wait_cap = d["inbox_cap"], d["flight_cap"], d["wait_cap"]
        links = (LinkDesc * max(1, len(pipe["links"])))()
        for l, d in enumerate(pipe["links"]):
            links[l] = LinkDesc(d["src"], d["dst"], d["net"], d["chunk"], MODES[d["mode"]], d.get("pacing_gap", 0))
        desc = PipelineDesc(len(pipe["roles"]), C.cast(roles, C.POINTER(RoleDesc)), len(pipe["links"]),
                            C.cast(links, C.POINTER(LinkDesc)), pipe["feedback_role"], pipe["request_cap"],
                            pipe["window"], pipe["slo"], *_kv_fields(pipe))
        h = C.c_void_p()
        _check(lib().sdas_pipeline_create(C.byref(desc), C.byref(h)))
        self.h = h
        self.n_inst = sum(d["n_instances"] for d in pipe["roles"])

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.sdas_pipeline_destroy(self.h)
            self.h = None

    def set(self, knob, value):
        _check(lib().sdas_set(self.h, knob.encode(), int(value)))

    def reset(self, knob):
        _check(lib().sdas_reset(self.h, knob.encode()))

    def get(self, knob):
        v = C.c_int64()
        _check(lib().sdas_get(self.h, knob.encode(), C.byref(v)))
        return v.value


def results_layout(pipeline, gv):
    L = Layout()
    _check(lib().sdas_results_layout(pipeline.h, gv.ref(), C.byref(L)))
    return L


class Result:
    """Device buffers of one call (torch uint8 tensors) plus the layout."""

    def __init__(self, layout, tensors):
        self.layout = layout
        self.t = tensors

    def buffers(self):
        b = Buffers()
        for n in BUFFER_NAMES:
            x = self.t.get(n)
            setattr(b, n, C.c_void_p(x.data_ptr()) if x is not None and x.numel() else None)
        return b

    def summary(self):
        n = self.layout.n_local_replicas
        raw = self.t["summary"][: n * SUMMARY_DTYPE.itemsize].cpu().numpy()
        return raw.view(SUMMARY_DTYPE)

    def records(self, N):
        n = self.layout.n_local_replicas
        return self.t["records"][: n * N * 8].cpu().numpy().view(np.uint32).reshape(n, N, 2)

    def series(self, slots, windows, n_inst):
        return self.t["series"][: slots * windows * n_inst * 16].cpu().numpy().view(SERIES_DTYPE).reshape(
            slots, windows, n_inst)

    def cells(self):
        nc = self.layout.n_cells
        cnt = self.t["cell_cnt"][: nc * NCNT * 8].cpu().numpy().view(np.int64).reshape(nc, NCNT)
        hist = self.t["cell_hist"][: nc * NHIST * NBINS * 4].cpu().numpy().view(np.int32).reshape(nc, NHIST, NBINS)
        return cnt, hist

    def cell_series(self, windows, n_inst):
        """M15 cell-summed series: (n_cells, windows, n_inst, 8) u64, fields CELL_SERIES_FIELDS."""
        nc = self.layout.n_cells
        return self.t["cell_series"][: nc * windows * n_inst * 64].cpu().numpy().view(np.uint64).reshape(
            nc, windows, n_inst, 8)

    def best_group(self):
        return self.t["best_group"][: self.layout.n_local_groups * 4].cpu().numpy().view(np.int32)

    def best_row(self):
        return self.t["best_row"][: self.layout.n_rows * 4].cpu().numpy().view(np.int32)

    def trace(self):
        raw = self.t["trace"].cpu().numpy()
        n = int(raw[:8].view(np.uint64)[0])
        cap = (len(raw) - 8) // 24
        return raw[8: 8 + 24 * min(n, cap)].view(TRACE_DTYPE)


def _needs(layout, flags):
    """Byte size of every buffer a call with `flags` writes (sdas_results_layout)."""
    return {"params": layout.params_bytes, "work": layout.work_bytes, "summary": layout.summary_bytes,
            "records": layout.records_bytes if flags & FLAG_RECORDS else 0,
            "series": layout.series_bytes if flags & FLAG_SERIES else 0,
            "cell_cnt": layout.cell_cnt_bytes, "cell_hist": layout.cell_hist_bytes,
            "best_group": layout.best_group_bytes, "best_row": layout.best_row_bytes,
            "trace": layout.trace_bytes if flags & FLAG_TRACE else 0,
            "cell_series": layout.cell_series_bytes if flags & FLAG_CELL_SERIES else 0}


def allocate(layout, device, flags):
    import torch
    need = _needs(layout, flags)
    t = {k: torch.empty(int(v), dtype=torch.uint8, device=device) for k, v in need.items()
         if v and k not in ("cell_cnt", "cell_hist", "cell_series")}
    t["cell_cnt"] = torch.zeros(int(layout.cell_cnt_bytes), dtype=torch.uint8, device=device)
    t["cell_hist"] = torch.zeros(int(layout.cell_hist_bytes), dtype=torch.uint8, device=device)
    if flags & FLAG_CELL_SERIES and layout.cell_series_bytes:
        t["cell_series"] = torch.zeros(int(layout.cell_series_bytes), dtype=torch.uint8, device=device)
    return t


def check_buffers(result, layout, flags, device):
    """A reused Result must hold every buffer the new layout needs, large enough, on `device`: the C-ABI
    carries no buffer sizes, so a smaller buffer would let the kernels write out of bounds."""
    import torch
    dev = torch.device(device)
    for name, nbytes in _needs(layout, flags).items():
        if not nbytes:
            continue
        x = result.t.get(name)
        if x is None or x.numel() < nbytes:
            raise SdasError(E_BUFFER, "result buffer '%s' holds %d bytes, the grid needs %d"
                            % (name, 0 if x is None else x.numel(), nbytes))
        if x.device.type != dev.type or (dev.index is not None and x.device.index != dev.index):
            raise SdasError(E_BUFFER, "result buffer '%s' is on %s, the call runs on %s" % (name, x.device, dev))


def _stream(device):
    import torch
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def simulate(pipeline, gv, device="cuda", result=None, objective=None, objective_slo=0):
    """sdas_simulate (objective None) or sdas_control_sweep (objective given) into device buffers."""
    import torch
    if not torch.cuda.is_available():
        raise SdasError(E_CUDA, "no CUDA device: the SDAS simulator has no CPU path")
    L = results_layout(pipeline, gv)
    if result is None:
        result = Result(L, allocate(L, device, gv.flags))
    else:
        check_buffers(result, L, gv.flags, device)
        result.layout = L
    bufs = result.buffers()
    if objective is None:
        _check(lib().sdas_simulate(pipeline.h, gv.ref(), C.byref(bufs), _stream(device)))
    else:
        _check(lib().sdas_control_sweep(pipeline.h, gv.ref(), OBJECTIVES[objective], objective_slo, C.byref(bufs),
                                        _stream(device)))
    return result


def control_sweep(pipeline, gv, objective="p99_e2e", objective_slo=0, device="cuda", result=None):
    return simulate(pipeline, gv, device=device, result=result, objective=objective, objective_slo=objective_slo)


def group_argmin(pipeline, gv, result, objective="p99_e2e", objective_slo=0, device="cuda"):
    """sdas_group_argmin: K3 alone on summaries already in `result`."""
    bufs = result.buffers()
    _check(lib().sdas_group_argmin(pipeline.h, gv.ref(), OBJECTIVES[objective], objective_slo, C.byref(bufs),
                                   _stream(device)))
    return result


def finalize(pipeline, gv, result, objective="p99_e2e", objective_slo=0, device="cuda"):
    bufs = result.buffers()
    _check(lib().sdas_finalize(pipeline.h, gv.ref(), OBJECTIVES[objective], objective_slo, C.byref(bufs),
                               _stream(device)))
    return result


def metrics(pipeline, gv, host, scope, index):
    """sdas_metrics on host numpy copies: host = {name: np.ndarray(uint8)}."""
    b = Buffers()
    keep = []
    for n in BUFFER_NAMES:
        a = host.get(n)
        if a is not None:
            a = np.ascontiguousarray(a)
            keep.append(a)
            setattr(b, n, C.c_void_p(a.ctypes.data))
    out = MetricsOut()
    _check(lib().sdas_metrics(pipeline.h, gv.ref(), C.byref(b), SCOPES[scope], index, C.byref(out)))
    return {f: getattr(out, f) for f, _ in MetricsOut._fields_ if f != "series"}
