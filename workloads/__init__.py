"""Seeded synthetic input generators shared by the oracle and the CUDA path.

This module holds *only data*: pipeline parameter sets, candidate lists and
replica grids, as plain Python dicts.  It contains none of the method's
arithmetic (no sampling, no event logic, no metrics) -- the oracle
(``oracle/``) and the product binding (``paper_2601_03197_b200.sdas``) each
translate these dicts into their own structs.  The random numbers the method
draws are NOT generated here: both sides implement the same counter-based
Philox4x32-10 generator keyed by (master_seed, seed coordinate, ...)
(rule M2).

Parameter sets follow SURVEY.md §8(d.2) (derived from SPEC.md:222, 556 and
PAPER.md:17-18, 38); configs follow BASELINE.json ``configs`` as concretised in
SURVEY.md §8(d.3).  All times are integer microsecond ticks (rule M0).

Dict vocabulary (both consumers accept exactly this):

pipeline = {
  "roles": [ {"name", "n_instances", "cost": {h, alpha, beta, tau0, gamma, large},
              "inst_cost": None | [cost dict per instance],
              "max_num_seqs", "out": (fixed, num, den), "n_functions",
              "svc": "det"|"exp", "route": "jsq"|"rr"|"fixed"|"select", "route_fixed",
              "inbox_cap", "flight_cap", "wait_cap"} ... ],   # role 0 = the source
  "links": [ {"src", "dst", "net", "chunk", "mode": "batch"|"function"|"token"} ...],
  "feedback_role", "request_cap", "window", "slo" }
grid = { "candidates": [cand ...], "arrivals": [[arr per profile k] per rate i],
         "n_seeds", "seed_offset", "master_seed", "n_requests", "max_ticks",
         "series_stride", "series_slots", "series_windows" }
cand = { "kind": "static"|"adaptive", "modes": [mode|None per link],
         "ctl_links": [link ids], "metric": "busy"|"load", "lo", "hi", "dwell",
         "band": [mode_low, mode_mid, mode_high], "route": None|"jsq"|"rr",
         "batch_roles": [role ids], "q_hi", "select_role": None|int, "policy_slo" }
arr = { "kind": "poisson"|"mmpp2"|"det"|"list", "gap": [M0, M1], "sojourn": [D0, D1],
        "list": [ticks], "prompt": (lo, hi), "output": (lo, hi) }
"""

import copy

MASTER_SEED = 260103197  # any fixed constant; recorded in results
W_DEFAULT = 1_000_000    # 1 s windows


def cost(h=0, alpha=5000, beta=50, tau0=15000, gamma=1000, large=0):
    return {"h": h, "alpha": alpha, "beta": beta, "tau0": tau0, "gamma": gamma, "large": large}


def role(name, n_instances=1, c=None, inst_cost=None, max_num_seqs=8, out=(0, 1, 1),
         n_functions=1, svc="det", route="jsq", route_fixed=0,
         inbox_cap=256, flight_cap=64, wait_cap=256):
    return {"name": name, "n_instances": n_instances, "cost": c if c is not None else cost(),
            "inst_cost": inst_cost, "max_num_seqs": max_num_seqs, "out": tuple(out),
            "n_functions": n_functions, "svc": svc, "route": route, "route_fixed": route_fixed,
            "inbox_cap": inbox_cap, "flight_cap": flight_cap, "wait_cap": wait_cap}


def link(src, dst, net=1000, chunk=16, mode="batch", pacing_gap=0):
    return {"src": src, "dst": dst, "net": net, "chunk": chunk, "mode": mode, "pacing_gap": pacing_gap}


def pipeline(roles, links, feedback_role=None, request_cap=256, window=W_DEFAULT, slo=8_000_000):
    return {"roles": roles, "links": links,
            "feedback_role": len(roles) - 1 if feedback_role is None else feedback_role,
            "request_cap": request_cap, "window": window, "slo": slo}


def poisson(mean_gap, prompt=(64, 256), output=(128, 128)):
    return {"kind": "poisson", "gap": [int(mean_gap), 0], "sojourn": [0, 0], "list": [],
            "prompt": tuple(prompt), "output": tuple(output)}


def det(gap, prompt=(64, 256), output=(128, 128)):
    return {"kind": "det", "gap": [int(gap), 0], "sojourn": [0, 0], "list": [],
            "prompt": tuple(prompt), "output": tuple(output)}


def arr_list(ticks, prompt=(4, 4), output=(4, 4)):
    return {"kind": "list", "gap": [0, 0], "sojourn": [0, 0], "list": [int(t) for t in ticks],
            "prompt": tuple(prompt), "output": tuple(output)}


def mmpp2(gap_lo, gap_hi, soj_lo, soj_hi, prompt=(64, 256), output=(128, 128)):
    return {"kind": "mmpp2", "gap": [int(gap_lo), int(gap_hi)], "sojourn": [int(soj_lo), int(soj_hi)],
            "list": [], "prompt": tuple(prompt), "output": tuple(output)}


def static(*modes):
    return {"kind": "static", "modes": list(modes), "ctl_links": [], "metric": "busy",
            "lo": 400, "hi": 800, "dwell": 1, "band": ["token", "function", "batch"],
            "route": None, "batch_roles": [], "q_hi": 2, "select_role": None, "policy_slo": 0}


def adaptive(modes, ctl_links=(0,), metric="busy", lo=400, hi=800, dwell=1,
             band=("token", "function", "batch"), route=None, batch_roles=(), q_hi=2,
             select_role=None, policy_slo=0):
    return {"kind": "adaptive", "modes": list(modes), "ctl_links": list(ctl_links), "metric": metric,
            "lo": lo, "hi": hi, "dwell": dwell, "band": list(band), "route": route,
            "batch_roles": list(batch_roles), "q_hi": q_hi, "select_role": select_role,
            "policy_slo": policy_slo}


def grid(candidates, arrivals, n_seeds=1, n_requests=1, seed_offset=0, master_seed=MASTER_SEED,
         max_ticks=0, series_stride=0, series_slots=0, series_windows=0):
    # arrivals: list over rates i of list over profiles k
    arrivals = [a if isinstance(a, list) else [a] for a in arrivals]
    return {"candidates": candidates, "arrivals": arrivals, "n_seeds": n_seeds,
            "seed_offset": seed_offset, "master_seed": master_seed, "n_requests": n_requests,
            "max_ticks": max_ticks, "series_stride": series_stride, "series_slots": series_slots,
            "series_windows": series_windows}


def grid_size(g):
    return len(g["candidates"]) * len(g["arrivals"]) * len(g["arrivals"][0]) * g["n_seeds"]


# --------------------------------------------------------------------------------------------
# Parameter sets
# --------------------------------------------------------------------------------------------

def p2_spec(mode="batch", chunk=16, n_functions=4):
    """Developer -> tester with SPEC defaults."""
    dev = role("dev", c=cost(h=0), max_num_seqs=8, n_functions=n_functions)
    tester = role("tester", c=cost(h=1000), max_num_seqs=8, out=(0, 1, 2))
    return pipeline([dev, tester], [link(0, 1, net=1000, chunk=chunk, mode=mode)])


def p2_x(mode="function", request_cap=128):
    """Calibrated dev -> tester set where no static mode dominates."""
    dev = role("dev", c=cost(h=0), max_num_seqs=16, n_functions=4,
               inbox_cap=request_cap, wait_cap=request_cap)
    tester = role("tester", c=cost(h=20000), max_num_seqs=8, out=(0, 1, 1),
                  inbox_cap=256, flight_cap=64, wait_cap=512)   # wait <= R_cap * F = 512 never overflows
    return pipeline([dev, tester], [link(0, 1, net=1000, chunk=4, mode=mode)],
                    request_cap=request_cap)


def p4_chain(mode="batch", request_cap=128):
    """planner(1) -> coder(2) -> tester(2) -> reviewer(1)."""
    planner = role("planner", 1, cost(h=0), n_functions=2, inbox_cap=request_cap, wait_cap=request_cap)
    coder = role("coder", 2, cost(h=5000), out=(0, 2, 1), n_functions=4, inbox_cap=256, wait_cap=256)
    tester = role("tester", 2, cost(h=5000), out=(0, 1, 2), n_functions=2, inbox_cap=256, wait_cap=256)
    reviewer = role("reviewer", 1, cost(h=5000), out=(32, 1, 4), inbox_cap=512, wait_cap=512)
    links = [link(0, 1, chunk=16, mode=mode), link(1, 2, chunk=16, mode=mode),
             link(2, 3, chunk=16, mode=mode)]
    return pipeline([planner, coder, tester, reviewer], links, request_cap=request_cap)


LARGE = cost(h=0, alpha=5000, beta=50, tau0=15000, gamma=1000, large=1)
SMALL = cost(h=0, alpha=2000, beta=20, tau0=6000, gamma=400, large=0)


def p2_ms(request_cap=128):
    """Model selection: dev role = {LARGE, SMALL} instances, SELECT routing."""
    dev = role("dev", 2, LARGE, inst_cost=[dict(LARGE), dict(SMALL)], max_num_seqs=8,
               n_functions=4, route="select", inbox_cap=request_cap, wait_cap=request_cap)
    tester = role("tester", c=cost(h=1000), max_num_seqs=8, out=(0, 1, 2), inbox_cap=256, wait_cap=256)
    return pipeline([dev, tester], [link(0, 1, chunk=16, mode="batch")], request_cap=request_cap,
                    slo=6_000_000)


def toy_ht(mode):
    """HT-1..HT-3 toy pipeline."""
    dev = role("dev", c=cost(h=0, alpha=5, beta=1, tau0=10, gamma=2), max_num_seqs=2, n_functions=2)
    tester = role("tester", c=cost(h=3, alpha=5, beta=1, tau0=10, gamma=2), max_num_seqs=2, out=(0, 1, 2))
    return pipeline([dev, tester], [link(0, 1, net=1, chunk=1, mode=mode)])


def tool1(service, svc="det", beta=0, request_cap=256):
    """Single tool (out = 0 items): Lindley recursion C_j = max(A_j, C_{j-1}) + S_j (HT-6)."""
    t = role("tool", c=cost(h=0, alpha=service, beta=beta, tau0=1, gamma=0), svc=svc,
             inbox_cap=request_cap, wait_cap=request_cap)
    return pipeline([t], [], request_cap=request_cap)


def tandem(s1, s2, d, svc="det", request_cap=256):
    """Two tools in tandem with network delay d (HT-6)."""
    t1 = role("tool1", c=cost(h=0, alpha=s1, beta=0, tau0=1, gamma=0), svc=svc,
              inbox_cap=request_cap, wait_cap=request_cap)
    t2 = role("tool2", c=cost(h=0, alpha=s2, beta=0, tau0=1, gamma=0), svc=svc, out=(0, 0, 1),
              inbox_cap=request_cap, flight_cap=request_cap, wait_cap=request_cap)
    return pipeline([t1, t2], [link(0, 1, net=d, chunk=1, mode="batch")], request_cap=request_cap)


# --------------------------------------------------------------------------------------------
# BASELINE.json configs
# --------------------------------------------------------------------------------------------

P2X_RATE_F = [0.1, 0.25, 0.4, 0.55, 0.7, 0.85, 1.0, 1.15]
P2X_GAPS = [3994000, 1597600, 998500, 726182, 570571, 469882, 399400, 347304]


def config1(n_seeds=16, n_requests=10_000, rates=None):
    """Config 1: 2-agent dev->tester, 3 static modes x 8 Poisson rates x 16 seeds, 10k requests."""
    gaps = P2X_GAPS if rates is None else [P2X_GAPS[i] for i in rates]
    cands = [static("batch"), static("function"), static("token")]
    return p2_x(), grid(cands, [poisson(m) for m in gaps], n_seeds=n_seeds, n_requests=n_requests)


def config2_candidates():
    out = []
    for lo in (200, 300, 400, 500):
        for hi in (600, 700, 800, 900):
            for d in (1, 2, 4, 8):
                out.append(adaptive(["function"], ctl_links=[0], lo=lo, hi=hi, dwell=d))
    return out


def config2(n_seeds=2048, n_requests=1000, series_stride=4096, series_windows=512):
    """Config 2: per-1 s-window mode control, 64 policies x 8 rates x 2048 seeds = 1M replicas."""
    return p2_x(), grid(config2_candidates(), [poisson(m) for m in P2X_GAPS], n_seeds=n_seeds,
                        n_requests=n_requests, series_stride=series_stride,
                        series_slots=(64 * 8 * n_seeds + series_stride - 1) // series_stride if series_stride else 0,
                        series_windows=series_windows)


def config3_candidates():
    out = []
    for m in ("batch", "function", "token", "adaptive"):
        for r in ("rr", "jsq"):
            for bc in (False, True):
                roles = [1, 2] if bc else []
                if m == "adaptive":
                    out.append(adaptive(["function"] * 3, ctl_links=[0, 1, 2], route=r, batch_roles=roles,
                                        q_hi=2, policy_slo=8_000_000))
                elif bc:
                    out.append(adaptive([m] * 3, ctl_links=[], route=r, batch_roles=roles, q_hi=2,
                                        policy_slo=8_000_000))
                else:
                    c = static(m, m, m)
                    c["route"] = r
                    out.append(c)
    return out


def config3(n_seeds=4096, n_requests=1000):
    """Config 3: 4-agent DAG, routing over 2 replicas, SLO batch control; 16 x 16 x 4096 = 1M."""
    gaps = [round(197000 / (0.075 * k)) for k in range(1, 17)]
    return p4_chain(), grid(config3_candidates(), [poisson(m, output=(64, 64)) for m in gaps],
                            n_seeds=n_seeds, n_requests=n_requests)


def config4_candidates():
    out = []
    for lo in range(100, 900, 50):
        for delta in range(50, 850, 50):
            for d in (1, 2, 4, 8):
                for slo_half_s in range(6, 22):  # 3.0 .. 10.5 s step 0.5
                    out.append(adaptive(["batch"], ctl_links=[], lo=lo, hi=min(1000, lo + delta), dwell=d,
                                        select_role=0, policy_slo=slo_half_s * 500_000))
    return out


def config4(n_seeds=16, n_requests=1000, candidates=None):
    """Config 4: bursty MMPP-2 + model selection, 16384 x 16 x 4 x 16 = 16.7M replicas."""
    cands = config4_candidates() if candidates is None else candidates
    arrs = []
    for q in range(1, 17):
        lam = 0.25 * q
        row = []
        for b in (2, 4, 8, 16):
            m_lo = round(1e6 * (0.75 + 0.25 * b) / lam)
            row.append(mmpp2(m_lo, round(m_lo / b), 60_000_000, 20_000_000))
        arrs.append(row)
    return p2_ms(), grid(cands, arrs, n_seeds=n_seeds, n_requests=n_requests)


MAPPINGS = {"TFB": ("token", "function", "batch"), "FFB": ("function", "function", "batch"),
            "FBB": ("function", "batch", "batch"), "TBB": ("token", "batch", "batch")}


def config5_candidates(n=4096):
    out = [static("batch"), static("function"), static("token")]
    for name in ("TFB", "FFB", "FBB", "TBB"):
        for d in (1, 2, 4, 8):
            for lo in range(100, 900, 50):
                for delta in range(50, 850, 50):
                    if len(out) >= n:
                        return out
                    out.append(adaptive(["function"], ctl_links=[0], lo=lo, hi=min(1000, lo + delta),
                                        dwell=d, band=MAPPINGS[name]))
    return out


def config5(n_seeds=128, n_requests=1000, n_rates=128, n_candidates=4096):
    """Config 5: full strategy x rate x seed x policy sweep, 4096 x 128 x 128 = 64M replicas."""
    gaps = [round(399400 / (k / 100)) for k in range(1, n_rates + 1)]
    return p2_x(), grid(config5_candidates(n_candidates), [poisson(m) for m in gaps], n_seeds=n_seeds,
                        n_requests=n_requests)


def with_requests(g, n):
    g = copy.deepcopy(g)
    g["n_requests"] = n
    return g


def sample_ids(n_total, n_sample=4096):
    """Deterministic sample: every floor(R/n)-th id plus the extremes."""
    if n_total <= n_sample:
        return list(range(n_total))
    step = n_total // n_sample
    ids = sorted(set(list(range(0, n_total, step))[: n_sample - 1] + [n_total - 1]))
    return ids


# --------------------------------------------------------------------------------------------
# f1: KV-cache transfer + controller hints + load balancing (Fig. 6; rules M21-M24)
# --------------------------------------------------------------------------------------------
KV_POLICIES = ("affinity", "recompute", "posthoc", "hint")


def with_kv(cand, kv):
    c = dict(cand)
    c["kv"] = kv
    return c


def p2_kv(ctx_tokens=4000, tau_xfer=20, home_skew=750, request_cap=128):
    """One software-engineering agent feeding two tester instances that hold per-request KV context
    ("one instance of the software engineering agent and two instances of the testing
    agent").  tau_xfer = 0.02 ms/token and prefill 0.05 ms/token as SPEC.md:222; a request's context
    lives on tester 0 with probability home_skew/1000 (hot sessions), else on a uniform tester."""
    dev = role("dev", c=cost(h=0), max_num_seqs=32, n_functions=4, inbox_cap=request_cap, wait_cap=request_cap)
    tester = role("tester", 2, cost(h=1000), max_num_seqs=8, out=(0, 1, 1), route="jsq",
                  inbox_cap=256, flight_cap=64, wait_cap=256)
    p = pipeline([dev, tester], [link(0, 1, net=1000, chunk=16, mode="batch")], request_cap=request_cap,
                 slo=10_000_000)
    p["kv"] = {"role": 1, "ctx_tokens": ctx_tokens, "tau_xfer": tau_xfer, "home_skew": home_skew}
    return p


def config_kv(n_seeds=8, n_requests=1000, gaps=(1000000, 500000, 350000, 280000, 240000, 210000)):
    """Simulated Fig. 6: no load balancing (affinity) vs JSQ with recompute / post-hoc transfer /
    hinted transfer, over request rates."""
    cands = [with_kv(static("batch"), k) for k in KV_POLICIES]
    return p2_kv(), grid(cands, [poisson(m) for m in gaps], n_seeds=n_seeds, n_requests=n_requests)


# ------------------------------------------------------------------ f2: priority classes and admission
def with_classes(arrival, interactive_permille):
    """An arrival profile whose requests are interactive with probability permille/1000 (M26)."""
    a = copy.deepcopy(arrival)
    a["interactive"] = int(interactive_permille)
    return a


def with_prio(cand, prio=True, admit=False, admit_band=(400, 800)):
    """Candidate with M27 priority service and/or the M28 admission gate (the gate needs ADAPTIVE)."""
    c = copy.deepcopy(cand)
    c["prio"] = bool(prio)
    c["admit"] = bool(admit)
    c["admit_band"] = tuple(admit_band)
    if admit:
        c["kind"] = "adaptive"
    return c


def config_prio(n_seeds=8, n_requests=1000, interactive=300,
                gaps=(1597600, 726182, 469882, 399400, 347304)):
    """f2 workload: P2-X with an interactive share; FIFO vs interactive-first service x admission gate
    (PAPER.md:49/126 pipeline-wide prioritization, "admit only high-priority requests under
    load") x BATCH / TOKEN."""
    cands = []
    for mode in ("batch", "token"):
        for prio in (False, True):
            for admit in (False, True):
                cands.append(with_prio(static(mode), prio, admit, (500, 850)))
    arrs = [with_classes(poisson(g), interactive) for g in gaps]
    return p2_x(), grid(cands, arrs, n_seeds=n_seeds, n_requests=n_requests)


# ------------------------------------------------------------------ f4: data-plane pacing
def with_pacing(cand, gap):
    """Candidate that dispatches every link's messages at least `gap` ticks apart (M30)."""
    c = copy.deepcopy(cand)
    c["pacing_gap"] = int(gap)
    return c


def with_stale_jsq(cand, stale=True):
    """Candidate whose JSQ routing ranks the loads polled at the last window close (M31)."""
    c = copy.deepcopy(cand)
    c["stale_jsq"] = bool(stale)
    return c


def config_pace(n_seeds=8, n_requests=1000, gaps=(1597600, 726182, 469882),
                pacing=(0, 2000, 8000, 20000)):
    """f4 workload: P2-X with token streaming / per-function pipelining, swept over the link pacing gap
    ("priorities, and pacing strategies")."""
    cands = [with_pacing(static(m), g) for m in ("token", "function", "batch") for g in pacing]
    return p2_x(), grid(cands, [poisson(m) for m in gaps], n_seeds=n_seeds, n_requests=n_requests)
