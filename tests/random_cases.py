"""Seeded random pipelines / grids that combine the model's features (test infrastructure).

Each case: a DAG of 1-4 roles (fan-out <= 2, one in-link per role, 1-2 instances per role, JSQ / RR /
FIXED routing), LLM roles and tools (det / exp service), random costs, capacities, chunks, modes and
pacing gaps, Poisson / DET / MMPP-2 arrivals, and candidates mixing static modes, the three-band
controller (busy / load), SLO batch control, route overrides, M25 guards, f2 priority / admission
(with request classes) or f1 KV policies, pacing overrides and snapshot (stale) JSQ."""
import numpy as np

import workloads as W

OBJECTIVES = ["p99_e2e", "p50_e2e", "p99_ff", "throughput", "goodput", "p90_e2e", "p99_e2e_int"]
MODES = ["batch", "function", "token"]


def make_case(seed):
    r = np.random.default_rng(1000 + seed)
    rs = np.random.default_rng(5000 + seed)
    n_roles = int(r.integers(1, 5))
    n_inst = [1] * n_roles
    for k in range(1, n_roles):
        if r.random() < 0.45:
            n_inst[k] = 2
    roles, links, fan = [], [], [0] * n_roles
    for k in range(n_roles):
        tool = k > 0 and r.random() < 0.3
        c = W.cost(h=int(r.choice([0, 500, 5000])), alpha=int(r.integers(500, 6000)), beta=int(r.integers(0, 60)),
                   tau0=int(r.integers(2000, 16000)), gamma=int(r.integers(0, 1200)))
        out = (0, 0, 1) if tool else (int(r.choice([0, 8, 32])), int(r.choice([0, 1, 2])), int(r.choice([1, 2, 4])))
        if not tool and out[0] == 0 and out[1] == 0:
            out = (16, 0, 1)
        route = str(r.choice(["jsq", "rr", "fixed"])) if n_inst[k] > 1 else "jsq"
        roles.append(W.role("r%d" % k, n_inst[k], c, max_num_seqs=int(r.choice([1, 2, 4, 8, 16])),
                            out=out, n_functions=int(r.integers(1, 5)),
                            svc=str(r.choice(["det", "exp"])) if tool else "det", route=route,
                            route_fixed=int(r.integers(0, n_inst[k])),
                            inbox_cap=int(r.choice([64, 128, 256])), flight_cap=int(r.choice([32, 64, 128])),
                            wait_cap=int(r.choice([64, 256, 512]))))
        if k > 0:
            parents = [q for q in range(k) if fan[q] < 2]
            q = int(r.choice(parents))
            fan[q] += 1
            links.append(W.link(q, k, net=int(r.choice([1, 100, 1000])), chunk=int(r.choice([1, 4, 16])),
                                mode=str(r.choice(MODES)), pacing_gap=int(r.choice([0, 0, 0, 500, 3000]))))
    p = W.pipeline(roles, links, feedback_role=int(r.integers(0, n_roles)),
                   request_cap=int(r.choice([16, 64, 128])), window=int(r.choice([200_000, 1_000_000])),
                   slo=int(r.choice([2_000_000, 8_000_000])))
    multi = [k for k in range(1, n_roles) if n_inst[k] > 1]
    kv = bool(multi) and r.random() < 0.25
    if kv:
        p["kv"] = {"role": int(r.choice(multi)), "ctx_tokens": int(r.choice([500, 2000])), "tau_xfer": 20,
                   "home_skew": int(r.choice([0, 500, 1000]))}
    cls = (not kv) and r.random() < 0.4
    arrs = []
    for _ in range(int(r.integers(1, 3))):
        kind = r.choice(["poisson", "poisson", "det", "mmpp2"])
        gap = int(r.integers(60_000, 600_000))
        prompt = (int(r.integers(1, 64)), int(r.integers(64, 300)))
        output = (0, 0) if r.random() < 0.1 else (int(r.integers(1, 32)), int(r.integers(32, 160)))
        if kind == "poisson":
            a = W.poisson(gap, prompt=prompt, output=output)
        elif kind == "det":
            a = W.det(gap, prompt=prompt, output=output)
        else:
            a = W.mmpp2(gap, gap // 4, 3_000_000, 1_000_000, prompt=prompt, output=output)
        if cls:
            a = W.with_classes(a, int(r.choice([200, 500])))
        arrs.append(a)
    nl = len(links)
    cands = []
    for _ in range(int(r.integers(3, 7))):
        modes = [str(r.choice(MODES)) for _ in range(max(1, nl))]
        if r.random() < 0.5 or nl == 0:
            c = W.static(*modes)
        else:
            ctl = [l for l in range(nl) if r.random() < 0.7] or [0]
            c = W.adaptive(modes, ctl_links=ctl, metric=str(r.choice(["busy", "load"])),
                           lo=int(r.integers(100, 500)), hi=int(r.integers(500, 950)), dwell=int(r.integers(1, 4)),
                           batch_roles=[k for k in range(n_roles) if r.random() < 0.3], q_hi=int(r.integers(1, 4)),
                           policy_slo=int(r.choice([1_000_000, 4_000_000])))
        if any(n > 1 for n in n_inst) and r.random() < 0.3:
            c["route"] = str(r.choice(["jsq", "rr"]))
        if nl and r.random() < 0.25:
            c["kind"] = "adaptive"
            c["guard_links"] = [l for l in range(nl) if r.random() < 0.6] or [0]
            c["guard_pct"] = int(r.choice([90, 99]))
            c["policy_slo"] = int(r.choice([1_000_000, 3_000_000]))
        if cls:
            c = W.with_prio(c, prio=bool(r.random() < 0.6), admit=bool(r.random() < 0.4),
                            admit_band=(int(r.integers(100, 500)), int(r.integers(500, 950))))
        if kv:
            c = W.with_kv(c, str(r.choice(list(W.KV_POLICIES))))
        if nl and r.random() < 0.2:
            c = W.with_pacing(c, int(r.choice([0, 1000, 5000])))
        if rs.random() < 0.3:                        # M31 (own stream: earlier draws are unchanged)
            c = W.with_stale_jsq(c)
        cands.append(c)
    g = W.grid(cands, arrs, n_seeds=2, n_requests=int(r.choice([60, 150])),
               max_ticks=int(r.choice([0, 0, 0, 40_000_000])))
    obj = str(r.choice(OBJECTIVES[:6] + (["p99_e2e_int"] if cls else [])))
    return p, g, obj


def make_lean_case(seed):
    """make_case(seed) with the level-0 / level-1 features stripped (KV, classes, pacing, LOAD metric,
    truncation, extra instances, fan-out, route overrides, stale JSQ), so it runs on the LEAN K1 and its
    shortcuts (lazy deliveries, silent RECVs, emit-ahead, chained resume) while keeping
    the random costs, capacities, modes, controllers and arrivals."""
    p, g, obj = make_case(seed)
    p.pop("kv", None)
    for r in p["roles"]:
        r["n_instances"] = 1
        r["route"] = "jsq"
        r["inst_cost"] = None
    for k, l in enumerate(p["links"]):
        l["src"], l["dst"], l["pacing_gap"] = k, k + 1, 0
    for a in g["arrivals"]:
        for x in a:
            x.pop("interactive", None)
    for c in g["candidates"]:
        for key in ("prio", "admit", "admit_band", "kv", "pacing_gap", "stale_jsq"):
            c.pop(key, None)
        c["route"] = None
        if c.get("metric") == "load":
            c["metric"] = "busy"
        c["select_role"] = None
    g["max_ticks"] = 0
    return p, g, ("p99_e2e" if obj == "p99_e2e_int" else obj)
