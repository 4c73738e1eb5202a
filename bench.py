#!/usr/bin/env python
"""Benchmark of the SDAS strategy-simulation hot path (BASELINE.json metric: simulated message events/s
and replicas/s at 1/2/4/8 B200, p99 exactness).

Workload at N=1: BASELINE config 2 -- the P2-X developer->tester pipeline with the metrics-driven
controller switching the message granularity per 1 s window: 64 policies x 8 Poisson rates x 2048
seeds = 1,048,576 replicas of 1000 requests.  One step = one pass of the whole hot
path over one batch of fresh synthetic input (seed offset advances every step): K1 simulation with
in-loop control + metrics + exact percentiles + cell merge, K3 per-group argmin, the NCCL collective
(N>1), K4/K5 pooled per-rate argmin.  Scaling is weak: each GPU simulates 1M replicas per step.

  python bench.py [--gpus N --steps K --warmup W]          # product (libsdas, sm_100a)
  python bench.py --impl reference ...                      # the CPU oracle on host cores
Multi-GPU: python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402

METRIC = "simulated message events/sec"
UNIT = "message_events/s"
ALG_WARP_INSTR_PER_DES_EVENT = 20   # SURVEY.md §8(d.4) algorithmic floor, DESIGN.md §"Roofline"


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


DEFAULT_SEEDS = {2: 2048, 3: 4096, 4: 1, 5: 2}           # 1,048,576 replicas per GPU in every config
OBJECTIVE = {4: ("large_under_slo", 6_000_000)}           # config 4 ranks by the large fraction under the SLO


def workload(args, world):
    """(pipeline, grid) of the timed workload: BASELINE config 2 (default) or 3, or the full config 4 / 5 grid
    (every candidate x rate x profile) with fewer seeds: 1 (config 4) / 2 (config 5) per GPU = 1M replicas."""
    seeds = args.seeds * world                          # weak scaling: args.seeds per GPU
    if args.config == 3:
        return W.config3(n_seeds=seeds, n_requests=args.requests)
    if args.config == 4:
        return W.config4(n_seeds=seeds, n_requests=args.requests)
    if args.config == 5:
        return W.config5(n_seeds=seeds, n_requests=args.requests)
    # the per-window mode / queue series of every 4096th replica is written in the timed step
    return W.config2(n_seeds=seeds, n_requests=args.requests, series_stride=4096, series_windows=512)


def workload_name(args):
    if args.config == 4:
        return ("config4 grid at %d seed(s)/GPU: P2-MS dev{LARGE,SMALL}->tester, MMPP-2 bursts, model selection, "
                "16384 policies x 16 mean rates x 4 burst ratios, N=%d requests/replica (objective large_under_slo, "
                "6 s); the full 16M-replica config is 16 seeds" % (args.seeds, args.requests))
    if args.config == 5:
        return ("config5 grid at %d seeds/GPU: P2-X, 4096 strategies (3 static + 4093 adaptive policies) x 128 "
                "rates, N=%d requests/replica; the full 64M-replica config is 128 seeds" % (args.seeds, args.requests))
    if args.config == 3:
        return ("config3: P4-chain planner->coder(2)->tester(2)->reviewer, 16 candidates (modes x RR/JSQ routing x "
                "SLO batch control) x 16 Poisson rates x %d seeds/GPU, N=%d requests/replica" % (args.seeds,
                                                                                                 args.requests))
    return ("config2: P2-X dev->tester, per-1s-window mode control, 64 policies x 8 Poisson rates x %d seeds/GPU, "
            "N=%d requests/replica" % (args.seeds, args.requests))


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                       "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        self.f.seek(0)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_baseline(args, target_s=15.0):
    """The oracle as it stands, on this host's cores, on a bounded sample of the same workload."""
    import oracle
    pipe, grid = workload(args, 1)
    R = W.grid_size(grid)
    threads = os.cpu_count() or 1
    probe = W.sample_ids(R, 128)
    t0 = time.perf_counter()
    oracle.simulate(pipe, grid, ids=probe, threads=threads, records=False, hists=False)
    dt = max(1e-3, time.perf_counter() - t0)
    n = int(min(R, max(128, 128 * target_s / dt)))
    ids = W.sample_ids(R, n)
    t0 = time.perf_counter()
    o = oracle.simulate(pipe, grid, ids=ids, threads=threads, records=False, hists=False)
    dt = time.perf_counter() - t0
    s = o["summary"]
    msg = int(s["arrivals"].astype(np.int64).sum() + s["deliveries"].astype(np.int64).sum())
    des = msg + int(s["recv_steps"].astype(np.int64).sum() + s["decode_steps"].astype(np.int64).sum() +
                    s["window_closes"].astype(np.int64).sum())
    ids1 = W.sample_ids(R, 48)                                 # single-thread rate
    t1 = time.perf_counter()
    s1 = oracle.simulate(pipe, grid, ids=ids1, threads=1, records=False, hists=False)["summary"]
    dt1 = time.perf_counter() - t1
    msg1 = int(s1["arrivals"].astype(np.int64).sum() + s1["deliveries"].astype(np.int64).sum())
    return {"value": msg / dt, "unit": UNIT, "cores": threads, "kind": "oracle",
            "single_thread": {"value": msg1 / dt1, "unit": UNIT, "sample": "%d replicas" % len(ids1)},
            "sample": "%d of %d config-%d replicas (every floor(R/n)-th id + last), N=%d requests, %.1f s" % (
                len(ids), R, args.config, args.requests, dt),
            "replicas_per_s": len(ids) / dt, "des_events_per_s": des / dt, "seconds": dt}


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    import oracle
    pipe, grid = workload(args, 1)
    R = W.grid_size(grid)
    threads = os.cpu_count() or 1
    per_step = args.ref_sample
    tot_msg, tot_t, tot_rep = 0, 0.0, 0
    for k in range(args.warmup + args.steps):
        ids = (np.asarray(W.sample_ids(R, per_step), dtype=np.uint64) + k) % R   # fresh replicas each step
        t0 = time.perf_counter()
        o = oracle.simulate(pipe, grid, ids=ids, threads=threads, records=False, hists=False)
        dt = time.perf_counter() - t0
        if k >= args.warmup:
            s = o["summary"]
            tot_msg += int(s["arrivals"].astype(np.int64).sum() + s["deliveries"].astype(np.int64).sum())
            tot_t += dt
            tot_rep += len(ids)
    v = tot_msg / tot_t
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000 * tot_t / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": workload_name(args) + " (sampled)", "sample_per_step": per_step},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": "%d replicas per step of %d (config %d)" % (per_step, R, args.config)},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "replicas_per_s": tot_rep / tot_t}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="sdas", choices=["sdas", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=[2, 3, 4, 5],
                    help="BASELINE config timed: 2 (default, the headline), 3 (4-agent routed DAG), or a 1M-replica "
                         "per GPU slice of 4 (MMPP + model selection) / 5 (full strategy sweep)")
    ap.add_argument("--seeds", type=int, default=None, help="seeds per GPU (default: 1M replicas per GPU)")
    ap.add_argument("--requests", type=int, default=1000)
    ap.add_argument("--ref-sample", type=int, default=512)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-flush-leg", action="store_true", help="skip the FLAG_RECORDS metric-flush leg")
    ap.add_argument("--generic", action="store_true", help="A/B only: disable the K1 specialisations")
    ap.add_argument("--mid", action="store_true", help="A/B only: at most the level-1 K1 specialisation")
    args = ap.parse_args()
    if args.seeds is None:
        args.seeds = DEFAULT_SEEDS[args.config]
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    from paper_2601_03197_b200 import parallel, sdas

    rank, world, local = env_rank()
    assert world == args.gpus, "launch N>1 under torch.distributed.run with --nproc-per-node N"
    # SDAS_BENCH_BACKEND=gloo: test hook only (tests/test_gpu_bench_multirank.py) -- several ranks share the
    # box's GPU(s) with host-staged collectives, to exercise the N > 1 code path on a one-GPU box; the driver's
    # runs use NCCL, one rank per GPU
    backend = os.environ.get("SDAS_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    pipe, grid = workload(args, world)
    P = sdas.Pipeline(pipe)
    S_total = grid["n_seeds"]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)     # > 126 MB L2
    stream = torch.cuda.current_stream(dev)

    def grid_for(step):
        g = dict(grid)
        g["seed_offset"] = step * S_total                              # fresh synthetic input per step
        return g

    kflags = (sdas.FLAG_GENERIC if args.generic else 0) | (sdas.FLAG_MID if args.mid else 0)
    if grid["series_stride"]:
        kflags |= sdas.FLAG_SERIES
    obj, obj_slo = OBJECTIVE.get(args.config, ("p99_e2e", 0))
    gv0 = sdas.GridView(pipe, grid_for(0), flags=kflags, rank=rank, world=world)
    L = sdas.results_layout(P, gv0)
    res = sdas.Result(L, sdas.allocate(L, dev, kflags))
    acc_local = torch.zeros(sdas.NCNT, dtype=torch.int64, device=dev)
    acc_global = torch.zeros(sdas.NCNT, dtype=torch.int64, device=dev)

    def one_step(step, timed, ev):
        gv = sdas.GridView(pipe, grid_for(step), flags=kflags, rank=rank, world=world)
        res.t["cell_cnt"].zero_()
        res.t["cell_hist"].zero_()
        flush.fill_(step & 0xFF)                                       # L2 flush before the step
        ev[0].record(stream)
        sdas.simulate(P, gv, device=dev, result=res)                   # K1
        ev[1].record(stream)
        sdas.group_argmin(P, gv, res, objective=obj, objective_slo=obj_slo, device=dev)  # K3
        ev[2].record(stream)
        cnt_view = res.t["cell_cnt"][: L.n_cells * sdas.NCNT * 8].view(torch.int64).view(L.n_cells, sdas.NCNT)
        if timed:
            acc_local.add_(cnt_view.sum(0))
        ev[3].record(stream)
        if world > 1:                                                  # the one exchange step
            parallel.reduce_cells(res)
            parallel.gather_best_groups(res, L.n_groups, rank, world)
        ev[4].record(stream)
        sdas.finalize(P, gv, res, objective=obj, objective_slo=obj_slo, device=dev)     # K4 + K5
        ev[5].record(stream)
        if timed:
            acc_global.add_(cnt_view.sum(0))

    mk = lambda: [torch.cuda.Event(enable_timing=True) for _ in range(6)]  # noqa: E731
    for k in range(args.warmup):
        one_step(1000 + k, False, mk())
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    evs = [mk() for _ in range(args.steps)]
    for k in range(args.steps):
        one_step(k, True, evs[k])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    step_ms = [e[0].elapsed_time(e[5]) - e[2].elapsed_time(e[3]) for e in evs]    # excludes accounting adds
    k1_ms = [e[0].elapsed_time(e[1]) for e in evs]
    k3_ms = [e[1].elapsed_time(e[2]) for e in evs]
    coll_ms = [e[3].elapsed_time(e[4]) for e in evs]
    fin_ms = [e[4].elapsed_time(e[5]) for e in evs]
    def max_over_ranks(v):                                             # device time, max over ranks
        x = torch.tensor([v], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        if world > 1:
            dist.all_reduce(x, op=dist.ReduceOp.MAX)
        return float(x.item())

    total_ms = max_over_ranks(sum(step_ms))
    loc = acc_local.cpu().numpy()
    glob = acc_global.cpu().numpy()
    if world == 1:
        glob = loc
    F = {n: i for i, n in enumerate(sdas.CELL_FIELDS)}
    msg = int(glob[F["arrivals"]] + glob[F["deliveries"]])
    des = msg + int(glob[F["recv_steps"]] + glob[F["decode_steps"]] + glob[F["window_closes"]])
    reps = int(glob[F["n_replicas"]])
    loc_des = int(loc[F["arrivals"]] + loc[F["deliveries"]] + loc[F["recv_steps"]] + loc[F["decode_steps"]] +
                  loc[F["window_closes"]])
    value = msg / (total_ms / 1e3)

    # roofline of the dominant kernel K1: integer-issue bound (no tensor cores, HBM traffic << roof)
    pk = peaks()
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    f_mhz = float(pk.get("sm_max_mhz", 1965.0))
    peak = n_sm * 4 * f_mhz * 1e6 / 1e12                               # warp-instructions per second (x1e12)
    k1_avg_s = statistics.mean(k1_ms) / 1e3
    achieved = ALG_WARP_INSTR_PER_DES_EVENT * (loc_des / args.steps) / k1_avg_s / 1e12
    traffic = None
    issue = None
    try:   # DRAM bytes of one K1 launch of exactly this workload, measured by ncu at bench size
        dm = json.load(open(os.path.join(ROOT, "profiles", "k1_dram_bench_config%d.json" % args.config)))
        if dm["replicas"] == reps // args.steps and dm["n_requests"] == args.requests and world == 1:
            traffic = dm["dram_bytes_per_launch"]
    except Exception:
        pass
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "k1_ncu_summary.json" if args.config == 2 else
                                           "k1_ncu_summary_config%d.json" % args.config)))
        if prof.get("warp_instr_per_des_event") is not None:
            # the same roofline with the ncu-MEASURED instructions per DES event (profiles/): issue utilisation
            w = float(prof["warp_instr_per_des_event"])
            issue = {"warp_instr_per_des_event": w,
                     "achieved": w * (loc_des / args.steps) / k1_avg_s / 1e12,
                     "frac": w * (loc_des / args.steps) / k1_avg_s / 1e12 / peak}
    except Exception:
        pass

    e2e = None
    if not args.no_e2e:
        # end to end through the public API: host descriptors -> H2D (inside sdas_simulate), the whole
        # sweep + collective, D2H of every result (summaries, cells, best tables) into pinned memory
        pinned = {n: torch.empty(int(getattr(L, n + "_bytes")), dtype=torch.uint8, pin_memory=True)
                  for n in ("summary", "cell_cnt", "cell_hist", "best_group", "best_row") +
                  (("series",) if kflags & sdas.FLAG_SERIES else ())}
        h2d = 0
        e2e_ms = []
        for k in range(args.steps):
            g = grid_for(100 + k)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            flush.fill_(k & 0xFF)
            a.record(stream)
            res.t["cell_cnt"].zero_()
            res.t["cell_hist"].zero_()
            r2, table, _, gvk = parallel.sweep(pipe, g, objective=obj, objective_slo=obj_slo, rank=rank, world=world,
                                                device=dev, flags=kflags,
                                                result=res, pipeline=P)
            for n, h in pinned.items():
                h.copy_(res.t[n][: h.numel()], non_blocking=True)
            b.record(stream)
            b.synchronize()
            e2e_ms.append(a.elapsed_time(b))
            h2d = L.params_bytes
        d2h = sum(h.numel() for h in pinned.values())
        e2e = {"value": msg / (max_over_ranks(sum(e2e_ms)) / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h)}

    flush_leg = None
    if world == 1 and not args.no_flush_leg:
        # the metric flush with exact per-request records on (FLAG_RECORDS, SURVEY §8 d.4 "K2"): it is fused
        # into K1's finalize, so its HBM bytes are averaged over the K1 launch that produces them
        fflags = kflags | sdas.FLAG_RECORDS
        gvf = sdas.GridView(pipe, grid_for(500), flags=fflags)
        Lf = sdas.results_layout(P, gvf)
        rf = sdas.Result(Lf, sdas.allocate(Lf, dev, fflags))
        flush.fill_(7)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        sdas.simulate(P, gvf, device=dev, result=rf)
        b.record(stream)
        b.synchronize()
        ms = a.elapsed_time(b)
        per_rep = args.requests * 8 + sdas.SUMMARY_DTYPE.itemsize
        nbytes = Lf.n_local_replicas * per_rep
        gbs = nbytes / (ms / 1e3) / 1e9
        flush_leg = {"bytes_per_replica": per_rep, "bytes": nbytes, "k1_ms_with_records": ms,
                     "k1_ms_without_records": statistics.mean(k1_ms), "achieved_gbs": gbs,
                     "peak_gbs": float(pk.get("hbm_gbs", 7700.0)), "frac": gbs / float(pk.get("hbm_gbs", 7700.0)),
                     "note": "records (N x 8 B) + summary written by K1's fused finalize; GB/s = those bytes / the "
                             "K1 launch that writes them (the flush is not a separate phase)"}
        try:
            dmr = json.load(open(os.path.join(ROOT, "profiles", "k1_dram_bench_config%d_records.json" % args.config)))
            if dmr["replicas"] == Lf.n_local_replicas:
                flush_leg["dram_bytes_measured"] = dmr["dram_bytes_per_launch"]
        except Exception:
            pass
        del rf

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": workload_name(args),
                       "replicas_per_step": reps // args.steps, "n_requests": args.requests,
                       "l2": "flushed (256 MiB write) before every step",
                       "parallelism": "replica-grid dp%d (group-interleaved), %s all_reduce of cells" % (
                           world, "NCCL" if backend == "nccl" else backend)},
            "replicas_per_s": reps / (total_ms / 1e3),
            "des_events_per_s": des / (total_ms / 1e3),
            "events_per_step": {"message": msg // args.steps, "des": des // args.steps},
            "phase_ms": {"k1_simulate": statistics.mean(k1_ms), "k3_group_argmin": statistics.mean(k3_ms),
                         "collective": statistics.mean(coll_ms), "k4k5_finalize": statistics.mean(fin_ms)},
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "warp-instr/s x1e12",
                         "frac": achieved / peak, "traffic": traffic, "measured_issue": issue,
                         "note": "K1; achieved = %d algorithmic warp-instr per DES event (SURVEY §8d.4 floor) x "
                                 "DES events / K1 time; peak = %d SMs x 4 issue/clk x %.0f MHz (MEASURED_PEAKS "
                                 "sm_max_mhz)" % (ALG_WARP_INSTR_PER_DES_EVENT, n_sm, f_mhz)},
            "gpu_launches": 4 * args.steps,   # per timed step: K1, K3, K4, K5
            "clocks": clk,
            "e2e": e2e,
            "metric_flush": flush_leg,
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(args)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
