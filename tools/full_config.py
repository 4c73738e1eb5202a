"""A BASELINE config at full size on one GPU (config 5: 4096 x 128 x 128 = 67,108,864 replicas; config 4:
16384 x 16 x 4 x 16 = 16,777,216; config 3: 16 x 16 x 4096 = 1,048,576; all x 1000 requests): one
sdas_control_sweep + sdas_finalize, timed with CUDA events, and a deterministic sample of replicas
re-simulated by the oracle and compared field by field.  Prints one JSON line (a measurement record for
profiles/, not the bench contract).
usage: python tools/full_config.py <config3|config4|config5> [n_sample]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from bench import ClockSampler  # noqa: E402
from paper_2601_03197_b200 import sdas  # noqa: E402

cfg = sys.argv[1]
n_sample = int(sys.argv[2]) if len(sys.argv) > 2 else 256
pipe, grid = getattr(W, cfg)()
objective, slo = ("large_under_slo", 6_000_000) if cfg == "config4" else ("p99_e2e", 0)
R = W.grid_size(grid)
P = sdas.Pipeline(pipe)
gv = sdas.GridView(pipe, grid)
L = sdas.results_layout(P, gv)
res = sdas.Result(L, sdas.allocate(L, torch.device("cuda", 0), 0))
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
torch.cuda.synchronize()
clocks = ClockSampler(0)                                  # nvidia-smi clocks / throttle reasons during the run
clocks.start()
e[0].record()
sdas.control_sweep(P, gv, objective=objective, objective_slo=slo, result=res)
e[1].record()
sdas.finalize(P, gv, res, objective=objective, objective_slo=slo)
e[2].record()
torch.cuda.synchronize()
clk = clocks.stop()
k1k3_ms, fin_ms = e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2])
cnt, _ = res.cells()
F = {n: i for i, n in enumerate(sdas.CELL_FIELDS)}
tot = cnt.sum(0)
msg = int(tot[F["arrivals"]] + tot[F["deliveries"]])
des = msg + int(tot[F["recv_steps"]] + tot[F["decode_steps"]] + tot[F["window_closes"]])
out = {"workload": "%s full: %d replicas x %d requests, 1 GPU, objective %s" % (cfg, R, grid["n_requests"], objective),
       "k1_k3_ms": k1k3_ms, "k4_k5_ms": fin_ms, "replicas": int(tot[F["n_replicas"]]),
       "msg_events_per_s": msg / ((k1k3_ms + fin_ms) / 1e3), "des_events_per_s": des / ((k1k3_ms + fin_ms) / 1e3),
       "replicas_per_s": R / ((k1k3_ms + fin_ms) / 1e3), "k1_variant": L.k1_variant, "ring_s": L.ring_s,
       "warps_per_sm": L.warps_per_block * L.blocks_per_sm, "clocks": clk}
if n_sample:
    import oracle
    from gpu_parity import compare_summaries
    summ = res.summary()
    ids = np.asarray(W.sample_ids(R, n_sample), dtype=np.uint64)
    t0 = time.perf_counter()
    o = oracle.simulate(pipe, grid, ids=ids, records=False, hists=False)
    compare_summaries(summ[ids.astype(np.int64)], o["summary"], where="%s full sample" % cfg)
    out["oracle_sample"] = {"replicas": len(ids), "bit_exact": True, "seconds": time.perf_counter() - t0}
    out["best_row"] = res.best_row().tolist()[:8]
print(json.dumps(out), flush=True)
