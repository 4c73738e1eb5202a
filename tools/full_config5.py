"""Config 5 at full size on one GPU: 4096 candidates x 128 rates x 128 seeds = 67,108,864 replicas x 1000
requests (BASELINE.json config 5), one sdas_control_sweep + sdas_finalize, timed with CUDA events, and a
deterministic sample of replicas re-simulated by the oracle and compared field by field.  Prints one
JSON line (a measurement record for profiles/, not the bench contract).
usage: python tools/full_config5.py [n_sample]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2601_03197_b200 import sdas  # noqa: E402

n_sample = int(sys.argv[1]) if len(sys.argv) > 1 else 256
pipe, grid = W.config5()
R = W.grid_size(grid)
P = sdas.Pipeline(pipe)
gv = sdas.GridView(pipe, grid)
L = sdas.results_layout(P, gv)
res = sdas.Result(L, sdas.allocate(L, torch.device("cuda", 0), 0))
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
torch.cuda.synchronize()
e[0].record()
sdas.control_sweep(P, gv, objective="p99_e2e", result=res)
e[1].record()
sdas.finalize(P, gv, res, objective="p99_e2e")
e[2].record()
torch.cuda.synchronize()
k1k3_ms, fin_ms = e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2])
cnt, _ = res.cells()
F = {n: i for i, n in enumerate(sdas.CELL_FIELDS)}
tot = cnt.sum(0)
msg = int(tot[F["arrivals"]] + tot[F["deliveries"]])
des = msg + int(tot[F["recv_steps"]] + tot[F["decode_steps"]] + tot[F["window_closes"]])
out = {"workload": "config5 full: 4096 x 128 x 1 x 128 = %d replicas x 1000 requests, 1 GPU" % R,
       "k1_k3_ms": k1k3_ms, "k4_k5_ms": fin_ms, "replicas": int(tot[F["n_replicas"]]),
       "msg_events_per_s": msg / ((k1k3_ms + fin_ms) / 1e3), "des_events_per_s": des / ((k1k3_ms + fin_ms) / 1e3),
       "replicas_per_s": R / ((k1k3_ms + fin_ms) / 1e3), "k1_variant": L.k1_variant}
if n_sample:
    import oracle
    from gpu_parity import compare_summaries
    summ = res.summary()
    ids = np.asarray(W.sample_ids(R, n_sample), dtype=np.uint64)
    t0 = time.perf_counter()
    o = oracle.simulate(pipe, grid, ids=ids, records=False, hists=False)
    compare_summaries(summ[ids.astype(np.int64)], o["summary"], where="config5 full sample")
    out["oracle_sample"] = {"replicas": len(ids), "bit_exact": True, "seconds": time.perf_counter() - t0}
    out["best_row"] = res.best_row().tolist()[:8]
print(json.dumps(out), flush=True)
