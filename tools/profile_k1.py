"""One K1 (+K3/K4/K5) launch of a BASELINE config grid, for ncu captures (not a bench number).
--seeds sets the size (config 2 / 3 at 2048 / 4096 seeds = the bench's 1M replicas); --records / --series
turn on the per-request records (the metric flush) and the bench's mode series."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2601_03197_b200 import sdas  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seeds", type=int, default=16)
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--requests", type=int, default=1000)
ap.add_argument("--records", action="store_true")
ap.add_argument("--series", action="store_true")
a = ap.parse_args()
if a.config == 2:
    pipe, grid = W.config2(n_seeds=a.seeds, n_requests=a.requests, series_stride=4096 if a.series else 0)
elif a.config == 1:
    pipe, grid = W.config1(n_seeds=a.seeds, n_requests=a.requests)
elif a.config == 3:
    pipe, grid = W.config3(n_seeds=a.seeds, n_requests=a.requests)
flags = (sdas.FLAG_RECORDS if a.records else 0) | (sdas.FLAG_SERIES if a.series and grid["series_stride"] else 0)
P = sdas.Pipeline(pipe)
gv = sdas.GridView(pipe, grid, flags=flags)
r = sdas.control_sweep(P, gv, objective="p99_e2e")
sdas.finalize(P, gv, r)
torch.cuda.synchronize()
cnt, _ = r.cells()
F = {n: i for i, n in enumerate(sdas.CELL_FIELDS)}
tot = cnt.sum(0)
des = int(tot[F["arrivals"]] + tot[F["deliveries"]] + tot[F["recv_steps"]] + tot[F["decode_steps"]] +
          tot[F["window_closes"]])
print("replicas", int(tot[F["n_replicas"]]), "des_events", des, "msg_events", int(tot[F["arrivals"]] + tot[F["deliveries"]]),
      "layout smem/replica", r.layout.smem_per_replica, "wpb", r.layout.warps_per_block, "bps", r.layout.blocks_per_sm,
      "flags", flags, "n_requests", a.requests)
