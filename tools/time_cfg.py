"""A/B timing of K1 on a BASELINE config under each specialisation level (not a bench number).
usage: python tools/time_cfg.py <config> <n_seeds> [reps]   (prints: level k1_variant ms)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2601_03197_b200 import sdas  # noqa: E402

cfg, seeds = sys.argv[1], int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
kw = {"series_stride": 0} if cfg == "config2" else {}
pipe, grid = getattr(W, cfg)(n_seeds=seeds, **kw)
P = sdas.Pipeline(pipe)
for r in range(reps):
    for name, fl in (("auto", 0), ("mid", sdas.FLAG_MID), ("generic", sdas.FLAG_GENERIC)):
        gv = sdas.GridView(pipe, grid, flags=fl)
        res = sdas.simulate(P, gv)                       # warm (allocates)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sdas.simulate(P, gv, result=res)
        e1.record()
        torch.cuda.synchronize()
        print(cfg, name, res.layout.k1_variant, res.layout.ring_s, round(e0.elapsed_time(e1), 1), flush=True)
