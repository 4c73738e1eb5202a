"""A/B timing of K1 (auto specialisation) for prebuilt libraries: SDAS_LIB=<lib> python tools/time_lib.py
<config> <seeds> [reps] -- prints ring_s, resident warps/SM and K1 ms (not a bench number)."""
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
gv = sdas.GridView(pipe, grid)
res = sdas.simulate(P, gv)
torch.cuda.synchronize()
ref = res.summary().tobytes()
for r in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sdas.simulate(P, gv, result=res)
    e1.record()
    torch.cuda.synchronize()
    L = res.layout
    print(os.path.basename(os.environ.get("SDAS_LIB", "libsdas.so")), cfg, "lv", L.k1_variant, "ring_s", L.ring_s,
          "warps/SM", L.warps_per_block * L.blocks_per_sm, "ms", round(e0.elapsed_time(e1), 1),
          "same", res.summary().tobytes() == ref, flush=True)
