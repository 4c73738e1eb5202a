"""Print K1's launch layout (specialisation level, warps per block, blocks per SM, shared memory per replica)
and one K1 time for a BASELINE config: python tools/layout_probe.py <config> <n_seeds>  (GPU)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2601_03197_b200 import sdas  # noqa: E402

cfg, seeds = sys.argv[1], int(sys.argv[2])
pipe, grid = getattr(W, cfg)(n_seeds=seeds, **({"series_stride": 0} if cfg == "config2" else {}))
P = sdas.Pipeline(pipe)
gv = sdas.GridView(pipe, grid)
res = sdas.simulate(P, gv)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
sdas.simulate(P, gv, result=res)
e1.record()
torch.cuda.synchronize()
L = res.layout
print(cfg, "level", L.k1_variant, "ring_s", L.ring_s, "wpb", L.warps_per_block, "blocks/SM", L.blocks_per_sm,
      "smem/replica", L.smem_per_replica, "K1 ms", round(e0.elapsed_time(e1), 1), flush=True)
