"""Experiment (not a bench number): K1 event-loop iterations per replica vs model DES events, by rate and
candidate, from a -DK1_COUNT_ITERS build (summary word 42).  usage:
  SDAS_NVCC_EXTRA=-DK1_COUNT_ITERS python -c "from paper_2601_03197_b200 import build; build.build(True, out='$PWD/paper_2601_03197_b200/libsdas_iters.so')"
  SDAS_LIB=$PWD/paper_2601_03197_b200/libsdas_iters.so python tools/iters.py [config2|config3] [seeds]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2601_03197_b200 import sdas  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "config2"
seeds = int(sys.argv[2]) if len(sys.argv) > 2 else 16
kw = {"series_stride": 0} if cfg == "config2" else {}
p, g = getattr(W, cfg)(n_seeds=seeds, **kw)
for name, fl in (("auto", 0), ("generic", sdas.FLAG_GENERIC)):
    P = sdas.Pipeline(p)
    r = sdas.simulate(P, sdas.GridView(p, g, flags=fl))
    torch.cuda.synchronize()
    s = r.summary()
    it = s["reserved"][:, 0].astype(np.int64)
    des = (s["arrivals"].astype(np.int64) + s["deliveries"] + s["recv_steps"] + s["decode_steps"] + s["window_closes"])
    C, I = len(g["candidates"]), len(g["arrivals"])
    print(name, "lv", r.layout.k1_variant, "iterations/replica %.0f" % it.mean(), "DES/iteration %.2f" % (des.sum() / it.sum()))
    per_rate = it.reshape(I, -1).mean(1)
    print("  iterations/replica by rate:", " ".join("%.0f" % x for x in per_rate))
    print("  msg/replica by rate:", " ".join("%.0f" % x for x in (s["arrivals"] + s["deliveries"]).astype(np.int64).reshape(I, -1).mean(1)))
    w = r.t["work"][: 8 * 32].cpu().numpy().view(np.uint64)
    names = ["WINDOW", "COMPLETE_RECV", "COMPLETE_DECODE", "DELIVER", "ARRIVE", "START_RECV", "START_DECODE"]
    tot_it = it.sum()
    # work words: [0] replica counter, [1 + 1 + f] = pad[1 + f] iterations with flag f, [1 + 8 + f] only flag f
    print("  iterations with flag (share):", ", ".join("%s %.3f" % (n, w[2 + f] / tot_it) for f, n in enumerate(names)))
    print("  iterations with only that flag:", ", ".join("%s %.3f" % (n, w[9 + f] / tot_it) for f, n in enumerate(names)))
    if w[17]:   # pad[16..20]: non-closing RECVs while a batch is held (CHAIN candidates) and why one fails
        print("  chain candidates %d: inbox not empty %d, admission possible %d, delivery due %d, items waiting %d"
              % (w[17], w[18], w[19], w[20], w[21]))
