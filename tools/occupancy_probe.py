"""Experiment (not a bench number): K1 time vs resident warps at identical work.  Config-2 replicas with the
tester's inbox capacity padded (never reached: same results, larger shared-memory footprint -> fewer
resident replicas per SM).  usage: python tools/occupancy_probe.py [seeds]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2601_03197_b200 import sdas  # noqa: E402

seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 256
ref = None
for pad in (256, 1024, 1536, 2048, 3072):
    p, g = W.config2(n_seeds=seeds, series_stride=0)
    p["roles"][1]["inbox_cap"] = pad
    P = sdas.Pipeline(p)
    gv = sdas.GridView(p, g)
    r = sdas.simulate(P, gv)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sdas.simulate(P, gv, result=r)
    e1.record()
    torch.cuda.synchronize()
    s = r.summary().tobytes()
    ref = ref or s
    L = r.layout
    print("inbox_cap %5d smem/replica %6d warps/SM %2d (wpb %d x %d) K1 %.1f ms same=%s" % (
        pad, L.smem_per_replica, L.warps_per_block * L.blocks_per_sm, L.warps_per_block, L.blocks_per_sm,
        e0.elapsed_time(e1), s == ref), flush=True)
