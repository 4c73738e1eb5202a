"""Small coalesced-run cases for compute-sanitizer (racecheck / memcheck):
   compute-sanitizer --tool racecheck python tools/race_case.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
from paper_2601_03197_b200 import sdas

cases = {
    "config2": lambda: (W.p2_x(), W.grid(W.config2_candidates()[::16], [W.poisson(m) for m in W.P2X_GAPS[::3]],
                                         n_seeds=2, n_requests=120, series_stride=3, series_slots=40,
                                         series_windows=16)),
    "config3": lambda: W.config3(n_seeds=1, n_requests=60),
    "config4": lambda: W.config4(n_seeds=1, n_requests=80, candidates=W.config4_candidates()[::2000]),
    "config1_overload": lambda: W.config1(n_seeds=1, n_requests=300, rates=[6, 7]),
    "kv": lambda: W.config_kv(n_seeds=1, n_requests=80),
    "prio": lambda: W.config_prio(n_seeds=1, n_requests=80, gaps=(726182,)),
    "pace": lambda: W.config_pace(n_seeds=1, n_requests=80, gaps=(726182,)),
}
extra = int(os.environ.get("RACE_FLAGS", "0"))          # e.g. 64 = FLAG_SPILL (two-level rings), 128 cell series
for name in (sys.argv[1:] or list(cases)):
    p, g = cases[name]()
    if extra & sdas.FLAG_CELL_SERIES and not g["series_windows"]:
        g["series_windows"] = 16
    P = sdas.Pipeline(p)
    flags = sdas.FLAG_RECORDS | (sdas.FLAG_SERIES if g["series_stride"] else 0) | extra
    r = sdas.simulate(P, sdas.GridView(p, g, flags=flags))
    torch.cuda.synchronize()
    print(name, "ok", int(r.summary()["completed"].sum()), "k1_variant", r.layout.k1_variant)
