"""Experiment: GPU vs oracle on many more seeded random feature mixes than the test suite's 120
(tests/random_cases.py), counting the K1 level each case runs.  python tools/exp/random_sweep.py <first> <n>"""
import os
import sys
import collections
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from gpu_parity import full_check  # noqa: E402
from random_cases import make_case, make_lean_case  # noqa: E402

first, n = int(sys.argv[1]), int(sys.argv[2])
lean_only = len(sys.argv) > 3 and sys.argv[3] == "lean"


lv, bad = collections.Counter(), []
for seed in range(first, first + n):
    p, g, obj = (make_lean_case if lean_only else make_case)(seed)
    try:
        a, _ = full_check(p, g, objective=obj)
        lv[a["res"].layout.k1_variant] += 1
    except Exception:
        bad.append(seed)
        traceback.print_exc(limit=2)
print("levels", dict(lv), "failures", bad, flush=True)
