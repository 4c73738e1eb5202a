"""GPU vs oracle event-trace diff for one replica: python tools/trace_diff.py <case> [replica]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch, workloads as W, oracle
from paper_2601_03197_b200 import sdas
from debug_hang import CASES
case = sys.argv[1]; rep = int(sys.argv[2]) if len(sys.argv) > 2 else 0
p, g = eval(CASES[case])
P = sdas.Pipeline(p)
r = sdas.simulate(P, sdas.GridView(p, g, flags=sdas.FLAG_RECORDS, trace_replica=rep, trace_cap=1 << 20))
torch.cuda.synchronize()
o = oracle.simulate(p, g, trace_id=rep, trace_cap=1 << 20)
key = lambda x: (int(x["tick"]), int(x["code"]), int(x["a"]), int(x["b"]), int(x["c"]))
a = sorted(map(key, r.trace())); b = sorted(map(key, o["trace"]))
print(case, "gpu status", r.summary()[rep]["status"], "events", len(a), "oracle", len(b))
for k, (x, y) in enumerate(zip(a, b)):
    if x != y:
        print("first divergence at", k)
        for z in range(max(0, k - 12), min(len(a), k + 6)): print("  gpu", a[z], "   orc", b[z] if z < len(b) else None)
        break
