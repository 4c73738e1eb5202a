import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import oracle, workloads as W
from gpu_parity import run_gpu
p, g = W.config2(n_seeds=3, n_requests=400, series_stride=5, series_windows=64)
a = run_gpu(p, g, series=True); b = run_gpu(p, g, series=True, stepwise=True)
o = oracle.simulate(p, g, series=True)
sa, sb, so = a["series"], b["series"], o["series"]
print("shapes", sa.shape, so.shape)
d = np.argwhere(sa.view(np.uint8).reshape(sa.shape + (16,)).any(-1) != False)
diff = np.argwhere((sa.view(np.uint8).reshape(sa.shape+(16,)) != sb.view(np.uint8).reshape(sb.shape+(16,))).any(-1))
print("n diff (coalesced vs stepwise)", len(diff))
print("n diff (coalesced vs oracle)", int((sa.view(np.uint8).reshape(sa.shape+(16,)) != so.view(np.uint8).reshape(so.shape+(16,))).any(-1).sum()))
print("n diff (stepwise vs oracle)", int((sb.view(np.uint8).reshape(sb.shape+(16,)) != so.view(np.uint8).reshape(so.shape+(16,))).any(-1).sum()))
for k in diff[:10]:
    sl, w, i = k
    rid = sl * 5
    print(k, "rid", rid, "status", int(a["summary"][rid]["status"]), "A", sa[sl, w, i], "B", sb[sl, w, i], "O", so[sl, w, i])
