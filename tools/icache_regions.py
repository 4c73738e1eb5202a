"""Which source regions fill K1's instruction-cache footprint: per 128-B SASS line, its execution count (ncu
source page) and the event-loop statement that inlined it (nvdisasm -gi, the outermost inlined call site).
Prints, per call site, the lines needed for 90 / 99 / 99.9 % of executed instructions.
usage: python tools/icache_regions.py <rep.ncu-rep> <libsdas.so> <kernel-substr> [src-rev]"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, so, kname = sys.argv[1], sys.argv[2], sys.argv[3]
rev = sys.argv[4] if len(sys.argv) > 4 else None
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin") and "host" not in f][0]


def lines_of(flag):
    out = subprocess.run(["nvdisasm", flag, os.path.join(d, cub)], capture_output=True, text=True).stdout
    res, cur, inside = {}, None, False
    for line in out.splitlines():
        if line.startswith("//--------------------- .text."):
            inside = kname in line
            continue
        if not inside:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', line)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", line)
        if m:
            res[int(m.group(1), 16)] = cur
    return res


outer = lines_of("-gi")
csrc = os.path.join(os.path.dirname(os.path.abspath(so)), "csrc", "sdas_k1.cuh")
if rev:
    src = subprocess.run(["git", "show", "%s:paper_2601_03197_b200/csrc/sdas_k1.cuh" % rev], capture_output=True,
                         text=True).stdout.splitlines()
else:
    src = open(csrc).read().splitlines()
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ia, ie = hdr.index("Address"), hdr.index("Instructions Executed")
base, cnt = None, {}
for r in rows[2:]:
    try:
        a = int(r[ia], 16)
        n = float(r[ie].replace(",", "") or 0)
    except (ValueError, IndexError):
        continue
    base = a if base is None else base
    cnt[a - base] = n
tot = sum(cnt.values())
line_n, line_src = collections.Counter(), {}
for a, n in cnt.items():
    line_n[a // 128] += n
for ln in line_n:
    c = collections.Counter(outer.get(a) for a in range(ln * 128, ln * 128 + 128, 16))
    line_src[ln] = c.most_common(1)[0][0]
order = sorted(line_n, key=lambda k: -line_n[k])
band, acc = {}, 0.0
for ln in order:
    acc += line_n[ln]
    band[ln] = 0 if acc <= 0.9 * tot else 1 if acc <= 0.99 * tot else 2 if acc <= 0.999 * tot else 3
agg = collections.defaultdict(lambda: [0, 0, 0, 0, 0.0])
for ln in order:
    agg[line_src[ln]][band[ln]] += 1
    agg[line_src[ln]][4] += line_n[ln] / tot
print("call site (outermost inlined line)               lines <90%  90-99%  99-99.9%  >99.9%   share")
for k, v in sorted(agg.items(), key=lambda kv: -(kv[1][0] + kv[1][1] + kv[1][2])):
    txt = src[k[1] - 1].strip()[:48] if k and k[0] == "sdas_k1.cuh" and 0 < k[1] <= len(src) else ""
    print("%-16s %-48s %4d %7d %8d %7d  %6.2f%%" % ("%s:%d" % k if k else "?", txt, v[0], v[1], v[2], v[3], 100 * v[4]))
