"""Aggregate ncu per-SASS-instruction counts by CUDA source line (needs -lineinfo builds).
usage: python tools/sass_lines.py <report.ncu-rep> <libsdas.so> <kernel-substr> [top]
env: COL=<source-page column> ranks lines by that column (e.g. stall_no_inst); REV=<git rev> reads the
source text from that revision (when the profiled build is older than the tree)."""
import csv, io, os, re, subprocess, sys, tempfile, collections
rep, so, kname = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin") and "host" not in f][0]
sass = subprocess.run(["nvdisasm", "--print-line-info", os.path.join(d, cub)], capture_output=True, text=True).stdout
addr2line, cur, inside, fname = {}, None, False, None
for line in sass.splitlines():
    if line.startswith("//--------------------- .text."):
        inside = kname in line
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*)", line)
    if m and cur:
        addr2line[int(m.group(1), 16)] = (cur, m.group(2).strip())
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ia, ie = hdr.index("Address"), hdr.index("Instructions Executed")
isamp = hdr.index(os.environ["COL"]) if os.environ.get("COL") else (hdr.index("# Samples") if "# Samples" in hdr else None)
agg, samp, tot = collections.Counter(), collections.Counter(), 0
base = None
for r in rows[2:]:
    try:
        base = int(r[ia], 16); break
    except (ValueError, IndexError):
        continue
for r in rows[2:]:
    if len(r) <= ie:
        continue
    try:
        a = int(r[ia], 16) - base; n = float(r[ie].replace(",", "") or 0)
    except ValueError:
        continue
    key = addr2line.get(a, (("?", 0), ""))[0]
    agg[key] += n; tot += n
    if isamp is not None:
        try: samp[key] += float(r[isamp].replace(",", "") or 0)
        except ValueError: pass
src = {}
for (f, l) in agg:
    if f not in src:
        p = os.path.join(os.path.dirname(os.path.abspath(so)), "csrc", f)
        if os.environ.get("REV") and os.path.exists(p):
            rel = os.path.relpath(p, subprocess.run(["git", "rev-parse", "--show-toplevel"], capture_output=True,
                                                    text=True).stdout.strip())
            src[f] = subprocess.run(["git", "show", "%s:%s" % (os.environ["REV"], rel)], capture_output=True,
                                    text=True).stdout.splitlines()
        else:
            src[f] = open(p).read().splitlines() if os.path.exists(p) else []
print("total warp instructions %.4g; column %s total %.4g" % (tot, os.environ.get("COL", "# Samples"), sum(samp.values())))
for (f, l), n in (samp if os.environ.get("COL") else agg).most_common(top):
    n = agg[(f, l)]
    s = src.get(f, [])
    txt = s[l - 1].strip()[:90] if 0 < l <= len(s) else ""
    print("%6.2f%% %8.3g  smp %7d  %s:%d  %s" % (100 * n / tot, n, samp[(f, l)], f, l, txt))
