"""Print the SASS of a K1 source-line range with per-instruction execution counts from an ncu capture.
usage: python tools/sass_range.py <report.ncu-rep> <libsdas.so> <kernel-substr> <first_line> <last_line>"""
import csv, io, os, re, subprocess, sys, tempfile
rep, so, kname, lo, hi = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]), int(sys.argv[5])
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin") and "host" not in f][0]
sass = subprocess.run(["nvdisasm", "--print-line-info", os.path.join(d, cub)], capture_output=True, text=True).stdout
addr2line, cur, inside = {}, None, False
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
ia, ie, isrc = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Source")
base = None
for r in rows[2:]:
    try:
        a = int(r[ia], 16)
    except (ValueError, IndexError):
        continue
    if base is None:
        base = a
    off = a - base
    if off in addr2line:
        (f, ln), txt = addr2line[off]
        if f == "sdas_k1.cuh" and lo <= ln <= hi:
            print("%6x %5d %10.3g  %s" % (off, ln, float(r[ie] or 0), r[isrc].strip()[:90]))
