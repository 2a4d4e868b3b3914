"""Per-source-line executed warp instructions (and stall samples) of one kernel from an ncu report.

    python tools/inst_lines.py <rep> <kernel-regex> <cubin-substring> <mangled-substring> <source.cu> [top]
"""
import collections
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile

rep, kern, cub_sub, fun_sub, srcf = sys.argv[1:6]
top = int(sys.argv[6]) if len(sys.argv) > 6 else 30
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source=sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[1]
ie, si = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
rows = []
for x in r[2:]:
    if len(x) != len(h) or not x[0].startswith("0x"):
        if rows:
            break
        continue
    rows.append((int(x[0], 16), int(x[ie] or 0), int(x[si] or 0)))
base = rows[0][0]
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_2506_13059_b200", "libmpattn.so")], cwd=tmp,
               capture_output=True)
cub = [f for f in glob.glob(os.path.join(tmp, "*.cubin")) if cub_sub in f][0]
sass = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
line_of, cur, inf = {}, None, False
for ln in sass.splitlines():
    if ln.startswith("//----") and ".text." in ln:
        inf = fun_sub in ln
        continue
    if not inf:
        continue
    m = re.search(r'line (\d+)', ln)
    if ln.strip().startswith("//##") and m:
        cur = int(m.group(1))
        continue
    m = re.search(r'/\*([0-9a-f]{4,})\*/', ln)
    if m and cur is not None:
        line_of[int(m.group(1), 16)] = cur
ins, smp = collections.Counter(), collections.Counter()
for a, n, s in rows:
    ins[line_of.get(a - base, -1)] += n
    smp[line_of.get(a - base, -1)] += s
ti, ts = sum(ins.values()), sum(smp.values())
print(f"instructions {ti}  samples {ts}")
src = open(srcf).read().splitlines()
for l, n in ins.most_common(top):
    txt = src[l - 1].strip()[:70] if 0 < l <= len(src) else ""
    print(f"{l:5d} {n:9d} {100 * n / ti:5.1f}%  smp {100 * smp[l] / max(ts, 1):5.1f}%  {txt}")
