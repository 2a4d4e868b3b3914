"""Per-source-line warp-stall samples of one kernel: joins ncu's SASS source page (address,
samples) with nvdisasm -g line info from the built library.

    python tools/stall_lines.py <rep> <kernel-regex> <cubin-name-substring> <mangled-substring> [top]

e.g. python tools/stall_lines.py gpurun_out/step_r01.ncu-rep select_worklist mpa_lookup select_worklist_kernelILi4
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

rep, kern, cub_sub, fun_sub = sys.argv[1:5]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 30
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source=sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[1]
si = h.index("Warp Stall Sampling (All Samples)")
rows, seen_first = [], None
for x in r[2:]:
    if len(x) != len(h) or not x[0].startswith("0x"):
        if rows:
            break  # first profiled instance only
        continue
    rows.append((int(x[0], 16), int(x[si] or 0), x[1].strip()))
base = rows[0][0]

tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_2506_13059_b200", "libmpattn.so")], cwd=tmp,
               capture_output=True)
cub = [f for f in glob.glob(os.path.join(tmp, "*.cubin")) if cub_sub in f][0]
sass = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
line_of = {}
cur_line, in_fun = None, False
for ln in sass.splitlines():
    if ln.startswith("//----") and ".text." in ln:
        in_fun = fun_sub in ln
        continue
    if not in_fun:
        continue
    m = re.search(r'line (\d+)', ln)
    if ln.strip().startswith("//##") and m:
        cur_line = int(m.group(1))
        continue
    m = re.search(r'/\*([0-9a-f]{4,})\*/', ln)
    if m and cur_line is not None:
        line_of[int(m.group(1), 16)] = cur_line
agg = collections.Counter()
for addr, s, _ in rows:
    agg[line_of.get(addr - base, -1)] += s
tot = sum(agg.values())
print("samples", tot)
for line, s in agg.most_common(top):
    print(f"  line {line:5d}  {s:6d}  {100.0 * s / max(tot, 1):5.1f}%")
