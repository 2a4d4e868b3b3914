"""Aggregate per-instruction warp-stall samples of one kernel from an ncu report.

    python tools/sass_stalls.py <rep> <kernel-regex> [top]
"""
import csv, io, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source=sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[1]
rows = [x for x in r[2:] if len(x) == len(h) and x[0].startswith("0x")]
si = h.index("Warp Stall Sampling (All Samples)")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
agg = {c: sum(int(x[h.index(c)] or 0) for x in rows) for c in reasons}
tot = sum(int(x[si] or 0) for x in rows)
print("samples", tot)
for c, v in sorted(agg.items(), key=lambda kv: -kv[1])[:10]:
    print(f"  {c:24s} {v:6d} {100.0 * v / max(tot, 1):5.1f}%")
print("top instructions:")
for x in sorted(rows, key=lambda x: -int(x[si] or 0))[:top]:
    det = {c[6:]: int(x[h.index(c)] or 0) for c in reasons if int(x[h.index(c)] or 0) > 0}
    print(f"  {x[si]:>5s} {x[1].strip()[:60]:60s} {det}")
