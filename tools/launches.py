"""Print one line per launch (name, us, DRAM MB) from an ncu --csv --log-file launch list."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
H = {h: j for j, h in enumerate(rows[start])}
agg = {}
for r in rows[start + 1:]:
    if len(r) < len(H):
        continue
    k = (int(r[H["ID"]]), r[H["Kernel Name"]].split("(")[0][-48:])
    agg.setdefault(k, {})[r[H["Metric Name"]]] = float(r[H["Metric Value"]].replace(",", ""))
for (i, name), m in sorted(agg.items()):
    us = m.get("gpu__time_duration.sum", 0) / 1e3
    mb = (m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)) / 1e6
    print(f"{i:3d} {name:48s} {us:8.1f} us {mb:9.2f} MB {mb / max(us, 1e-9):6.2f} TB/s")
