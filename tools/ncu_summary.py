"""Summarise an ncu report (one line per profiled launch) from `ncu -i <rep> --page raw --csv`.

    python tools/ncu_summary.py gpurun_out/step_r01.ncu-rep [--json out.json]
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys

METRICS = {
    "us": "gpu__time_duration.sum",
    "dram_read_MB": "dram__bytes_read.sum",
    "dram_write_MB": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "tensor_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "fp64_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "issue_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "stall_long_sb": "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "stall_short_sb": "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "stall_barrier": "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "stall_wait": "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "stall_mio": "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "stall_math": "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
}
SCALE = {"dram_read_MB": ("byte", 1e-6), "dram_write_MB": ("byte", 1e-6), "us": ("nsecond", 1e-3)}


def rows(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    for row in r[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        rec = {"kernel": d.get("Kernel Name", "?")[:48]}
        for k, m in METRICS.items():
            if m not in d:
                continue
            try:
                v = float(d[m].replace(",", ""))
            except ValueError:
                continue
            unit = u.get(m, "")
            if k == "us":
                v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
                      "second": 1e6, "s": 1e6}.get(unit, 1.0)
            elif k in SCALE:  # bytes -> MB
                v *= {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0) * 1e-6
            rec[k] = round(v, 3)
        yield rec


def main():
    rep = sys.argv[1]
    recs = list(rows(rep))
    for r in recs:
        print(json.dumps(r))
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as fh:
            json.dump(recs, fh, indent=1)


if __name__ == "__main__":
    main()
