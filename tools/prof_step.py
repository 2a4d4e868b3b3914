"""Profiling driver: the bench workload (C2, batch 16) with only the steady-state decode steps
inside cudaProfilerStart/Stop, for

    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches.csv python tools/prof_step.py
    ncu --profile-from-start off --set full --clock-control none --import-source on \
        -k regex:decode_mma -c 2 -o gpurun_out/fused python tools/prof_step.py

Flags: --batch, --ctx, --budget, --steps (decode steps captured), --dense (also capture one
dense decode), --hier (C3-like 2-level hierarchy), --update (also capture one online update).
"""

from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--ctx", type=int, default=32768)
    ap.add_argument("--budget", type=int, default=512)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--dense", action="store_true")
    ap.add_argument("--update", action="store_true")
    ap.add_argument("--workload", default="c2", choices=["c2", "c3", "c4", "c5"])
    args = ap.parse_args()

    import torch

    import bench
    from paper_2506_13059_b200 import clustering

    ctx = {"c3": 65536, "c5": 131072, "c4": 16384}.get(args.workload, args.ctx)
    bargs = argparse.Namespace(batch=args.batch, ctx=ctx, budget=args.budget, steps=args.steps, warmup=3,
                               workload=args.workload)
    eng, Q, KN, VN, _ = bench.build_engine(bargs, 0, torch.device("cuda", 0))
    for i in range(3):
        eng.step(Q[i], KN[i], VN[i])
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    for i in range(args.steps):
        eng.step(Q[3 + i], KN[3 + i], VN[3 + i])
    if args.dense:
        eng.attend_dense(Q[0])
    if args.update:
        L = eng.cfg.local_buffer
        need = int(2 * L - (eng.cache_len[0] - eng.buffer_start[0]))
        if need > 0:
            torch.cuda.cudart().cudaProfilerStop()
            eng.write_tokens(torch.randn(eng.n_seq, eng.Hkv, need, eng.d, device=eng.device),
                             torch.randn(eng.n_seq, eng.Hkv, need, eng.d, device=eng.device))
            torch.cuda.synchronize()
            torch.cuda.cudart().cudaProfilerStart()
        clustering.online_update(eng, list(range(eng.n_seq)), eng.cursor)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("profiled", args)


if __name__ == "__main__":
    main()
