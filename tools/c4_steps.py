"""Per-step device times of the C4 timed loop (bench.py --workload c4): which steps are slow, and
whether they carry an online update.  python tools/c4_steps.py [--runs 1]"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import bench

    args = argparse.Namespace(batch=8, ctx=16384, budget=512, steps=512, warmup=130, workload="c4")
    eng, Q, KN, VN, _ = bench.build_engine(args, 0, torch.device("cuda", 0))
    flush = bench.L2Flush(eng.device)
    for i in range(args.warmup):
        eng.step(Q[i], KN[i], VN[i])
    torch.cuda.synchronize()
    if os.environ.get("ATTEND_LOOP"):  # what bench.py does before timing: 1.5 s of eager attends
        import time

        t_end = time.perf_counter() + 1.5
        while time.perf_counter() < t_end:
            for _ in range(20):
                eng.attend(Q[0])
            torch.cuda.synchronize()
    if os.environ.get("GCFREEZE"):
        import gc

        gc.collect()
        gc.freeze()
    evs, upd = [], []
    stream = torch.cuda.current_stream()
    for i in range(args.steps):
        flush(i)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        eng.step(Q[args.warmup + i], KN[args.warmup + i], VN[args.warmup + i])
        e1.record(stream)
        evs.append((e0, e1))
        upd.append(eng.last_update is not None)
    torch.cuda.synchronize()
    t = np.array([a.elapsed_time(b) * 1e3 for a, b in evs])
    print(f"mean {t.mean():.1f} us  median {np.median(t):.1f}  captures {eng.n_captures}")
    order = np.argsort(-t)[:10]
    for k in order:
        print(f"  step {k:4d} {t[k]:10.1f} us  update={upd[k]}")
    print("sum of update steps ms", round(t[np.array(upd)].sum() / 1e3, 2), "non-update mean",
          round(t[~np.array(upd)].mean(), 1))


if __name__ == "__main__":
    main()
