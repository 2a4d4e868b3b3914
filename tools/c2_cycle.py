"""Per-step device time of the C2 step (graph replay, L2 flushed before each step) across a whole
online-update cycle, bucketed by the local-buffer fill (tokens attended exactly besides the
selection).  python tools/c2_cycle.py [--steps 300]"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import bench

    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--batch", type=int, default=16)
    a = ap.parse_args()
    args = argparse.Namespace(batch=a.batch, ctx=32768, budget=512, steps=a.steps, warmup=3, workload="c2")
    eng, Q, KN, VN, _ = bench.build_engine(args, 0, torch.device("cuda", 0))
    flush = bench.L2Flush(eng.device)
    for i in range(3):
        eng.step(Q[i], KN[i], VN[i])
    torch.cuda.synchronize()
    evs, fill, upd = [], [], []
    st = torch.cuda.current_stream()
    for i in range(a.steps):
        flush(i)
        fill.append(int(eng.cache_len[0] - eng.buffer_start[0]))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        eng.step(Q[3 + i], KN[3 + i], VN[3 + i])
        e1.record(st)
        evs.append((e0, e1))
        upd.append(eng.last_update is not None)
    torch.cuda.synchronize()
    t = np.array([x.elapsed_time(y) * 1e3 for x, y in evs])
    fill, upd = np.array(fill), np.array(upd)
    print(f"captures {eng.n_captures}; update steps {int(upd.sum())}")
    for lo in range(0, 2 * eng.cfg.local_buffer + 1, 16):
        m = (fill >= lo) & (fill < lo + 16) & ~upd
        if m.any():
            print(f"buffer {lo:3d}-{lo + 15:3d}: {m.sum():3d} steps, median {np.median(t[m]):7.1f} us, "
                  f"max {t[m].max():7.1f}")


if __name__ == "__main__":
    main()
