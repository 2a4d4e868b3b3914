"""Warm (no L2 flush) CUDA-event timings of each decode-step kernel launched alone, of eager
prefixes of the step, and of the captured step graph -- the gaps between them show launch
overhead and branch overlap.  Bench workload (C2, batch 16) unless flags say otherwise.

    python tools/step_breakdown.py [--batch 16] [--ctx 32768] [--reps 50]
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
    ap.add_argument("--reps", type=int, default=50)
    a = ap.parse_args()

    import numpy as np
    import torch

    import bench
    from paper_2506_13059_b200._lib import call, ptr, stream_ptr

    bargs = argparse.Namespace(batch=a.batch, ctx=a.ctx, budget=a.budget, steps=4, warmup=3, workload="c2")
    eng, Q, KN, VN, _ = bench.build_engine(bargs, 0, torch.device("cuda", 0))
    for i in range(3):
        eng.step(Q[i], KN[i], VN[i])
    torch.cuda.synchronize()
    q = Q[0]

    def t(fn, reps=a.reps):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e3 / reps

    gk = torch.zeros(eng.n_seq, eng.Hkv, 1, eng.d, device=eng.device)

    def append_only():  # rewrites the same row: counters restored below
        call("mpa_kv_append", eng.cache_struct, ptr(gk), ptr(gk), eng.Hkv, 1, ptr(eng.cache_len_d),
             ptr(eng.ntok_dense_d), ptr(eng.inv_freq), ptr(eng.append_ticket), stream_ptr())
        eng.cache_len_d -= 1
        eng.ntok_dense_d -= 1

    rows = {
        "rotate(lookup view)": lambda: eng.rotate(q, exact=False, lookup=True),
        "rotate(exact view)": lambda: eng.rotate(q, exact=True, lookup=False),
        "lookup (logits + select)": lambda: eng.lookup(q),
        "fused decode": lambda: eng.fused(),
        "append (+2 tiny sub kernels)": append_only,
        "eager rotate+lookup": lambda: (eng.rotate(q), eng.lookup(q)),
        "eager attend": lambda: eng.attend(q),
    }
    out = {k: t(f) for k, f in rows.items()}
    # the step graph (replays advance the cache; bounded reps)
    n0 = int(eng.cache_len[0])
    out["graph step"] = t(lambda: eng.step(Q[1], KN[1], VN[1]), reps=min(a.reps, 40))
    out["graph replay only"] = t(lambda: eng._graph.replay(), reps=min(a.reps, 40))
    # cold: L2 flushed (write + read 256 MB) before each launch, flush excluded from the timing
    fl_a = torch.empty(64 << 20, dtype=torch.float32, device=eng.device)
    fl_b = torch.empty(64 << 20, dtype=torch.float32, device=eng.device)

    def cold(fn, reps=20):
        ts = []
        for _ in range(reps):
            fl_a.fill_(1.0)
            fl_b.sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            ts.append((e0, e1))
        torch.cuda.synchronize()
        return float(np.mean([x.elapsed_time(y) for x, y in ts])) * 1e3

    for k in ("lookup (logits + select)", "fused decode", "eager attend"):
        out[k + " [cold]"] = cold(rows[k])
    out["graph replay only [cold]"] = cold(lambda: eng._graph.replay())
    print(f"batch {a.batch} ctx {a.ctx}: warm per-launch us (cache_len {n0} -> {int(eng.cache_len[0])})")
    for k, v in out.items():
        print(f"  {k:32s} {v:8.1f}")


if __name__ == "__main__":
    main()
