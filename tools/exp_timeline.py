"""Timeline experiment for the fused kernel (needs a -DMPA_DEBUG_TRACE build in $MPATTN_LIB):
per-CTA globaltimer stamps (start, schedule done, first tile landed, loop done, end)."""
import argparse
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import bench
    from paper_2506_13059_b200 import _lib

    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--budget", type=int, default=512)
    a = ap.parse_args()
    args = argparse.Namespace(batch=a.batch, ctx=32768, budget=a.budget, steps=2, warmup=3)
    eng, Q, KN, VN, _ = bench.build_engine(args, 0, torch.device("cuda", 0))
    lib = _lib.lib()
    eng.rotate(Q[0])
    eng.lookup(Q[0])
    import torch as _t
    for _ in range(3):
        eng.lookup(Q[0])
    _t.cuda.synchronize()
    eng.lookup(Q[0])
    _t.cuda.synchronize()
    if os.environ.get("COLD"):
        fa = torch.empty(64 << 20, dtype=torch.float32, device=eng.device)
    for label, fn in (("sparse", lambda: eng.fused()), ("dense", lambda: eng.attend_dense(Q[0]))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        if os.environ.get("COLD"):
            fa.fill_(1.0)
            fa.sum()
            torch.cuda.synchronize()
        fn()
        torch.cuda.synchronize()
        buf = (C.c_ulonglong * (4096 * 8))()
        lib.mpa_debug_trace(buf, 4096 * 8)
        t = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 8).astype(np.int64)
        n = int((t[:, 0] > 0).sum())
        t = t[:296]
        t0 = t[:, 0][t[:, 0] > 0].min()
        rel = (t - t0) / 1e3
        rel[t == 0] = np.nan
        print(label, "ctas", n)
        slow = np.argsort(-np.nan_to_num(rel[:, 4]))[:3]
        for cidx in slow:
            print("   slow cta", cidx, np.round(rel[cidx], 2))
        names = ["start", "sched", "first", "loopend", "end", "seg_sync", "seg_fence", "seg_ticket"]
        if os.environ.get("RAMP"):
            names[5:] = ["ids_issued", "issue0_done", "issue1_done"]
        for k, name in enumerate(names):
            col = rel[:, k]
            print(f"  {name:8s} min {np.nanmin(col):7.2f} med {np.nanmedian(col):7.2f} max {np.nanmax(col):7.2f} us")


if __name__ == "__main__":
    main()
