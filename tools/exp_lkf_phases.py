"""Phase timeline of the single-launch decode-step kernel (mpa_decode_step) (needs a -DMPA_DEBUG_TRACE build in $MPATTN_LIB, see
tools/build_debug.sh): per-CTA globaltimer stamps at the phase boundaries, averaged over CTAs."""
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
    ap.add_argument("--cold", action="store_true", help="flush L2 (write + read 256 MB) before the traced launch")
    a = ap.parse_args()
    args = argparse.Namespace(batch=a.batch, ctx=32768, budget=a.budget, steps=2, warmup=3, workload="c2")
    eng, Q, KN, VN, _ = bench.build_engine(args, 0, torch.device("cuda", 0))
    lib = _lib.lib()
    for _ in range(5):
        eng.lookup(Q[0])
    torch.cuda.synchronize()
    if a.cold:
        fa = torch.empty(64 << 20, dtype=torch.float32, device=eng.device)
        fb = torch.empty(64 << 20, dtype=torch.float32, device=eng.device)
        fa.fill_(1.0)
        fb.sum()
        torch.cuda.synchronize()
    eng.lookup(Q[0])
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * (4096 * 16))()
    lib.mpa_debug_trace_step(buf, 4096 * 16)
    n = eng.L * max(1, 128 // eng.L)
    t = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 16).astype(np.int64)[:n]
    t = t[t[:, 15] > 0]
    rel = (t - t[:, 0].min()) / 1e3
    names = {0: "start", 1: "q rotated", 2: "logits", 3: "max", 4: "Z + exact q", 8: "keys", 9: "radix pass 0",
             10: "pass 1", 11: "pass >= 2", 5: "crossing found", 6: "flags + weights", 7: "token list",
             15: "end"}
    print(f"{len(t)} CTAs; mean / max us since the first CTA start")
    prev = 0
    for k, nm in names.items():
        ok = t[:, k] > 0
        if not ok.any():
            continue
        print(f"  {nm:14s} {rel[ok, k].mean():7.2f} {rel[ok, k].max():7.2f}   phase {np.mean(rel[ok, k] - rel[ok, prev]):6.2f}  ({ok.sum()} CTAs)")
        prev = k


if __name__ == "__main__":
    main()
