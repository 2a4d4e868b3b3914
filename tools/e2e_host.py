"""Host cost of the batched end-to-end step (DecodeEngine.step_host): per-call CPU time without
syncs, next to the device-timed e2e step (CUDA events, as bench.py measures it)."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import bench

    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=100)
    a = ap.parse_args()
    args = argparse.Namespace(batch=16, ctx=32768, budget=512, steps=a.steps + 10, warmup=3, workload="c2")
    dev = torch.device("cuda", 0)
    eng, Q, KN, VN, _ = bench.build_engine(args, 0, dev)
    b, Hq, d = Q.shape[1], Q.shape[2], Q.shape[3]
    qh = Q.cpu().pin_memory()
    kh, vh = KN.cpu().pin_memory(), VN.cpu().pin_memory()
    oh = torch.empty(b, Hq, d, dtype=torch.float32).pin_memory()
    for i in range(5):
        eng.step_host(qh[i], kh[i], vh[i], oh)
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    evs, host = [], []
    for i in range(a.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        t0 = time.perf_counter()
        eng.step_host(qh[5 + i], kh[5 + i], vh[5 + i], oh)
        host.append((time.perf_counter() - t0) * 1e6)
        e1.record(st)
        evs.append((e0, e1))
    torch.cuda.synchronize()
    dev_us = sorted(x.elapsed_time(y) * 1e3 for x, y in evs)
    host.sort()
    print(f"step_host: host {host[len(host) // 2]:.1f} us median (p90 {host[int(len(host) * 0.9)]:.1f}), "
          f"device e0->e1 {dev_us[len(dev_us) // 2]:.1f} us median")


if __name__ == "__main__":
    main()
